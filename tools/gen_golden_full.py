"""Write the full-size golden record of a BASELINE config from the CPU oracle ONLY.

    python tools/gen_golden_full.py --config C4 [--dtypes f32,f64] [--chunk 65536]

Output: ``tests/golden/full_<cfg>.json``.  Every value in it comes from ``oracle/``
(plain C, the paper's steps) on the seeded ``datagen`` inputs -- nothing from the CUDA
path -- so ``tests/test_gpu.py::test_full_size_golden_*`` can compare the GPU's full
arrays against it without feeding any CUDA-derived value into the oracle chain.

Per working precision (f32 = the float instantiation with the R16 sequence, f64 = the
fp64 oracle), over ALL nq queries:
* SHA-256 of r_obs (Eq. 3), of d1^2 (the nearest squared distance)
  and of the ascending k-distance lists (§3.1.2), little-endian, in
  query order; the same hashes per chunk of ``chunk`` queries (to localise a mismatch);
* min / max of r_obs and their first argmin / argmax (the GLOBAL bounds, PAPER.md:221-223,
  DESIGN.md R7).
Then, from the fp64 chain: the bbox area and r_exp (Eq. 2), the GLOBAL
R_min / R_max = min/max r_obs / r_exp, and on a fixed query sample (strided + the
extreme queries) r_obs, alpha (Eqs. 4-6) and Z (Eq. 1) in GLOBAL and FIXED(0, 2) modes.
If f64 is not requested, the sample's chain uses the f32 record's bounds (noted in the
file as ``bounds_from``).

Cost (oracle_knn ~4.5 ns (f32) / 6.5 ns (f64) per pair per core): C4 ~10 / 14 min on 8
cores, C5 ~80 / 115 min.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import datagen  # noqa: E402
import oracle  # noqa: E402


def sample_indices(nq: int, n: int = 1021) -> np.ndarray:
    step = max(1, nq // n)
    return np.unique(np.concatenate([np.arange(0, nq, step), [nq - 1]])).astype(np.int64)


def knn_record(x, y, qx, qy, k, dtype, chunk, log):
    fn = oracle.knn_f32 if dtype == "f32" else oracle.knn_f64
    npdt = np.float32 if dtype == "f32" else np.float64
    nq = len(qx)
    h = {n: hashlib.sha256() for n in ("r_obs", "d1sq", "dists")}
    chunks = {n: [] for n in h}
    robs_all = np.empty(nq, npdt)
    d1_all = np.empty(nq, npdt)
    t0 = time.time()
    for c0 in range(0, nq, chunk):
        c1 = min(nq, c0 + chunk)
        r, d, d1 = fn(x, y, qx[c0:c1], qy[c0:c1], k, want_dists=True, want_d1sq=True)
        robs_all[c0:c1] = r
        d1_all[c0:c1] = d1
        for n, a in (("r_obs", r), ("d1sq", d1), ("dists", d)):
            b = np.ascontiguousarray(a, dtype=np.dtype(npdt).newbyteorder("<")).tobytes()
            h[n].update(b)
            chunks[n].append(hashlib.sha256(b).hexdigest())
        el = time.time() - t0
        log(f"  {dtype} kNN {c1}/{nq} queries, {el:.0f} s (eta {el / c1 * (nq - c1):.0f} s)")
    rec = {
        "sha256": {n: v.hexdigest() for n, v in h.items()},
        "chunk_sha256": chunks,
        "r_obs_min": float(robs_all.min()), "r_obs_max": float(robs_all.max()),
        "argmin": int(np.argmin(robs_all)), "argmax": int(np.argmax(robs_all)),
        "kNN_seconds": time.time() - t0, "threads": oracle.num_threads(),
    }
    return rec, robs_all, d1_all


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--dtypes", default="f32,f64")
    ap.add_argument("--chunk", type=int, default=65536)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    cfg = datagen.CONFIGS[a.config]
    out = a.out or os.path.join(ROOT, "tests", "golden", f"full_{a.config}.json")
    log = lambda m: print(m, flush=True)  # noqa: E731

    x, y, z = datagen.make_data(a.config)
    qx, qy = datagen.make_queries(a.config)
    nd, nq, k = len(x), len(qx), cfg["k"]
    lv = datagen.ALPHA_LEVELS
    rec = {
        "config": a.config, "nd": nd, "nq": nq, "k": k, "levels": list(lv),
        "generator": "tools/gen_golden_full.py (oracle/ only; datagen inputs)",
        "layout": "little-endian, query order; dists [nq][k] ascending distances (sqrt of R16's s)",
        "chunk": a.chunk,
    }
    robs = {}
    for dt in a.dtypes.split(","):
        log(f"{a.config}: {dt} kNN over {nq} x {nd}")
        rec[dt], robs[dt], _ = knn_record(x, y, qx, qy, k, dt, a.chunk, log)
        with open(out + ".partial", "w") as f:
            json.dump(rec, f, indent=1)

    # the fp64 chain: Eq. 2 -> GLOBAL bounds -> Eqs. 4-6 -> Eq. 1 on the sample
    A = oracle.bbox_area(x, y)
    re = oracle.r_exp(nd, A)
    src = "f64" if "f64" in robs else "f32"
    rmin, rmax = oracle.r_bounds(robs[src].astype(np.float64), re, oracle.GLOBAL)
    sub = np.unique(np.concatenate([sample_indices(nq)] + [[rec[d]["argmin"], rec[d]["argmax"]] for d in robs]))
    r64 = oracle.knn_f64(x, y, qx[sub], qy[sub], k)
    a_g = oracle.alpha(r64, re, lv, rmin, rmax)
    a_f = oracle.alpha(r64, re, lv, 0.0, 2.0)
    log(f"  Z on {len(sub)} sampled queries")
    z_g = oracle.idw(x, y, z, qx[sub], qy[sub], a_g)
    z_f = oracle.idw(x, y, z, qx[sub], qy[sub], a_f)
    rec["chain"] = {
        "area": A, "r_exp": re, "R_min": rmin, "R_max": rmax, "bounds_from": src,
        "sample": sub.tolist(), "r_obs_f64": r64.tolist(),
        "alpha_global": a_g.tolist(), "Z_global": z_g.tolist(),
        "alpha_fixed_0_2": a_f.tolist(), "Z_fixed_0_2": z_f.tolist(),
    }
    with open(out, "w") as f:
        json.dump(rec, f, indent=1)
    if os.path.exists(out + ".partial"):
        os.remove(out + ".partial")
    log(f"wrote {out}")


if __name__ == "__main__":
    main()
