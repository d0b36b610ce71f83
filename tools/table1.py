"""N3: Table-1-shaped ablation on B200 (§4.1; Figs. 4-7).

The paper times, at n = m = 10K..1000K (K = 1024) random points in a square, its CPU
version (fp64, sequential) and four GPU versions (naive/tiled x SoA/AoaS, fp32), plus
fp64 GPU runs.  This script runs the same grid on one B200 with:
  * the paper's designs recompiled for sm_100a (aidw_paper_baseline: naive, tiled;
    SoA, AoaS; fp32, fp64) -- FIXED bounds (0, 2), the paper's per-thread structure;
  * this repo's path: fused FIXED kernel (aidw_run_fixed) and the GLOBAL 3-kernel path;
  * the CPU oracle (all host cores), timed on a query sample and scaled to the full
    size (per-query cost is exactly nd pairs) -- labelled as extrapolated.
Times are device times (CUDA events) of the compute only, median of 3 after 1 warm-up.
Writes a markdown table (stdout and --out) and JSON lines (--json).

usage: python tools/table1.py [--sizes 10,50,100,500,1000] [--out profiles/r01_table1.md]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import datagen
import paper_1511_02186_b200 as P

LV = datagen.ALPHA_LEVELS
PAPER_MS = {  # PAPER.md:555-593 (GT 730M / i7-4700MQ), sizes in K
    "cpu": {10: 6791, 50: 168234, 100: 673806, 500: 16852984, 1000: 67471402},
    "naive_soa": {10: 65.3, 50: 863, 100: 2884, 500: 63599, 1000: 250574},
    "naive_aoas": {10: 66.3, 50: 875, 100: 2933, 500: 64593, 1000: 254488},
    "tiled_soa": {10: 61.3, 50: 714, 100: 2242, 500: 43843, 1000: 168189},
    "tiled_aoas": {10: 61.6, 50: 722, 100: 2276, 500: 44891, 1000: 172605},
}


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="10,50,100,500,1000")
    ap.add_argument("--out", default=None)
    ap.add_argument("--json", default=None)
    ap.add_argument("--skip-fp64-paper-above", type=int, default=1000)
    ap.add_argument("--cpu-sample", type=int, default=64)
    args = ap.parse_args()
    sizes = [int(s) for s in args.sizes.split(",")]
    rows = []
    for K in sizes:
        n = K * datagen.K_SIZE
        x, y, z = datagen.make_data({"nd": n, "data": "uniform"}, seed=2000 + K)
        qx, qy = datagen.uniform_points(2000 + K, n, datagen.S_QX, datagen.S_QY)
        r = {"size_K": K, "n": n}
        for dt_name, dt in (("f32", torch.float32), ("f64", torch.float64)):
            eng = P.AIDW(x, y, z, dtype=dt)
            area = eng.area
            dev = torch.device("cuda")
            tq = lambda v: torch.as_tensor(v, dtype=dt, device=dev)
            tqx, tqy = tq(qx), tq(qy)
            zo = torch.empty(n, dtype=dt, device=dev)
            soa = torch.as_tensor(np.concatenate([x, y, z]), dtype=dt, device=dev)
            aoas = torch.as_tensor(np.stack([x, y, z, np.zeros_like(x)], 1).reshape(-1), dtype=dt, device=dev)
            r[f"ours_fixed_{dt_name}"] = timed(
                lambda: P.aidw_run_fixed(eng.h, tqx, tqy, 10, LV, 0.0, 2.0, P.NORMALIZED, zo))
            r[f"ours_global_{dt_name}"] = timed(lambda: eng.run(tqx, tqy, 10, LV, P.GLOBAL))
            if dt_name == "f64" and K > args.skip_fp64_paper_above:
                continue
            for var, vname in ((0, "naive"), (1, "tiled")):
                for lay, lname, buf in ((P.SOA, "soa", soa), (P.AOAS, "aoas", aoas)):
                    r[f"paper_{vname}_{lname}_{dt_name}"] = timed(
                        lambda: P.aidw_paper_baseline(var, buf, n, tqx, tqy, 10, LV, area, 0.0, 2.0, zo, lay),
                        reps=1 if K >= 500 else 3)
            eng.close()
        # CPU oracle on a sample, scaled (per query cost = n pairs x 2 passes)
        import oracle
        m = min(args.cpu_sample, n)
        t0 = time.perf_counter()
        robs = oracle.knn_f64(x, y, qx[:m], qy[:m], 10)
        a = oracle.alpha(robs, oracle.r_exp(n, oracle.bbox_area(x, y)), LV, 0.0, 2.0)
        oracle.idw(x, y, z, qx[:m], qy[:m], a)
        dt_cpu = time.perf_counter() - t0
        r["cpu_oracle_ms_extrapolated"] = dt_cpu * 1e3 * n / m
        r["cpu_cores"] = oracle.num_threads()
        rows.append(r)
        print(json.dumps(r), flush=True)

    def fmt(v):
        return "—" if v is None else (f"{v:,.1f}" if v < 1e5 else f"{v:,.0f}")

    lines = ["| version | layout | prec | " + " | ".join(f"{K}K" for K in sizes) + " |",
             "|---|---|---|" + "---|" * len(sizes)]
    spec = [("CPU oracle (all host cores, extrapolated)", "—", "f64", "cpu_oracle_ms_extrapolated")]
    for dt_name in ("f32", "f64"):
        for vname in ("naive", "tiled"):
            for lname in ("soa", "aoas"):
                spec.append((f"paper {vname} (sm_100a)", lname.upper() if lname == "soa" else "AoaS", dt_name,
                             f"paper_{vname}_{lname}_{dt_name}"))
        spec.append(("this repo: fused FIXED (aidw_run_fixed)", "SoA", dt_name, f"ours_fixed_{dt_name}"))
        spec.append(("this repo: GLOBAL 3 kernels", "SoA", dt_name, f"ours_global_{dt_name}"))
    for label, lay, prec, key in spec:
        lines.append(f"| {label} | {lay} | {prec} | " + " | ".join(fmt(r.get(key)) for r in rows) + " |")
    for key, label in (("cpu", "paper CPU (i7-4700MQ, 1 core)"), ("naive_soa", "paper naive SoA (GT 730M)"),
                       ("tiled_soa", "paper tiled SoA (GT 730M)")):
        lines.append(f"| {label} | | {'f64' if key == 'cpu' else 'f32'} | " +
                     " | ".join(fmt(PAPER_MS[key].get(K)) for K in sizes) + " |")
    table = "\n".join(lines)
    print(table)
    if args.out:
        with open(args.out, "w") as f:
            f.write("# Table-1-shaped ablation on one B200 (ms; N3, tools/table1.py)\n\n")
            f.write("Device time of the compute (CUDA events, median of 3; 1 rep at >= 500K for the paper "
                    "kernels). n = m = K x 1024 uniform points; k = 10; FIXED bounds (0, 2) except the GLOBAL row; "
                    "paper rows at the bottom are PAPER.md:555-593 (other hardware, context only).\n\n")
            f.write(table + "\n")
    if args.json:
        with open(args.json, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
