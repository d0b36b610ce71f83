"""Time every BASELINE.json config (C1..C5) on one GPU, GLOBAL bounds, per stage
(CUDA events, median of 3 after 1 warm-up), in each config's precision(s).
usage: python tools/configs_bench.py [--out profiles/r01_configs.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import datagen
import paper_1511_02186_b200 as P

LV = datagen.ALPHA_LEVELS


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        e[0].record()
        fn()
        e[1].record()
        e[1].synchronize()
        ts.append(e[0].elapsed_time(e[1]))
    return float(np.median(ts))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--configs", default="C1,C2,C3,C4,C5")
    ap.add_argument("--dtypes", default=None, help="override the configs' precisions, e.g. f64")
    args = ap.parse_args()
    res = []
    for name in args.configs.split(","):
        cfg = datagen.CONFIGS[name]
        x, y, z = datagen.make_data(name)
        qx, qy = datagen.make_queries(name)
        for dt_name in (args.dtypes.split(",") if args.dtypes else cfg["dtypes"]):
            dt = torch.float32 if dt_name == "f32" else torch.float64
            eng = P.AIDW(x, y, z, dtype=dt)
            dev = torch.device("cuda")
            tqx = torch.as_tensor(qx, dtype=dt, device=dev)
            tqy = torch.as_tensor(qy, dtype=dt, device=dev)
            nq, k = len(qx), cfg["k"]
            r = torch.empty(nq, dtype=dt, device=dev)
            d1 = torch.empty_like(r)
            mm = torch.empty(2, dtype=dt, device=dev)
            a = torch.empty_like(r)
            zo = torch.empty_like(r)
            knn = timed(lambda: P.aidw_knn_robs(eng.h, tqx, tqy, k, r, d1, mm))
            alp = timed(lambda: P.aidw_alpha(eng.h, r, LV, P.GLOBAL, 0, 0, mm, P.NORMALIZED, a))
            itp = timed(lambda: P.aidw_interpolate(eng.h, tqx, tqy, a, d1, zo))
            tot = knn + alp + itp
            row = {"config": name, "dtype": dt_name, "nd": len(x), "nq": nq, "k": k,
                   "data": cfg["data"], "queries": cfg["queries"], "knn_ms": knn, "alpha_ms": alp,
                   "interp_ms": itp, "total_ms": tot, "points_per_s": nq / (tot / 1e3),
                   "pair_evals_per_s": 2.0 * nq * len(x) / (tot / 1e3),
                   "frac_alpha_1": float((a == 1.0).float().mean()),
                   "frac_alpha_3": float((a == 3.0).float().mean())}
            res.append(row)
            print(json.dumps(row), flush=True)
            eng.close()
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
