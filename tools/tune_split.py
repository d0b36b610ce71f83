"""Small-nq data split sweep: kNN and weighting stage times for
C2 / C3 and the C4 data set with 1/2..1/64 of its queries (a strong-scaled rank's
share), under AIDW_SPLIT = 0 (off), auto, and forced factors.
usage: python tools/tune_split.py [--out profiles/r01_split.jsonl]"""
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


def timed(fn, reps=5):
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
    args = ap.parse_args()
    cases = [("C2", 1), ("C3", 1)] + [("C4", d) for d in (1, 2, 4, 8, 16, 64)]
    rows = []
    cache = {}
    for name, div in cases:
        cfg = datagen.CONFIGS[name]
        if name not in cache:
            cache[name] = (datagen.make_data(name), datagen.make_queries(name))
        (x, y, z), (qx, qy) = cache[name]
        nq = len(qx) // div
        eng = P.AIDW(x, y, z)
        tqx = torch.as_tensor(qx[:nq], device="cuda")
        tqy = torch.as_tensor(qy[:nq], device="cuda")
        k = cfg["k"]
        r, d1, mm = eng.knn_robs(tqx, tqy, k)
        a = eng.alpha(r, LV, P.GLOBAL, 0, 0, mm)
        for sv in ("0", "auto", "2", "4", "8", "16", "32"):
            if sv == "auto":
                os.environ.pop("AIDW_SPLIT", None)
            else:
                os.environ["AIDW_SPLIT"] = sv
            knn = timed(lambda: eng.knn_robs(tqx, tqy, k))
            itp = timed(lambda: eng.interpolate(tqx, tqy, a, d1))
            row = {"case": f"{name}/{div}", "nd": len(x), "nq": nq, "k": k, "split": sv, "knn_ms": knn,
                   "interp_ms": itp}
            rows.append(row)
            print(json.dumps(row), flush=True)
        os.environ.pop("AIDW_SPLIT", None)
        eng.close()
    if args.out:
        with open(args.out, "w") as f:
            for r in rows:
                f.write(json.dumps(r) + "\n")


if __name__ == "__main__":
    main()
