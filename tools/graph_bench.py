"""Eager stage calls vs one CUDA-graph replay of the whole path (AIDW.capture) for the
small BASELINE configs, where launch overhead is visible.  Device time per step
(CUDA events, median of 20 after warm-up).
usage: python tools/graph_bench.py [--out profiles/r01_graph.json]"""
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


def timed(fn, reps=20):
    for _ in range(3):
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
    rows = []
    for name, dt in (("C1", torch.float64), ("C2", torch.float32), ("C2", torch.float64), ("C3", torch.float32)):
        cfg = datagen.CONFIGS[name]
        x, y, z = datagen.make_data(name)
        qx, qy = datagen.make_queries(name)
        eng = P.AIDW(x, y, z, dtype=dt)
        tqx = torch.as_tensor(qx, dtype=dt, device="cuda")
        tqy = torch.as_tensor(qy, dtype=dt, device="cuda")
        k = cfg["k"]
        eager = timed(lambda: eng.run(tqx, tqy, k, LV, P.GLOBAL))
        g = eng.capture(len(qx), k, LV, P.GLOBAL)
        g.qx.copy_(tqx)
        g.qy.copy_(tqy)
        graph = timed(lambda: g.replay())
        same = bool(torch.equal(g.z, eng.run(tqx, tqy, k, LV, P.GLOBAL)))
        row = {"config": name, "dtype": str(dt).split(".")[-1], "nd": len(x), "nq": len(qx), "k": k,
               "eager_ms": eager, "graph_ms": graph, "bit_identical": same}
        rows.append(row)
        print(json.dumps(row), flush=True)
        eng.close()
    if args.out:
        json.dump(rows, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
