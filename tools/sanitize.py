"""Small end-to-end runs of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): GLOBAL and FIXED paths, fp32 + fp64, IDW, data-sharded partials, the paper
baselines, coincident queries and ragged sizes."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import datagen
import paper_1511_02186_b200 as P

LV = datagen.ALPHA_LEVELS
x, y, z, qx, qy = datagen.random_cloud(5, 3001, 777)
qx = np.concatenate([qx, x[:3]])
qy = np.concatenate([qy, y[:3]])
for dt in (torch.float32, torch.float64):
    eng = P.AIDW(x, y, z, dtype=dt)
    eng.run(qx, qy, 10, LV, P.GLOBAL)
    eng.run(qx, qy, 15, [1, 1, 2, 3, 3], P.FIXED, 0.0, 2.0)
    eng.run_fixed(qx, qy, 10)
    eng.idw(qx, qy, 2.0)
    eng.knn_robs(qx, qy, 32, want_dists=True)
    s = eng.knn_partial(qx, qy, 10)
    r, d1, mm = eng.knn_merge(s, 1, len(qx), 10)
    a = eng.alpha(r, LV, P.GLOBAL, 0, 0, mm)
    eng.finalize(eng.interpolate_partial(qx, qy, a, d1), 1, len(qx))
    t = torch.as_tensor(np.concatenate([x, y, z]), dtype=dt, device="cuda")
    zo = torch.empty(len(qx), dtype=dt, device="cuda")
    for v in (0, 1):
        P.aidw_paper_baseline(v, t, len(x), torch.as_tensor(qx, dtype=dt, device="cuda"),
                              torch.as_tensor(qy, dtype=dt, device="cuda"), 10, LV, eng.area, 0, 2, zo)
    # per-query seed at the sorted copy's end (nd close to k: j0 clamped to nd - k) and a
    # query outside the data bbox; small-grid (Q = 1) weighting
    small = P.AIDW(x[:40], y[:40], z[:40], dtype=dt)
    small.knn_robs(np.append(qx, 3.5), np.append(qy, -2.0), 32, want_dists=True)
    small.run(qx, qy, 32, LV, P.GLOBAL)
    small.close()
    # large batch: spatial query order + Q = 4 kNN (fp32), unsplit launches
    _, _, _, bx, by = datagen.random_cloud(6, 10, 40000)
    eng.run(bx, by, 10, LV, P.GLOBAL)
    eng.run_fixed(bx, by, 10)
    os.environ["AIDW_SPLIT"] = "0"
    eng.run(qx, qy, 10, LV, P.GLOBAL)
    eng.run(bx, by, 10, LV, P.GLOBAL)  # unsplit ordered batch (fp16 pre-filter from tile 1)
    del os.environ["AIDW_SPLIT"]
    os.environ["AIDW_KNN_H16"] = "2"  # the Q = 4 fp16 pre-filter kernel
    eng.run(bx, by, 10, LV, P.GLOBAL)
    del os.environ["AIDW_KNN_H16"]
    eng.run(bx, by, 15, LV, P.GLOBAL)  # k = 15 ordered: the fp16 kernel with the strip test
    os.environ["AIDW_KNN_STRIP"] = "0"  # the fp16 kernels without the strip pre-test
    eng.run(bx, by, 10, LV, P.GLOBAL)
    del os.environ["AIDW_KNN_STRIP"]
    # device-side bounds exchange with one rank (push, wait, acks)
    eng.exchange_connect([eng.exchange_setup(0, 1)])
    for _ in range(3):
        eng.run(qx, qy, 10, LV, P.GLOBAL)
    eng.exchange_close()
    torch.cuda.synchronize()
    eng.check()
print("sanitize run ok")
