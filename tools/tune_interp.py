"""Time interp variants (AIDW_INTERP_VARIANT) on C4 and check accuracy on a sample.
Run one variant per process (AIDW_INTERP_VARIANT=v): python tools/tune_interp.py [nq] [--check]"""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import datagen
import paper_1511_02186_b200 as P

nq = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 1024000
x, y, z = datagen.make_data("C4")
qx, qy = datagen.make_queries("C4", nq=nq)
eng = P.AIDW(x, y, z)
tq = lambda v: torch.as_tensor(v, dtype=torch.float32, device="cuda")
qx_t, qy_t = tq(qx), tq(qy)
r, d1, mm = eng.knn_robs(qx_t, qy_t, 10)
a = eng.alpha(r, datagen.ALPHA_LEVELS, P.GLOBAL, 0, 0, mm)
zo = torch.empty(nq, device="cuda")
for _ in range(2):
    P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
out = {"variant": os.environ.get("AIDW_INTERP_VARIANT", "0"), "q1": os.environ.get("AIDW_INTERP_Q1", "auto"),
       "nq": nq, "interp_ms": min(ts),
       "gpairs_per_s": nq * len(x) / (min(ts) / 1e3) / 1e9}
if "--check" in sys.argv:
    import oracle
    sub = np.arange(0, nq, max(1, nq // 48))
    Zo = oracle.idw(x, y, z, qx[sub], qy[sub], a.cpu().numpy()[sub].astype(np.float64))
    out["max_rel_err"] = float(np.max(np.abs(zo.cpu().numpy()[sub] - Zo) / Zo))
print(out, flush=True)
