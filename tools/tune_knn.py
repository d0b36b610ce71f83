"""Time kNN variants (AIDW_KNN_VARIANT, AIDW_KNN_FILTER) on C4; check r_obs bit-exact on a sample."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch

import datagen
import paper_1511_02186_b200 as P

CFG = os.environ.get("TUNE_CFG", "C4")  # any BASELINE config (its data, queries and k)
K = datagen.CONFIGS[CFG]["k"]
nq = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else datagen.CONFIGS[CFG]["nq"]
x, y, z = datagen.make_data(CFG)
qx, qy = datagen.make_queries(CFG, nq=nq)
eng = P.AIDW(x, y, z)
tq = lambda v: torch.as_tensor(v, dtype=torch.float32, device="cuda")
qx_t, qy_t = tq(qx), tq(qy)
r = torch.empty(nq, device="cuda"); d1 = torch.empty_like(r); mm = torch.empty(2, device="cuda")
for _ in range(2):
    P.aidw_knn_robs(eng.h, qx_t, qy_t, K, r, d1, mm)
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.aidw_knn_robs(eng.h, qx_t, qy_t, K, r, d1, mm); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
out = {"cfg": CFG, "nq": nq, "split": os.environ.get("AIDW_SPLIT", "auto"), "variant": os.environ.get("AIDW_KNN_VARIANT", "0"), "filter": os.environ.get("AIDW_KNN_FILTER", "1"),
       "knn_ms": min(ts), "gpairs_per_s": nq * len(x) / (min(ts) / 1e3) / 1e9}
if "--check" in sys.argv:
    import oracle
    sub = np.arange(0, nq, max(1, nq // 64))
    ro = oracle.knn_f32(x, y, qx[sub], qy[sub], K)
    out["bit_exact_sample"] = bool(np.array_equal(r.cpu().numpy()[sub], ro))
print(out, flush=True)
