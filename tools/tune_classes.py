"""Weighting-pass time per exact-exponent class: constant alpha in {1, 1.5, 2, 3} on C4."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import datagen
import paper_1511_02186_b200 as P

nq = int(sys.argv[1]) if len(sys.argv) > 1 else 1024000
x, y, z = datagen.make_data("C4")
qx, qy = datagen.make_queries("C4", nq=nq)
eng = P.AIDW(x, y, z)
tq = lambda v: torch.as_tensor(v, dtype=torch.float32, device="cuda")
qx_t, qy_t = tq(qx), tq(qy)
r, d1, mm = eng.knn_robs(qx_t, qy_t, 10)
zo = torch.empty(nq, device="cuda")
for av in (1.0, 1.5, 2.0, 3.0):
    a = torch.full((nq,), av, device="cuda")
    P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print({"alpha": av, "interp_ms": min(ts)}, flush=True)
# mixes
g = torch.Generator(device="cuda").manual_seed(0)
u = torch.rand(nq, device="cuda", generator=g)
for frac in (0.0, 0.2, 0.5):
    a = torch.where(u < frac, torch.tensor(1.0, device="cuda"), torch.tensor(1.5, device="cuda"))
    P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo)
    ts = []
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo); e1.record(); e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    print({"mix_frac_alpha1": frac, "interp_ms": min(ts)}, flush=True)
# the real GLOBAL alphas
a = eng.alpha(r, datagen.ALPHA_LEVELS, P.GLOBAL, 0, 0, mm)
print({"global_frac_alpha1": float((a == 1.0).float().mean()), "frac_alpha3": float((a == 3.0).float().mean())})
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); P.aidw_interpolate(eng.h, qx_t, qy_t, a, d1, zo); e1.record(); e1.synchronize()
    ts.append(e0.elapsed_time(e1))
print({"global_alphas_interp_ms": min(ts)}, flush=True)
