"""Probe: do the kNN pass of one batch and the weighting pass of another overlap on
one B200 when launched on two streams (two handles over the same data)?  Prints the
time of each alone and of both together (C4 sizes)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import datagen
import paper_1511_02186_b200 as P

x, y, z = datagen.make_data("C4")
qa, qb = datagen.make_queries("C4"), datagen.make_queries("C4", seed=77)
h1, h2 = P.AIDW(x, y, z), P.AIDW(x, y, z)
t = lambda v: torch.as_tensor(v, dtype=torch.float32, device="cuda")
ax, ay, bx, by = t(qa[0]), t(qa[1]), t(qb[0]), t(qb[1])
r, d1, mm = h1.knn_robs(ax, ay, 10)
al = h1.alpha(r, datagen.ALPHA_LEVELS, P.GLOBAL, 0, 0, mm)
pr = [int(v) for v in os.environ.get("PRIO", "0,0").split(",")]
s1 = torch.cuda.Stream(priority=pr[0])
s2 = torch.cuda.Stream(priority=pr[1])
rb = torch.empty(len(qb[0]), device="cuda"); d1b = torch.empty_like(rb); mmb = torch.empty(2, device="cuda")
zo = torch.empty(len(qa[0]), device="cuda")


def knn():
    P.aidw_knn_robs(h2.h, bx, by, 10, rb, d1b, mmb, stream=s1)


def interp():
    P.aidw_interpolate(h1.h, ax, ay, al, d1, zo, stream=s2)


def timed(fn, n=2):
    best = 1e30
    for _ in range(n):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        for s in (s1, s2):
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


torch.cuda.current_stream().synchronize()
for s in (s1, s2):
    s.wait_stream(torch.cuda.current_stream())
tk = timed(knn)
ti = timed(interp)
tki = timed(lambda: (knn(), interp()))
tik = timed(lambda: (interp(), knn()))
print({"prio": pr, "knn_ms": tk, "interp_ms": ti, "sum_ms": tk + ti, "both_knn_first_ms": tki,
       "both_interp_first_ms": tik}, flush=True)
