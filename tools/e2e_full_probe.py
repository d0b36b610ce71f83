"""Where the e2e_full time goes (bench.py e2e_full): aidw_create from pinned host data,
the first run_host step on the fresh handle (its scratch allocations), a second step on
the same handle, and aidw_destroy -- host wall clock, C4 sizes, 3 repetitions."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import datagen
import paper_1511_02186_b200 as P

x, y, z = datagen.make_data("C4")
qx, qy = datagen.make_queries("C4")
hdata = torch.stack([torch.as_tensor(v, dtype=torch.float32) for v in (x, y, z)]).contiguous().pin_memory()
hx = torch.as_tensor(qx, dtype=torch.float32).pin_memory()
hy = torch.as_tensor(qy, dtype=torch.float32).pin_memory()
hz = torch.empty(len(qx), dtype=torch.float32).pin_memory()
warm = P.AIDW.from_host(hdata, device=0)
warm.run_host(hx, hy, 10, datagen.ALPHA_LEVELS, P.GLOBAL, out=hz)
warm.close()
torch.cuda.synchronize()
for rep in range(3):
    t = [time.perf_counter()]
    eng = P.AIDW.from_host(hdata, device=0)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eng.run_host(hx, hy, 10, datagen.ALPHA_LEVELS, P.GLOBAL, out=hz)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eng.run_host(hx, hy, 10, datagen.ALPHA_LEVELS, P.GLOBAL, out=hz)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    eng.close()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    d = [1e3 * (b - a) for a, b in zip(t, t[1:])]
    print(json.dumps({"rep": rep, "create_ms": d[0], "first_step_ms": d[1], "second_step_ms": d[2], "destroy_ms": d[3]}),
          flush=True)

# stage split of a fresh handle's first step vs its second (device-resident queries)
dqx = hx.cuda()
dqy = hy.cuda()
for rep in range(2):
    eng = P.AIDW.from_host(hdata, device=0)
    torch.cuda.synchronize()
    for step in range(2):
        t = [time.perf_counter()]
        r, d1, mm = eng.knn_robs(dqx, dqy, 10)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        a = eng.alpha(r, datagen.ALPHA_LEVELS, P.GLOBAL, 0, 0, mm)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        zz = eng.interpolate(dqx, dqy, a, d1)
        torch.cuda.synchronize(); t.append(time.perf_counter())
        d = [1e3 * (b - a_) for a_, b in zip(t, t[1:])]
        print(json.dumps({"rep": rep, "step": step, "knn_ms": d[0], "alpha_ms": d[1], "interp_ms": d[2]}), flush=True)
    eng.close()
