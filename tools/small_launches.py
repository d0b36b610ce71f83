"""Run the whole GLOBAL path once per small config (C1, C2 f32/f64, C3) after a warm-up,
for an ncu launch list (`--metrics gpu__time_duration.sum --profile-from-start off`): which kernels the small
configs spend their time in.  usage: ncu ... python tools/small_launches.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import datagen
import paper_1511_02186_b200 as P

for name, dt in (("C1", torch.float64), ("C2", torch.float32), ("C2", torch.float64), ("C3", torch.float32)):
    x, y, z = datagen.make_data(name)
    qx, qy = datagen.make_queries(name)
    eng = P.AIDW(x, y, z, dtype=dt)
    tqx = torch.as_tensor(qx, dtype=dt, device="cuda")
    tqy = torch.as_tensor(qy, dtype=dt, device="cuda")
    k = datagen.CONFIGS[name]["k"]
    for _ in range(2):
        eng.run(tqx, tqy, k=k)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()  # ncu --profile-from-start off: only this run is listed
    eng.run(tqx, tqy, k=k)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(name, dt, flush=True)
    eng.close()
