"""Worker process of tests/test_gpu.py::test_bounds_exchange_two_processes (spawned, one
per rank; the ranks share the single GPU and map each other's exchange buffers)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import datagen  # noqa: E402


STEPS = 4


def step_queries(step, qx, qy):
    """Step 0 = the cloud's queries; later steps shrink them towards a corner so each
    step's GLOBAL bounds differ."""
    f = 1.0 - 0.2 * step
    return qx * f, qy * f


def run(rank, world, port, nq_split, out_dir):
    import paper_1511_02186_b200 as P
    from paper_1511_02186_b200.partition import connect_exchange, run_sharded
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    x, y, z, qx, qy = datagen.random_cloud(4242, 60000, 50000)
    eng = P.AIDW(x, y, z)
    connect_exchange(eng)
    s, e = nq_split[rank], nq_split[rank + 1]
    outs = []
    # several steps with DIFFERENT query batches (so stale bounds would show), enqueued
    # without a host sync in between: a rank may run a step ahead of its peer
    for step in range(STEPS):
        sx, sy = step_queries(step, qx, qy)
        outs.append(run_sharded(eng, sx[s:e], sy[s:e], 10, datagen.ALPHA_LEVELS, P.GLOBAL))
    eng.check()
    np.save(os.path.join(out_dir, f"z{rank}.npy"), np.stack([o.cpu().numpy() for o in outs]))
    dist.barrier()
    eng.close()
    dist.destroy_process_group()
