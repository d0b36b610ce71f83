"""Multi-rank query sharding on CPU: world_size-2 `gloo` process groups drive the
partitioner (paper_1511_02186_b200/partition.py) with a CPU engine built from the
oracle (test infrastructure), so the shard/allreduce/gather logic is checked
without GPUs.  The GPU side of the same logic is tests/test_gpu.py::test_sharding_bit_identical."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
from paper_1511_02186_b200 import partition

LV = datagen.ALPHA_LEVELS


def test_shard_bounds():
    for n in (0, 1, 7, 1000, 1024000, 8192000):
        for world in (1, 2, 3, 4, 8):
            b = [partition.shard(n, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            sizes = [e - s for s, e in b]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        partition.shard(10, 2, 2)


class OracleEngine:
    """CPU stand-in with the engine interface of paper_1511_02186_b200.AIDW."""

    def __init__(self, x, y, z):
        import oracle
        self.o = oracle
        self.x, self.y, self.z = x, y, z
        self.re = oracle.r_exp(len(x), oracle.bbox_area(x, y))
        self.allreduce_calls = 0

    def knn_robs(self, qx, qy, k):
        robs, d = self.o.knn_f64(self.x, self.y, qx, qy, k, want_dists=True)
        mm = torch.tensor([-robs.min() if len(robs) else -np.inf, robs.max() if len(robs) else -np.inf],
                          dtype=torch.float64)
        return torch.as_tensor(robs), torch.as_tensor(d[:, 0] ** 2), mm

    def alpha(self, r_obs, levels, rbounds, r_min, r_max, mm, muform):
        if rbounds == partition.GLOBAL:
            r_min, r_max = -float(mm[0]) / self.re, float(mm[1]) / self.re
        return torch.as_tensor(self.o.alpha(r_obs.numpy(), self.re, levels, r_min, r_max, muform))

    def interpolate(self, qx, qy, a, d1sq):
        return torch.as_tensor(self.o.idw(self.x, self.y, self.z, qx, qy, a.numpy()))


def _worker(rank, world, port, mode, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y, z, qx, qy = datagen.random_cloud(99, 3000, 501)
        eng = OracleEngine(x, y, z)
        s, e = partition.shard(len(qx), rank, world)
        rb = partition.GLOBAL if mode == "global" else partition.FIXED
        zl = partition.run_sharded(eng, qx[s:e], qy[s:e], 10, LV, rb, 0.0, 2.0, 0, dist.group.WORLD)
        zfull = partition.gather(zl, len(qx))
        if rank == 0:
            out_q.put(zfull.numpy())
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("mode", ["global", "fixed"])
def test_gloo_two_ranks_equal_single(orc, mode):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker, args=(2, _free_port(), mode, q), nprocs=2, join=True, start_method="spawn")
    z2 = q.get()
    x, y, z, qx, qy = datagen.random_cloud(99, 3000, 501)
    z1 = orc.aidw(x, y, z, qx, qy, 10, LV, mode=mode)
    assert np.array_equal(z2, z1)  # bit-identical: per-query math, exact min/max


def test_allreduce_negated_min_trick():
    """MAX over {-min, max} pairs gives {-global min, global max}."""
    parts = [torch.tensor([-3.0, 5.0]), torch.tensor([-1.5, 9.0]), torch.tensor([-np.inf, -np.inf])]
    m = torch.stack(parts).max(0).values
    assert m.tolist() == [-1.5, 9.0]
