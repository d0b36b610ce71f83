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


# ------------------------------------------------------------------ N4 on gloo
class NumpyShardEngine:
    """CPU stand-in for the data-sharded engine interface (test infrastructure): plain
    numpy definitions of the partial kNN lists, merge, partial Eq. 1 sums, finalize."""

    def __init__(self, x, y, z):
        import oracle
        self.o = oracle
        self.x, self.y, self.z = x, y, z
        self.nd = len(x)
        self.re = None

    def bbox(self):
        return [self.x.min(), self.x.max(), self.y.min(), self.y.max()]

    def set_extent_bbox(self, nd_total, bbox):
        self.re = self.o.r_exp(nd_total, (bbox[1] - bbox[0]) * (bbox[3] - bbox[2]))
        self.nd_total = nd_total

    def knn_partial(self, qx, qy, k):
        s = (np.asarray(qx)[:, None] - self.x[None]) ** 2 + (np.asarray(qy)[:, None] - self.y[None]) ** 2
        return torch.as_tensor(np.sort(s, axis=1)[:, :k].reshape(-1))

    def knn_merge(self, lists, P, nq, k):
        L = lists.numpy().reshape(P, nq, k).transpose(1, 0, 2).reshape(nq, P * k)
        s = np.sort(L, axis=1)[:, :k]
        d = np.sqrt(s)
        robs = np.zeros(nq)
        for i in range(k):
            robs = robs + d[:, i]
        robs = robs / k
        return torch.as_tensor(robs), torch.as_tensor(s[:, 0]), torch.tensor([-robs.min(), robs.max()])

    def alpha(self, r_obs, levels, rbounds, r_min, r_max, mm, muform):
        if rbounds == partition.GLOBAL:
            r_min, r_max = -float(mm[0]) / self.re, float(mm[1]) / self.re
        return torch.as_tensor(self.o.alpha(r_obs.numpy(), self.re, levels, r_min, r_max, muform))

    def interpolate_partial(self, qx, qy, a, d1sq):
        out = np.zeros((len(qx), 4))
        for q in range(len(qx)):
            d = np.sqrt((qx[q] - self.x) ** 2 + (qy[q] - self.y) ** 2)
            c = d == 0
            w = np.where(c, 0.0, np.where(c, 1.0, d) ** -float(a[q]))
            out[q] = [w.sum(), (w * self.z).sum(), self.z[c].sum(), c.sum()]
        return torch.as_tensor(out.reshape(-1))

    def finalize(self, parts, P, nq):
        p = parts.numpy().reshape(P, nq, 4)
        tot = np.zeros((nq, 4))
        for r in range(P):
            tot = tot + p[r]
        return torch.as_tensor(np.where(tot[:, 3] > 0, tot[:, 2] / np.maximum(tot[:, 3], 1), tot[:, 1] / tot[:, 0]))


def _worker_data(rank, world, port, out_q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        x, y, z, qx, qy = datagen.random_cloud(98, 3000, 201)
        s, e = partition.data_shard(len(x), rank, world)
        eng = NumpyShardEngine(x[s:e], y[s:e], z[s:e])
        eng.set_extent_bbox(*partition.global_extent(eng, dist.group.WORLD))
        zr = partition.run_data_sharded(eng, qx, qy, 10, LV, partition.GLOBAL, group=dist.group.WORLD)
        out_q.put((rank, zr.numpy()))
    finally:
        dist.destroy_process_group()


def test_gloo_data_sharded_two_ranks(orc):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    mp.start_processes(_worker_data, args=(2, _free_port(), q), nprocs=2, join=True, start_method="spawn")
    res = dict(q.get() for _ in range(2))
    x, y, z, qx, qy = datagen.random_cloud(98, 3000, 201)
    z1 = orc.aidw(x, y, z, qx, qy, 10, LV, mode="global")
    assert np.array_equal(res[0], res[1])  # every rank returns the full, identical result
    assert np.max(np.abs(res[0] - z1) / np.abs(z1)) < 1e-12


def test_data_shard_bounds():
    for nd in (1, 1000, 1024, 5000, 1024000):
        for world in (1, 2, 3, 8):
            b = [partition.data_shard(nd, r, world) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nd
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            assert all(s % 1024 == 0 for s, _ in b)


def test_check_data_shards():
    """Small data sets on many ranks: a clear error before any collective instead of an
    empty shard (aidw_create needs nd >= 1) or a shard with fewer than k points."""
    partition.check_data_shards(1024000, 8, 10)
    partition.check_data_shards(2048, 2, 10)
    for nd, world in ((5000, 8), (1030, 2), (1, 2)):
        with pytest.raises(ValueError, match="data-sharded mode"):
            partition.check_data_shards(nd, world, 10)
