"""Query-sharded multi-GPU AIDW.

The paper is single-GPU.  On an 8xB200 node the path shards
naturally: every query's result depends only on the (replicated) data points and,
in GLOBAL mode, on the job-wide R_min / R_max.  So:

* rank r owns the contiguous query block [r*nq/P, (r+1)*nq/P) (:func:`shard`);
* data points are replicated (each rank regenerates them from the seed, or
  receives one broadcast);
* the ONLY exchange is one allreduce(MAX) of the 2-vector {-min r_obs, max r_obs}
  between S2 and S4 (8 B fp32 / 16 B fp64 over NVLink via NCCL) -- min is carried
  negated so a single MAX collective reduces both; division by r_exp is
  monotone, so the bounds on R are exact;
* FIXED bounds need no collective at all.

Per-query arithmetic and order never depend on the shard, so outputs are
bit-identical for any number of GPUs (tests/test_partition.py, tests/test_gpu.py).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

GLOBAL, FIXED = 0, 1


def shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous block [start, end) of n items for `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (rank * n) // world, ((rank + 1) * n) // world


def allreduce_bounds(minmax: torch.Tensor, group=None) -> torch.Tensor:
    """In-place allreduce(MAX) of {-min r_obs, max r_obs} (the north star's
    'one NCCL allreduce(min/max) of R')."""
    dist.all_reduce(minmax, op=dist.ReduceOp.MAX, group=group)
    return minmax


def run_sharded(engine, qx, qy, k, levels, rbounds=GLOBAL, r_min=0.0, r_max=2.0, muform=0, group=None):
    """Run S1..S5 on this rank's queries ``qx, qy`` with any engine exposing
    ``knn_robs(qx, qy, k) -> (r_obs, d1sq, minmax)``, ``alpha(...)`` and
    ``interpolate(...)`` (the CUDA :class:`~paper_1511_02186_b200.AIDW`; tests
    inject a CPU engine to exercise this logic with gloo)."""
    r_obs, d1sq, mm = engine.knn_robs(qx, qy, k)
    if rbounds == GLOBAL and group is not None and dist.is_initialized():
        allreduce_bounds(mm, group)
    a = engine.alpha(r_obs, levels, rbounds, r_min, r_max, mm, muform)
    return engine.interpolate(qx, qy, a, d1sq)


def gather(z_local: torch.Tensor, nq: int, group=None) -> torch.Tensor:
    """Optional all-gather of the per-rank Z blocks into the full [nq] result."""
    world = dist.get_world_size(group)
    sizes = [e - s for s, e in (shard(nq, r, world) for r in range(world))]
    m = max(sizes)
    buf = torch.zeros(m, dtype=z_local.dtype, device=z_local.device)  # equal-size blocks
    buf[: z_local.numel()] = z_local
    parts = [torch.empty(m, dtype=z_local.dtype, device=z_local.device) for _ in range(world)]
    dist.all_gather(parts, buf, group=group)
    return torch.cat([p[:n] for p, n in zip(parts, sizes)])
