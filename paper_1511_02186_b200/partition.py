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
    inject a CPU engine to exercise this logic with gloo).  An engine with a
    connected device-side bounds exchange (:func:`connect_exchange`) needs no
    host collective: its alpha kernel waits for the peers' pushed bounds."""
    r_obs, d1sq, mm = engine.knn_robs(qx, qy, k)
    if rbounds == GLOBAL and getattr(engine, "exchanged", False):
        a = engine.alpha(r_obs, levels, rbounds, r_min, r_max, None, muform)
        return engine.interpolate(qx, qy, a, d1sq)
    if rbounds == GLOBAL and group is not None and dist.is_initialized():
        allreduce_bounds(mm, group)
    a = engine.alpha(r_obs, levels, rbounds, r_min, r_max, mm, muform)
    return engine.interpolate(qx, qy, a, d1sq)


def connect_exchange(engine, group=None):
    """Set up the device-side GLOBAL-bounds exchange (aidw_exchange_*):
    every rank allocates its buffer, the 64-byte CUDA IPC handles are all-gathered
    once over ``group`` (any backend), and each rank maps its peers' buffers.  After
    this, every kNN launch pushes its bounds to all ranks from its last CTA and the
    alpha kernel reads them on the device -- no collective per step."""
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    mine = engine.exchange_setup(rank, world)
    handles = [None] * world
    if world > 1:
        dist.all_gather_object(handles, mine, group=group)
    else:
        handles = [mine]
    engine.exchange_connect(handles)
    return engine


# ---------------------------------------------------------------------------------
# N4: data-sharded mode.  The DATA points are split across ranks (shard boundaries at
# multiples of `align` points so the fp32 tile sums are the single-device ones); every
# rank evaluates ALL queries against its shard.  Exchanges per run: one all-gather of the
# k smallest squared distances (k * nq values per rank) and one all-gather of the Eq. 1
# partial sums (4 fp64 per query per rank); both are reduced in rank order on the device
# (aidw_knn_merge, aidw_finalize), so results are deterministic for a given world size.
# The merged kNN lists, r_obs, the GLOBAL R bounds and alpha are bit-identical to one
# device; Z differs from it only in the fp64 order of the cross-shard sum.

def data_shard(nd: int, rank: int, world: int, align: int = 1024) -> tuple[int, int]:
    """[start, end) of the data points of `rank`; interior boundaries are multiples of align."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    blocks = (nd + align - 1) // align
    s, e = shard(blocks, rank, world)
    return min(nd, s * align), min(nd, e * align)


def global_extent(engine, group=None):
    """(nd_total, bbox) of the whole data set from every rank's shard: one allreduce(MAX)
    of {-min x, max x, -min y, max y} (negation carries the minima through the MAX, as
    for the r_obs bounds) and one allreduce(SUM) of the shard sizes.  Eq. 2's area and
    r_exp are then computed behind the C ABI (``engine.set_extent_bbox``)."""
    x0, x1, y0, y1 = engine.bbox()
    dev = getattr(engine, "device", torch.device("cpu"))
    t = torch.tensor([-x0, x1, -y0, y1], dtype=torch.float64, device=dev)
    n = torch.tensor([float(engine.nd)], dtype=torch.float64, device=dev)
    if group is not None and dist.is_initialized():
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
        dist.all_reduce(n, op=dist.ReduceOp.SUM, group=group)
    t = t.cpu().tolist()
    return int(n.item()), [-t[0], t[1], -t[2], t[3]]


def check_data_shards(nd_total: int, world: int, k: int, align: int = 1024) -> None:
    """Raise (identically on every rank, before any collective) if some rank's data shard
    would hold fewer than max(k, 1) points: a shard needs k real points for its partial
    kNN list and at least one for its handle.  Use fewer ranks for such small data sets."""
    for r in range(world):
        s, e = data_shard(nd_total, r, world, align)
        if e - s < max(k, 1):
            raise ValueError(f"data-sharded mode: rank {r} of {world} gets {e - s} of {nd_total} data points "
                             f"(< k = {k}; shards are whole blocks of {align}); use at most "
                             f"{max(1, nd_total // max(align, k))} ranks")


def _all_gather_cat(x: torch.Tensor, group=None) -> torch.Tensor:
    world = dist.get_world_size(group) if group is not None and dist.is_initialized() else 1
    if world == 1:
        return x
    parts = [torch.empty_like(x) for _ in range(world)]
    dist.all_gather(parts, x.contiguous(), group=group)
    return torch.cat(parts)


def run_data_sharded(engine, qx, qy, k, levels, rbounds=GLOBAL, r_min=0.0, r_max=2.0, muform=0, group=None):
    """Full AIDW with the data split across ranks; every rank returns Z for ALL queries.
    `engine` holds this rank's data shard with the global extent set
    (``engine.set_extent_bbox(*global_extent(engine, group))``)."""
    world = dist.get_world_size(group) if group is not None and dist.is_initialized() else 1
    check_data_shards(getattr(engine, "nd_total", engine.nd), world, k)
    nq = len(qx)
    s_local = engine.knn_partial(qx, qy, k)
    lists = _all_gather_cat(s_local, group)
    r_obs, d1sq, mm = engine.knn_merge(lists, world, nq, k)  # mm already covers all queries
    a = engine.alpha(r_obs, levels, rbounds, r_min, r_max, mm, muform)
    part = engine.interpolate_partial(qx, qy, a, d1sq)
    parts = _all_gather_cat(part, group)
    return engine.finalize(parts, world, nq)


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
