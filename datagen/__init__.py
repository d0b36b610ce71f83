"""Seeded synthetic inputs for the AIDW hot path (shared by tests, bench and smoke).

This module holds NO arithmetic of the method (no distances, no kNN, no weights):
it only draws point sets and a value field.  Both the CUDA path and the CPU oracle
receive the arrays it returns.

Recipe (SURVEY.md §8(d) "Synthetic inputs"):

* Counter-based generator: ``u64(seed, stream, i) = mix(mix(seed*G + stream) + i*G)``
  with ``mix`` the splitmix64 finaliser and ``G = 0x9E3779B97F4A7C15``.  Any element
  can be regenerated independently, so every rank of a multi-GPU run can build the
  same data without communication.
* Coordinates live on the dyadic grid ``u * 2**-24`` (``u`` a 24-bit integer), so
  they are exactly representable in fp32 and fp64 and coordinate differences are
  exact in both precisions (reading R16).
* Streams: 0 data-x, 1 data-y, 2 z-noise, 3 query-x, 4 query-y, 5-8 clustered
  layout draws.  The paper only says points are "randomly created within a
  square" (§4); the unit square is used.
* Value field ``z = 1 + 0.25 sin(2 pi x) cos(2 pi y) + 0.05 u`` in fp64, rounded to
  fp32 so both precisions see identical values; z in [0.75, 1.30) keeps relative
  error well defined.  The paper gives no value model.
"""
from __future__ import annotations

import numpy as np

GOLDEN = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
GRID_BITS = 24
GRID = float(2 ** GRID_BITS)

# stream ids
S_DX, S_DY, S_DZ, S_QX, S_QY, S_CL_SEL, S_CL_IDX, S_CL_GAUSS, S_CL_PARAM = range(9)

K_SIZE = 1024  # "K = 1024"; "1000K = 1024000"

CONFIGS = {
    # name: (nd, nq, k, dtypes, data distribution, query distribution)
    "C1": dict(nd=1 * K_SIZE, nq=1 * K_SIZE, k=10, dtypes=("f64",), data="uniform", queries="uniform"),
    "C2": dict(nd=10 * K_SIZE, nq=10 * K_SIZE, k=10, dtypes=("f32", "f64"), data="uniform", queries="uniform"),
    "C3": dict(nd=100 * K_SIZE, nq=100 * K_SIZE, k=15, dtypes=("f32",), data="clustered", queries="uniform"),
    "C4": dict(nd=1000 * K_SIZE, nq=1000 * K_SIZE, k=10, dtypes=("f32",), data="uniform", queries="uniform"),
    "C5": dict(nd=1000 * K_SIZE, nq=4096 * 2000, k=10, dtypes=("f32",), data="uniform", queries="grid"),
}
ALPHA_LEVELS = (1.0, 1.5, 2.0, 2.5, 3.0)  # DESIGN.md reading R13 (paper gives none)


def _mix(z: np.ndarray) -> np.ndarray:
    z = z.astype(np.uint64, copy=True)
    with np.errstate(over="ignore"):
        z ^= z >> np.uint64(30)
        z *= _M1
        z ^= z >> np.uint64(27)
        z *= _M2
        z ^= z >> np.uint64(31)
    return z


def u64(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Counter-based 64-bit draws for indices ``idx`` of (seed, stream)."""
    with np.errstate(over="ignore"):
        key = _mix(np.asarray([np.uint64(seed) * GOLDEN + np.uint64(stream)], dtype=np.uint64))[0]
        return _mix(key + np.asarray(idx, dtype=np.uint64) * GOLDEN)


def grid24(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n dyadic coordinates u*2^-24 in [0,1), u the top 24 bits of u64."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    u = (u64(seed, stream, idx) >> np.uint64(64 - GRID_BITS)).astype(np.float64)
    return u / GRID


def unit(seed: int, stream: int, n: int, offset: int = 0) -> np.ndarray:
    """n doubles in [0,1) with 53 random bits."""
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    return (u64(seed, stream, idx) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def snap24(v: np.ndarray) -> np.ndarray:
    """Round to the 2^-24 grid and wrap into [0,1)."""
    u = np.rint(np.asarray(v, dtype=np.float64) * GRID).astype(np.int64) % (1 << GRID_BITS)
    return u.astype(np.float64) / GRID


def value_field(x: np.ndarray, y: np.ndarray, seed: int) -> np.ndarray:
    """z = 1 + 0.25 sin(2 pi x) cos(2 pi y) + 0.05 u, rounded to fp32 (returned as float64)."""
    u = unit(seed, S_DZ, x.shape[0])
    z = 1.0 + 0.25 * np.sin(2.0 * np.pi * x) * np.cos(2.0 * np.pi * y) + 0.05 * u
    return z.astype(np.float32).astype(np.float64)


def uniform_points(seed: int, n: int, sx: int, sy: int, offset: int = 0):
    return grid24(seed, sx, n, offset), grid24(seed, sy, n, offset)


def clustered_points(seed: int, n: int, n_blobs: int = 32, frac_blob: float = 0.9):
    """90% in 32 isotropic Gaussian blobs (centres U[0.05,0.95]^2, sigma U[0.005,0.03]),
    10% uniform background, wrapped mod 1 and snapped to the 2^-24 grid."""
    par = unit(seed, S_CL_PARAM, 3 * n_blobs)
    cx = 0.05 + 0.9 * par[0:n_blobs]
    cy = 0.05 + 0.9 * par[n_blobs:2 * n_blobs]
    sig = 0.005 + 0.025 * par[2 * n_blobs:3 * n_blobs]
    sel = unit(seed, S_CL_SEL, n) < frac_blob
    blob = (u64(seed, S_CL_IDX, np.arange(n, dtype=np.uint64)) % np.uint64(n_blobs)).astype(np.int64)
    g = unit(seed, S_CL_GAUSS, 2 * n)
    u1 = np.maximum(g[0::2], 2.0 ** -53)
    u2 = g[1::2]
    r = np.sqrt(-2.0 * np.log(u1))
    gx = r * np.cos(2.0 * np.pi * u2)
    gy = r * np.sin(2.0 * np.pi * u2)
    bx, by = grid24(seed, S_DX, n), grid24(seed, S_DY, n)
    x = np.where(sel, cx[blob] + sig[blob] * gx, bx)
    y = np.where(sel, cy[blob] + sig[blob] * gy, by)
    return snap24(x), snap24(y)


def grid_queries(nx: int = 4096, ny: int = 2000):
    """Cell centres ((i+1/2)/nx, (j+1/2)/ny), snapped to the 2^-24 grid (C5), row-major in j."""
    xs = snap24((np.arange(nx, dtype=np.float64) + 0.5) / nx)
    ys = snap24((np.arange(ny, dtype=np.float64) + 0.5) / ny)
    qx = np.tile(xs, ny)
    qy = np.repeat(ys, nx)
    return qx, qy


def make_data(name_or_cfg, seed: int | None = None, nd: int | None = None):
    """Data points (x, y, z) as float64 arrays holding fp32-exact values."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    if seed is None:
        seed = 1000 + int(name_or_cfg[1:]) if isinstance(name_or_cfg, str) else 1000
    n = cfg["nd"] if nd is None else nd
    if cfg["data"] == "uniform":
        x, y = uniform_points(seed, n, S_DX, S_DY)
    elif cfg["data"] == "clustered":
        x, y = clustered_points(seed, n)
    else:
        raise ValueError(cfg["data"])
    return x, y, value_field(x, y, seed)


def make_queries(name_or_cfg, seed: int | None = None, nq: int | None = None, offset: int = 0):
    """Query points (x, y) as float64 arrays of fp32-exact values.  ``offset`` selects a
    contiguous slice [offset, offset+nq) of the uniform stream (query sharding)."""
    cfg = CONFIGS[name_or_cfg] if isinstance(name_or_cfg, str) else name_or_cfg
    if seed is None:
        seed = 1000 + int(name_or_cfg[1:]) if isinstance(name_or_cfg, str) else 1000
    n = cfg["nq"] if nq is None else nq
    if cfg["queries"] == "uniform":
        return uniform_points(seed, n, S_QX, S_QY, offset)
    if cfg["queries"] == "grid":
        qx, qy = grid_queries()
        return qx[offset:offset + n], qy[offset:offset + n]
    raise ValueError(cfg["queries"])


def random_cloud(seed: int, nd: int, nq: int):
    """Small uniform cloud + queries for tests (fp32-exact grid values)."""
    x, y = uniform_points(seed, nd, S_DX, S_DY)
    qx, qy = uniform_points(seed, nq, S_QX, S_QY)
    return x, y, value_field(x, y, seed), qx, qy
