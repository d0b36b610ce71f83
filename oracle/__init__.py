"""CPU oracle for the AIDW hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1511_02186_b200``) never imports it and shares no code with it.

``oracle/aidw_oracle.c`` holds the arithmetic (plain C, fp64, OpenMP over queries);
this module only marshals numpy arrays through ctypes and composes the steps in
the paper's order (§2.2 Steps 1-3 then Eq. 1).

Parity status per function: every function below is
pinned by tests/test_oracle.py against closed forms, brute force, paper/spec
worked values or invariants; none is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "aidw_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

GLOBAL, FIXED = "global", "fixed"
NORMALIZED, PRINTED = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle (gcc -O2 -fopenmp -ffp-contract=off, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call([
            "gcc", "-O2", "-fopenmp", "-ffp-contract=off", "-fno-fast-math", "-std=c11",
            "-fPIC", "-shared", "-Wall", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        D = ctypes.c_double
        L.oracle_knn_insert.argtypes = [P, ctypes.c_int, D]
        L.oracle_knn_f64.argtypes = [P, P, I64, P, P, I64, ctypes.c_int, P, P, P]
        L.oracle_knn_f64.restype = ctypes.c_int
        L.oracle_knn_f32.argtypes = [P, P, I64, P, P, I64, ctypes.c_int, P, P, P]
        L.oracle_knn_f32.restype = ctypes.c_int
        L.oracle_bbox_area.argtypes = [P, P, I64]
        L.oracle_bbox_area.restype = D
        L.oracle_r_exp.argtypes = [I64, D]
        L.oracle_r_exp.restype = D
        L.oracle_mu.argtypes = [D, D, D, ctypes.c_int]
        L.oracle_mu.restype = D
        L.oracle_alpha_of_mu.argtypes = [D, P]
        L.oracle_alpha_of_mu.restype = D
        L.oracle_alpha.argtypes = [P, I64, D, P, D, D, ctypes.c_int, P, P, P]
        L.oracle_idw.argtypes = [P, P, P, I64, P, P, P, I64, P]
        L.oracle_num_threads.restype = ctypes.c_int
        L.oracle_set_num_threads.argtypes = [ctypes.c_int]
        _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None else None


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def num_threads() -> int:
    return lib().oracle_num_threads()


def set_num_threads(n: int) -> None:
    lib().oracle_set_num_threads(int(n))


def knn_insert(buf, dist):
    """§3.1.2 Step 3 on one ascending buffer.  Returns a new array."""
    b = _f64(buf).copy()
    lib().oracle_knn_insert(_p(b), b.shape[0], float(dist))
    return b


def _knn(fn, cast, npdt, x, y, qx, qy, k, want_dists, want_d1sq):
    x, y, qx, qy = cast(x), cast(y), cast(qx), cast(qy)
    nq = qx.shape[0]
    robs = np.empty(nq, npdt)
    d = np.empty((nq, k), npdt) if want_dists else None
    d1 = np.empty(nq, npdt) if want_d1sq else None
    rc = fn(_p(x), _p(y), x.shape[0], _p(qx), _p(qy), nq, int(k), _p(d), _p(robs), _p(d1))
    if rc != 0:
        raise ValueError("oracle kNN: k out of range or nd < k")
    out = (robs,) + ((d,) if want_dists else ()) + ((d1,) if want_d1sq else ())
    return out if len(out) > 1 else robs


def knn_f64(x, y, qx, qy, k, want_dists=False, want_d1sq=False):
    """k nearest distances (ascending) and r_obs per query, fp64 (§3.1.2, Eq. 3);
    optionally the nearest squared distance min_i s_i (R16/R20).
    Returns robs, or (robs[, dists][, d1sq])."""
    return _knn(lib().oracle_knn_f64, _f64, np.float64, x, y, qx, qy, k, want_dists, want_d1sq)


def knn_f32(x, y, qx, qy, k, want_dists=False, want_d1sq=False):
    """The fp32 instantiation (REAL = float; R16)."""
    return _knn(lib().oracle_knn_f32, _f32, np.float32, x, y, qx, qy, k, want_dists, want_d1sq)


def bbox_area(x, y) -> float:
    x, y = _f64(x), _f64(y)
    return lib().oracle_bbox_area(_p(x), _p(y), x.shape[0])


def r_exp(nd: int, area: float) -> float:
    """Eq. 2."""
    return lib().oracle_r_exp(int(nd), float(area))


def mu(R, rmin, rmax, form=NORMALIZED) -> float:
    """Eq. 5."""
    return lib().oracle_mu(float(R), float(rmin), float(rmax), int(form))


def alpha_of_mu(m, levels) -> float:
    """Eq. 6."""
    lv = _f64(levels)
    return lib().oracle_alpha_of_mu(float(m), _p(lv))


def alpha(robs, r_exp_, levels, rmin, rmax, form=NORMALIZED, trace=False):
    """Eq. 4 -> Eq. 5 -> Eq. 6 per query."""
    robs = _f64(robs)
    lv = _f64(levels)
    nq = robs.shape[0]
    a = np.empty(nq, np.float64)
    R = np.empty(nq, np.float64) if trace else None
    m = np.empty(nq, np.float64) if trace else None
    lib().oracle_alpha(_p(robs), nq, float(r_exp_), _p(lv), float(rmin), float(rmax), int(form),
                       _p(a), _p(R), _p(m))
    return (a, R, m) if trace else a


def idw(x, y, z, qx, qy, alpha_q):
    """Eq. 1 with per-query alpha over all data points."""
    x, y, z, qx, qy = _f64(x), _f64(y), _f64(z), _f64(qx), _f64(qy)
    nq = qx.shape[0]
    a = np.broadcast_to(np.asarray(alpha_q, np.float64), (nq,)).copy()
    out = np.empty(nq, np.float64)
    lib().oracle_idw(_p(x), _p(y), _p(z), x.shape[0], _p(qx), _p(qy), _p(a), nq, _p(out))
    return out


def r_bounds(robs_all, r_exp_, mode, r_min=0.0, r_max=2.0):
    """R_min / R_max: FIXED user values (paper default 0, 2) or
    GLOBAL min/max of R = r_obs / r_exp over all queries (R7)."""
    if mode == FIXED:
        return float(r_min), float(r_max)
    robs_all = _f64(robs_all)
    return float(robs_all.min()) / r_exp_, float(robs_all.max()) / r_exp_


def aidw(x, y, z, qx, qy, k, levels, mode=GLOBAL, r_min=0.0, r_max=2.0, form=NORMALIZED,
         area=None, trace=False):
    """Full AIDW in fp64 in the paper's order: kNN -> r_obs (Eq. 3), r_exp (Eq. 2),
    R (Eq. 4), mu (Eq. 5), alpha (Eq. 6), then Eq. 1."""
    nd = len(x)
    A = bbox_area(x, y) if area is None else float(area)
    re = r_exp(nd, A)
    robs = knn_f64(x, y, qx, qy, k)
    rmin, rmax = r_bounds(robs, re, mode, r_min, r_max)
    a, R, m = alpha(robs, re, levels, rmin, rmax, form, trace=True)
    Z = idw(x, y, z, qx, qy, a)
    if trace:
        return Z, dict(r_exp=re, area=A, r_obs=robs, R=R, mu=m, alpha=a, r_min=rmin, r_max=rmax)
    return Z
