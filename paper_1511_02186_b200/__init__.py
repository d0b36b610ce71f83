"""B200-native AIDW hot path (arXiv 1511.02186) -- thin Python binding of libaidw.so.

Every step of the path runs in the sm_100a kernels behind the C ABI declared in
``include/aidw.h``; this module only marshals torch tensors (device memory) and
CUDA streams through ctypes.  There is NO CPU fallback: if the extension is
missing, :func:`lib` raises.

Low-level functions carry the ABI names (``aidw_create``, ``aidw_knn_robs``,
``aidw_alpha``, ``aidw_interpolate``, ``aidw_destroy``, ``aidw_run_host``,
``aidw_check``).  :class:`AIDW` wraps a handle; :mod:`.partition` shards queries
across ranks.
"""
from __future__ import annotations

import ctypes
import os

import torch

from ._build import LIB as _LIB_PATH
from ._build import build as build_extension

__all__ = [
    "AIDW", "AidwError", "lib", "build_extension",
    "aidw_create", "aidw_knn_robs", "aidw_alpha", "aidw_interpolate", "aidw_destroy",
    "aidw_run_host", "aidw_check", "aidw_run_fixed", "aidw_idw", "GLOBAL", "FIXED", "NORMALIZED", "PRINTED",
]

F32, F64 = 0, 1
SOA, AOS, AOAS = 0, 1, 2
GLOBAL, FIXED = 0, 1
NORMALIZED, PRINTED = 0, 1
KMAX = 32
LEVELS_DEFAULT = (1.0, 1.5, 2.0, 2.5, 3.0)

_STATUS = {
    0: "AIDW_OK", 1: "AIDW_E_INVALID_ARG", 2: "AIDW_E_INSUFFICIENT_DATA", 3: "AIDW_E_DEGENERATE_EXTENT",
    4: "AIDW_E_INVALID_AREA", 5: "AIDW_E_INVALID_BOUNDS", 6: "AIDW_E_NONFINITE_INPUT",
    7: "AIDW_E_UNSUPPORTED", 8: "AIDW_E_CUDA", 9: "AIDW_E_NOMEM",
}

# Every symbol include/aidw.h declares (checked by tests/test_abi.py).
EXPORTS = (
    "aidw_abi_version", "aidw_status_string", "aidw_last_error", "aidw_create", "aidw_nd",
    "aidw_area", "aidw_r_exp", "aidw_dtype_of", "aidw_knn_robs", "aidw_alpha", "aidw_interpolate",
    "aidw_run_host", "aidw_check", "aidw_launch_count", "aidw_destroy", "aidw_run_fixed", "aidw_idw",
    "aidw_paper_baseline", "aidw_set_extent", "aidw_set_extent_bbox", "aidw_bbox", "aidw_knn_partial", "aidw_knn_merge",
    "aidw_interpolate_partial", "aidw_finalize", "aidw_exchange_setup", "aidw_exchange_connect",
    "aidw_exchange_close",
)


class AidwError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        self.name = _STATUS.get(status, f"status {status}")
        super().__init__(f"{self.name}: {msg}")


_lib = None


def lib():
    """Load libaidw.so.  Raises if the extension was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"libaidw.so not built ({_LIB_PATH}); run __graft_entry__.build()")
        L = ctypes.CDLL(_LIB_PATH)
        P, I64, D, I = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int
        sig = {
            "aidw_abi_version": ([], I),
            "aidw_status_string": ([I], ctypes.c_char_p),
            "aidw_last_error": ([P], ctypes.c_char_p),
            "aidw_create": ([ctypes.POINTER(P), I, I, I, P, I64, D, P], I),
            "aidw_nd": ([P], I64),
            "aidw_area": ([P], D),
            "aidw_r_exp": ([P], D),
            "aidw_dtype_of": ([P], I),
            "aidw_knn_robs": ([P, P, P, I64, I, P, P, P, P, P], I),
            "aidw_alpha": ([P, P, I64, P, I, D, D, P, I, P, P], I),
            "aidw_interpolate": ([P, P, P, I64, P, P, P, P], I),
            "aidw_run_host": ([P, P, P, I64, I, P, I, D, D, I, P, P], I),
            "aidw_check": ([P, P], I),
            "aidw_launch_count": ([P], I64),
            "aidw_run_fixed": ([P, P, P, I64, I, P, D, D, I, P, P, P, P], I),
            "aidw_idw": ([P, P, P, I64, D, P, P], I),
            "aidw_paper_baseline": ([I, I, I, P, I64, P, P, I64, I, P, D, D, D, P, P], I),
            "aidw_set_extent": ([P, I64, D], I),
            "aidw_bbox": ([P, P], I),
            "aidw_set_extent_bbox": ([P, I64, P], I),
            "aidw_knn_partial": ([P, P, P, I64, I, P, P], I),
            "aidw_knn_merge": ([P, P, I, I64, I, P, P, P, P], I),
            "aidw_interpolate_partial": ([P, P, P, I64, P, P, P, P], I),
            "aidw_finalize": ([P, P, I, I64, P, P], I),
            "aidw_exchange_setup": ([P, I, I, P], I),
            "aidw_exchange_connect": ([P, P], I),
            "aidw_exchange_close": ([P], I),
            "aidw_destroy": ([P], I),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = res
        _lib = L
    return _lib


def _err(h, st):
    if st != 0:
        msg = lib().aidw_last_error(h)
        raise AidwError(st, msg.decode() if msg else "")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None, device=None):
    if stream is None:
        stream = torch.cuda.current_stream(device)
    return ctypes.c_void_p(stream.cuda_stream)


class _nullctx:
    def __enter__(self):
        return self

    def __exit__(self, *a):
        return False


def _levels(levels):
    lv = (ctypes.c_double * 5)(*[float(v) for v in levels])
    if len(levels) != 5:
        raise ValueError("alpha levels must be 5 values (Eq. 6)")
    return lv


# ------------------------------------------------------------------ ABI-named calls
def aidw_create(data, nd, dtype=F32, layout=SOA, area=0.0, device=0, stream=None):
    """Create a handle from a tensor ``data`` (CUDA or host) in ``layout``."""
    h = ctypes.c_void_p()
    st = lib().aidw_create(ctypes.byref(h), int(device), int(dtype), int(layout), _ptr(data), int(nd),
                           float(area), _stream(stream, device))
    if st != 0:
        _err(None, st)
    return h


def aidw_knn_robs(h, qx, qy, k, r_obs, d1sq=None, minmax=None, dists=None, stream=None):
    _err(h, lib().aidw_knn_robs(h, _ptr(qx), _ptr(qy), qx.numel(), int(k), _ptr(r_obs), _ptr(d1sq),
                                _ptr(minmax), _ptr(dists), _stream(stream)))


def aidw_alpha(h, r_obs, levels, rbounds, r_min, r_max, minmax, muform, alpha, stream=None):
    _err(h, lib().aidw_alpha(h, _ptr(r_obs), r_obs.numel(), _levels(levels), int(rbounds), float(r_min),
                             float(r_max), _ptr(minmax), int(muform), _ptr(alpha), _stream(stream)))


def aidw_interpolate(h, qx, qy, alpha, d1sq, z, stream=None):
    _err(h, lib().aidw_interpolate(h, _ptr(qx), _ptr(qy), qx.numel(), _ptr(alpha), _ptr(d1sq), _ptr(z),
                                   _stream(stream)))


def aidw_run_host(h, qx_host, qy_host, k, levels, rbounds, r_min, r_max, muform, z_host, stream=None):
    _err(h, lib().aidw_run_host(h, _ptr(qx_host), _ptr(qy_host), qx_host.numel(), int(k), _levels(levels),
                                int(rbounds), float(r_min), float(r_max), int(muform), _ptr(z_host),
                                _stream(stream)))


def aidw_run_fixed(h, qx, qy, k, levels, r_min, r_max, muform, z, r_obs=None, alpha=None, stream=None):
    _err(h, lib().aidw_run_fixed(h, _ptr(qx), _ptr(qy), qx.numel(), int(k), _levels(levels), float(r_min),
                                 float(r_max), int(muform), _ptr(z), _ptr(r_obs), _ptr(alpha), _stream(stream)))


def aidw_idw(h, qx, qy, alpha, z, stream=None):
    _err(h, lib().aidw_idw(h, _ptr(qx), _ptr(qy), qx.numel(), float(alpha), _ptr(z), _stream(stream)))


def aidw_paper_baseline(variant, data, nd, qx, qy, k, levels, area, r_min, r_max, z, layout=SOA, stream=None):
    """N3 ablation: the paper's naive (0) / tiled (1) kernel designs on sm_100a."""
    dt = F32 if data.dtype == torch.float32 else F64
    _err(None, lib().aidw_paper_baseline(int(variant), dt, int(layout), _ptr(data), int(nd), _ptr(qx), _ptr(qy),
                                         qx.numel(), int(k), _levels(levels), float(area), float(r_min),
                                         float(r_max), _ptr(z), _stream(stream)))


def aidw_check(h, stream=None):
    _err(h, lib().aidw_check(h, _stream(stream)))


def aidw_destroy(h):
    lib().aidw_destroy(h)


# ------------------------------------------------------------------ handle wrapper
_TORCH_DT = {F32: torch.float32, F64: torch.float64}


class AIDW:
    """One handle: the data points resident on one GPU, queried many times.

    ``x, y, z``: 1-D tensors / arrays of the data point coordinates and values
    (the paper's dx, dy, dz).  ``dtype``: torch.float32 (REAL =
    float) or torch.float64.  ``area``: 0 -> bounding box (Eq. 2's A).
    """

    def __init__(self, x, y, z, dtype=torch.float32, device=None, area=0.0, _data=None):
        lib()
        if device is None:
            device = torch.cuda.current_device()
        self.device = torch.device("cuda", device) if isinstance(device, int) else torch.device(device)
        self.dt = F32 if dtype == torch.float32 else F64
        self.tdtype = _TORCH_DT[self.dt]
        if _data is not None:  # [3, nd] SoA, host (pinned: aidw_create copies it) or device
            data = _data
        else:
            data = torch.stack([torch.as_tensor(v, dtype=self.tdtype).reshape(-1) for v in (x, y, z)])
            data = data.to(self.device).contiguous()
        self.nd = data.shape[1]
        with torch.cuda.device(self.device):
            self.h = aidw_create(data, self.nd, self.dt, SOA, area, self.device.index)
        self.r_exp = lib().aidw_r_exp(self.h)
        self.area = lib().aidw_area(self.h)
        self.exchanged = False

    @classmethod
    def from_host(cls, data, device=None, area=0.0):
        """Handle from a HOST [3, nd] SoA tensor (x, y, z rows; pinned memory makes the
        copy asynchronous): aidw_create stages it to the device itself (S0)."""
        if data.is_cuda or data.dim() != 2 or data.shape[0] != 3:
            raise ValueError("from_host needs a host [3, nd] tensor")
        return cls(None, None, None, dtype=data.dtype, device=device, area=area, _data=data.contiguous())

    def close(self):
        if getattr(self, "h", None):
            aidw_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @property
    def launches(self) -> int:
        return lib().aidw_launch_count(self.h)

    def _empty(self, n):
        return torch.empty(n, dtype=self.tdtype, device=self.device)

    def _q(self, v):
        return torch.as_tensor(v, dtype=self.tdtype, device=self.device).reshape(-1).contiguous()

    # S1 + S2
    def knn_robs(self, qx, qy, k, want_dists=False, stream=None):
        qx, qy = self._q(qx), self._q(qy)
        n = qx.numel()
        r_obs, d1sq, mm = self._empty(n), self._empty(n), self._empty(2)
        dists = self._empty(n * k) if want_dists else None
        aidw_knn_robs(self.h, qx, qy, k, r_obs, d1sq, mm, dists, stream)
        if want_dists:
            return r_obs, d1sq, mm, dists.view(n, k)
        return r_obs, d1sq, mm

    # S4
    def alpha(self, r_obs, levels=LEVELS_DEFAULT, rbounds=GLOBAL, r_min=0.0, r_max=2.0, minmax=None,
              muform=NORMALIZED, stream=None):
        a = self._empty(r_obs.numel())
        aidw_alpha(self.h, r_obs, levels, rbounds, r_min, r_max, minmax, muform, a, stream)
        return a

    # S5
    def interpolate(self, qx, qy, alpha, d1sq=None, stream=None):
        qx, qy = self._q(qx), self._q(qy)
        z = self._empty(qx.numel())
        aidw_interpolate(self.h, qx, qy, alpha, d1sq, z, stream)
        return z

    def run(self, qx, qy, k=10, levels=LEVELS_DEFAULT, rbounds=GLOBAL, r_min=0.0, r_max=2.0,
            muform=NORMALIZED, group=None, stream=None, trace=False):
        """Whole path for this rank's queries; GLOBAL bounds are allreduced over
        ``group`` (torch.distributed) when given."""
        from .partition import allreduce_bounds
        nvtx = torch.cuda.nvtx
        qx, qy = self._q(qx), self._q(qy)
        nvtx.range_push("aidw.knn_robs")  # NVTX ranges for Nsight timelines (SURVEY §5 tracing)
        r_obs, d1sq, mm = self.knn_robs(qx, qy, k, stream=stream)
        nvtx.range_pop()
        if rbounds == GLOBAL and self.exchanged:  # bounds pushed/read on the device (§5)
            nvtx.range_push("aidw.alpha")
            a = self.alpha(r_obs, levels, rbounds, r_min, r_max, None, muform, stream)
            nvtx.range_pop()
            z = self.interpolate(qx, qy, a, d1sq, stream)
            if trace:
                return z, dict(r_obs=r_obs, d1sq=d1sq, minmax=mm, alpha=a)
            return z
        if rbounds == GLOBAL and group is not None:
            nvtx.range_push("aidw.allreduce_bounds")
            # the collective runs on torch's current stream: make it `stream` so it is
            # ordered after the kNN that writes mm and before the alpha that reads it
            with torch.cuda.stream(stream) if stream is not None else _nullctx():
                allreduce_bounds(mm, group)
            nvtx.range_pop()
        nvtx.range_push("aidw.alpha")
        a = self.alpha(r_obs, levels, rbounds, r_min, r_max, mm, muform, stream)
        nvtx.range_pop()
        nvtx.range_push("aidw.interpolate")
        z = self.interpolate(qx, qy, a, d1sq, stream)
        nvtx.range_pop()
        if trace:
            return z, dict(r_obs=r_obs, d1sq=d1sq, minmax=mm, alpha=a)
        return z

    def run_fixed(self, qx, qy, k=10, levels=LEVELS_DEFAULT, r_min=0.0, r_max=2.0, muform=NORMALIZED,
                  stream=None, trace=False):
        """N1: FIXED-bounds AIDW in one fused launch (aidw_run_fixed)."""
        qx, qy = self._q(qx), self._q(qy)
        n = qx.numel()
        z = self._empty(n)
        r_obs = self._empty(n) if trace else None
        a = self._empty(n) if trace else None
        aidw_run_fixed(self.h, qx, qy, k, levels, r_min, r_max, muform, z, r_obs, a, stream)
        if trace:
            return z, dict(r_obs=r_obs, alpha=a)
        return z

    def idw(self, qx, qy, alpha=2.0, stream=None):
        """N2: standard IDW with a constant power (aidw_idw)."""
        qx, qy = self._q(qx), self._q(qy)
        z = self._empty(qx.numel())
        aidw_idw(self.h, qx, qy, alpha, z, stream)
        return z

    # ---- N4: data-sharded mode (this handle holds one shard of the data points)
    def set_extent(self, nd_total, area):
        _err(self.h, lib().aidw_set_extent(self.h, int(nd_total), float(area)))
        self.r_exp = lib().aidw_r_exp(self.h)
        self.area = lib().aidw_area(self.h)
        self.nd_total = int(nd_total)

    def set_extent_bbox(self, nd_total, bbox):
        """Eq. 2 for the whole (sharded) data set from the job-wide bbox (aidw_set_extent_bbox)."""
        b = (ctypes.c_double * 4)(*[float(v) for v in bbox])
        _err(self.h, lib().aidw_set_extent_bbox(self.h, int(nd_total), b))
        self.r_exp = lib().aidw_r_exp(self.h)
        self.area = lib().aidw_area(self.h)
        self.nd_total = int(nd_total)

    def bbox(self):
        out = (ctypes.c_double * 4)()
        _err(self.h, lib().aidw_bbox(self.h, out))
        return list(out)

    def knn_partial(self, qx, qy, k, stream=None):
        qx, qy = self._q(qx), self._q(qy)
        s = self._empty(qx.numel() * k)
        _err(self.h, lib().aidw_knn_partial(self.h, _ptr(qx), _ptr(qy), qx.numel(), int(k), _ptr(s),
                                            _stream(stream)))
        return s

    def knn_merge(self, lists, P, nq, k, stream=None):
        r_obs, d1sq, mm = self._empty(nq), self._empty(nq), self._empty(2)
        _err(self.h, lib().aidw_knn_merge(self.h, _ptr(lists), int(P), int(nq), int(k), _ptr(r_obs), _ptr(d1sq),
                                          _ptr(mm), _stream(stream)))
        return r_obs, d1sq, mm

    def interpolate_partial(self, qx, qy, alpha, d1sq, stream=None):
        qx, qy = self._q(qx), self._q(qy)
        part = torch.empty(qx.numel() * 4, dtype=torch.float64, device=self.device)
        _err(self.h, lib().aidw_interpolate_partial(self.h, _ptr(qx), _ptr(qy), qx.numel(), _ptr(alpha),
                                                    _ptr(d1sq), _ptr(part), _stream(stream)))
        return part

    def finalize(self, partials, P, nq, stream=None):
        z = self._empty(nq)
        _err(self.h, lib().aidw_finalize(self.h, _ptr(partials), int(P), int(nq), _ptr(z), _stream(stream)))
        return z

    # ---- device-side GLOBAL-bounds exchange (N4 push; aidw_exchange_*)
    def exchange_setup(self, rank, world) -> bytes:
        """Allocate this rank's exchange buffer; returns its 64-byte IPC handle."""
        buf = ctypes.create_string_buffer(64)
        _err(self.h, lib().aidw_exchange_setup(self.h, int(rank), int(world), buf))
        return buf.raw

    def exchange_connect(self, handles):
        """Map every rank's buffer (``handles``: the all-gathered 64-byte handles)."""
        blob = b"".join(handles)
        _err(self.h, lib().aidw_exchange_connect(self.h, ctypes.c_char_p(blob)))
        self.exchanged = True

    def exchange_close(self):
        _err(self.h, lib().aidw_exchange_close(self.h))
        self.exchanged = False

    def run_host(self, qx_host, qy_host, k=10, levels=LEVELS_DEFAULT, rbounds=GLOBAL, r_min=0.0, r_max=2.0,
                 muform=NORMALIZED, out=None, stream=None):
        """Single-GPU path from HOST buffers through the C ABI (aidw_run_host)."""
        qx_host = torch.as_tensor(qx_host, dtype=self.tdtype).contiguous()
        qy_host = torch.as_tensor(qy_host, dtype=self.tdtype).contiguous()
        if out is None:
            out = torch.empty(qx_host.numel(), dtype=self.tdtype, pin_memory=qx_host.is_pinned())
        with torch.cuda.device(self.device):
            aidw_run_host(self.h, qx_host, qy_host, k, levels, rbounds, r_min, r_max, muform, out, stream)
        return out

    def check(self, stream=None):
        aidw_check(self.h, stream)

    # ---- CUDA graph of the whole path for a fixed batch shape (serving loops)
    def capture(self, nq, k=10, levels=LEVELS_DEFAULT, rbounds=GLOBAL, r_min=0.0, r_max=2.0,
                muform=NORMALIZED, group=None):
        """Capture S1..S5 for batches of ``nq`` queries into one CUDA graph.

        Returns an :class:`AidwGraph` whose static ``qx`` / ``qy`` device buffers the
        caller fills before :meth:`AidwGraph.replay`; ``z`` (and ``r_obs``, ``alpha``)
        hold the results.  One eager warm-up sizes the handle's scratch first (no
        allocation may happen inside a capture).  Replays launch the same kernels
        with the same launch shapes as an eager :meth:`run`, so results are
        bit-identical to it."""
        return AidwGraph(self, nq, k, levels, rbounds, r_min, r_max, muform, group)


class AidwGraph:
    """A captured AIDW step (see :meth:`AIDW.capture`)."""

    def __init__(self, eng, nq, k, levels, rbounds, r_min, r_max, muform, group):
        from .partition import allreduce_bounds
        self.eng, self.nq = eng, int(nq)
        self.qx, self.qy = eng._empty(self.nq), eng._empty(self.nq)
        self.qx.zero_()
        self.qy.zero_()
        self.r_obs, self.d1sq, self.alpha, self.z = (eng._empty(self.nq) for _ in range(4))
        self.minmax = eng._empty(2)
        lv = tuple(float(v) for v in levels)

        def step():
            st = torch.cuda.current_stream(eng.device)
            aidw_knn_robs(eng.h, self.qx, self.qy, k, self.r_obs, self.d1sq, self.minmax, None, st)
            exch = rbounds == GLOBAL and eng.exchanged  # bounds from the device-side exchange
            if rbounds == GLOBAL and group is not None and not exch:
                allreduce_bounds(self.minmax, group)
            aidw_alpha(eng.h, self.r_obs, lv, rbounds, r_min, r_max, None if exch else self.minmax, muform,
                       self.alpha, st)
            aidw_interpolate(eng.h, self.qx, self.qy, self.alpha, self.d1sq, self.z, st)

        side = torch.cuda.Stream(eng.device)
        side.wait_stream(torch.cuda.current_stream(eng.device))
        with torch.cuda.device(eng.device), torch.cuda.stream(side):
            step()  # warm-up: sizes the split / order scratch outside the capture
        torch.cuda.current_stream(eng.device).wait_stream(side)
        torch.cuda.synchronize(eng.device)
        self.graph = torch.cuda.CUDAGraph()
        with torch.cuda.device(eng.device), torch.cuda.graph(self.graph):
            step()

    def replay(self, qx=None, qy=None):
        """Copy new queries into the static buffers (optional) and replay the graph."""
        if qx is not None:
            self.qx.copy_(torch.as_tensor(qx, dtype=self.qx.dtype).reshape(-1), non_blocking=True)
        if qy is not None:
            self.qy.copy_(torch.as_tensor(qy, dtype=self.qy.dtype).reshape(-1), non_blocking=True)
        self.graph.replay()
        return self.z
