"""B200-native Peaceman–Rachford ADI (arXiv:2006.07583) — Python binding.

A thin ctypes layer over ``libadi.so`` (the C-ABI of ``include/adi.h``).  It
only marshals arguments: every step of the method runs in the library's
sm_100a CUDA kernels.  There is no CPU fallback; if the library or a CUDA
device is missing, calls raise.

Module-level functions carry the C names (``adi_create``, ``adi_step`` ...);
``AdiSolver`` wraps a handle.  Host arrays are numpy float64 (C order); device
arrays are anything exposing ``data_ptr()`` (torch CUDA tensors, float64,
contiguous).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

from .build import LIB_PATH, build as build_library  # noqa: F401

ADI_CFD = 0
ADI_MFD = 1
ADI_CFD_FULL = 2   # the full-matrix CFD variant with a Cerjan layer (f4)
ADI_OK = 0
ADI_EINVAL = -1
ADI_ENOMEM = -2
ADI_ECUDA = -3
ADI_EZEROPIVOT = -4
ADI_ENONFINITE = -5
ADI_ESTATE = -6
ADI_ENCCL = -7
ADI_WUNSTABLE = 1
ADI_K_SWEEPS = 0
ADI_RHO = 1
ADI_CHECK_FINITE = 2
ADI_TILE_CHUNKS = 3
ADI_TIMING = 4
ADI_EPS = 5
ADI_K_MIN = 6
ADI_ABSORB_WIDTH = 7
ADI_ABSORB_RATE = 8
ADI_PREFETCH = 9
ADI_CARRY = 10
ADI_GRAPH = 11
ADI_THREAD_LINES = 12
ADI_ASYNC_STORE = 13
ADI_DIST_FUSED = 14
ADI_WARP_LINES = 15
ADI_STEP_INDEX = 16
ADI_FRAG_TILES = 17
# kernel kinds (adi_get_kernel_times index, include/adi.h enum adi_kernel_kind)
ADI_KK_PROLOGUE = 0
ADI_KK_ROW = 1
ADI_KK_COL = 2
ADI_KK_FINAL = 3
ADI_KK_EDGE = 4
ADI_NKINDS = 5
ADI_DIST_HALO = 0
ADI_DIST_TRANSPOSE = 1
KERNEL_KINDS = ("prologue", "row", "col", "final", "edge")

_STATUS = {0: "ADI_OK", -1: "ADI_EINVAL", -2: "ADI_ENOMEM", -3: "ADI_ECUDA", -4: "ADI_EZEROPIVOT",
           -5: "ADI_ENONFINITE", -6: "ADI_ESTATE", -7: "ADI_ENCCL", 1: "ADI_WUNSTABLE"}


class AdiError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"{_STATUS.get(code, code)}: {msg}")
        self.code = code


class adi_stats(ctypes.Structure):
    _fields_ = [("steps", ctypes.c_longlong), ("t", ctypes.c_double), ("nonfinite", ctypes.c_int),
                ("k_sweeps", ctypes.c_int), ("kernel_launches", ctypes.c_longlong),
                ("last_test", ctypes.c_double * 2), ("last_k", ctypes.c_int * 2),
                ("device_bytes", ctypes.c_longlong), ("host_launches", ctypes.c_longlong)]


_lib = None


def lib():
    """Load libadi.so (built in-tree by ``build()``); raise if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"CUDA extension {LIB_PATH} is missing: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        I, D, P = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
        H = ctypes.c_void_p
        L.adi_create.argtypes = [I, I, D, D, D, I, ctypes.POINTER(H)]
        L.adi_create_batch.argtypes = [I, I, D, D, D, I, I, ctypes.POINTER(H)]
        L.adi_set_param.argtypes = [H, I, D]
        L.adi_set_stream.argtypes = [H, P]
        L.adi_set_fields.argtypes = [H, P, P, P]
        L.adi_set_fields_device.argtypes = [H, P, P, P]
        L.adi_set_fields_async.argtypes = [H, P, P, P]
        L.adi_get_fields_async.argtypes = [H, P, P, P]
        L.adi_set_source.argtypes = [H, P, I, I, P, I]
        L.adi_set_point_sources.argtypes = [H, P, P, P, I]
        L.adi_set_boundary.argtypes = [H, P, P, I]
        L.adi_set_media.argtypes = [H, P, P, P]
        L.adi_create_dist.argtypes = [I, I, D, D, D, I, I, P, I, I, ctypes.POINTER(H)]
        L.adi_nccl_unique_id.argtypes = [P]
        L.adi_dist_bands.argtypes = [I, I, P]
        try:   # (absent from libraries built before round 2: tools/ab_lib.py loads those too)
            L.adi_create_dist_ex.argtypes = [I, I, D, D, D, I, I, P, I, I, I, ctypes.POINTER(H)]
            L.adi_create_dist_local_ex.argtypes = [I, I, D, D, D, I, I, I, I, ctypes.POINTER(H)]
            L.adi_dist_info.argtypes = [H] + [ctypes.POINTER(I)] * 5
            L.adi_check_guards.argtypes = [H, ctypes.POINTER(ctypes.c_longlong)]
            L.adi_plan_halo.argtypes = [I, ctypes.POINTER(I)]
            L.adi_create_dist_local.argtypes = [I, I, D, D, D, I, I, I, ctypes.POINTER(H)]
            L.adi_step_dist_local.argtypes = [ctypes.POINTER(H), I, I]
        except AttributeError:
            pass
        L.adi_step.argtypes = [H, I]
        L.adi_get_fields.argtypes = [H, P, P, P]
        L.adi_get_fields_device.argtypes = [H, P, P, P]
        L.adi_get_stats.argtypes = [H, ctypes.POINTER(adi_stats)]
        L.adi_get_kernel_times.argtypes = [H, P, P, I]
        L.adi_set_trace.argtypes = [H, P, ctypes.c_longlong, I]
        L.adi_get_last_sweeps.argtypes = [H, ctypes.POINTER(I), ctypes.POINTER(I)]
        for f in ("adi_step_begin",):
            getattr(L, f).argtypes = [H, I]
        for f in ("adi_step_rows", "adi_step_cols", "adi_step_end"):
            getattr(L, f).argtypes = [H]
        L.adi_set_band.argtypes = [H, I, I]
        L.adi_band_info.argtypes = [H, P, P, P, P]
        L.adi_halo_bytes.argtypes = [H, I, I, ctypes.POINTER(ctypes.c_size_t)]
        L.adi_halo_pack.argtypes = [H, I, I, P]
        L.adi_halo_unpack.argtypes = [H, I, I, P]
        L.adi_last_error.argtypes = [H]
        L.adi_last_error.restype = ctypes.c_char_p
        L.adi_destroy.argtypes = [H]
        L.adi_destroy.restype = None
        L.adi_version.restype = ctypes.c_char_p
        _lib = L
    return _lib


EXPORTS = ["adi_create", "adi_create_batch", "adi_set_param", "adi_set_stream", "adi_set_fields",
           "adi_set_fields_device", "adi_set_source", "adi_set_point_sources", "adi_set_boundary",
           "adi_set_media", "adi_create_dist", "adi_nccl_unique_id", "adi_dist_bands", "adi_plan_halo", "adi_create_dist_local", "adi_step_dist_local", "adi_create_dist_ex",
           "adi_create_dist_local_ex", "adi_dist_info", "adi_check_guards", "adi_step", "adi_step_begin", "adi_step_rows", "adi_step_cols", "adi_step_end", "adi_set_band",
           "adi_band_info", "adi_halo_bytes", "adi_halo_pack", "adi_halo_unpack",
           "adi_get_fields", "adi_get_fields_device", "adi_set_fields_async", "adi_get_fields_async", "adi_get_stats", "adi_get_kernel_times",
           "adi_set_trace", "adi_get_last_sweeps", "adi_last_error",
           "adi_destroy", "adi_version"]


def _ptr(a):
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return ctypes.c_void_p(a.data_ptr())
    return a.ctypes.data_as(ctypes.c_void_p)


def _host(a, dtype=np.float64):
    return None if a is None else np.ascontiguousarray(a, dtype=dtype)


def _check(h, rc, what):
    if rc < 0:
        msg = lib().adi_last_error(h).decode() if h else ""
        raise AdiError(rc, f"{what}: {msg}")
    return rc


# ---- C-named functions ------------------------------------------------------
def adi_create(nx, ny, h, dt, c, method):
    return adi_create_batch(nx, ny, h, dt, c, method, 1)


def adi_create_batch(nx, ny, h, dt, c, method, batch):
    hd = ctypes.c_void_p()
    rc = lib().adi_create_batch(nx, ny, h, dt, c, method, batch, ctypes.byref(hd))
    _check(None, rc, "adi_create")
    return hd, rc


def adi_nccl_unique_id():
    """The 128-byte NCCL unique id for adi_create_dist (call on one rank, share with all)."""
    buf = ctypes.create_string_buffer(128)
    _check(None, lib().adi_nccl_unique_id(buf), "adi_nccl_unique_id")
    return buf.raw


def adi_create_dist(nx, ny, h, dt, c, method, batch, unique_id, rank, nranks):
    """One rank of a line-sharded grid with the NCCL halo exchange inside adi_step."""
    hd = ctypes.c_void_p()
    uid = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
    rc = lib().adi_create_dist(nx, ny, h, dt, c, method, batch, uid, rank, nranks, ctypes.byref(hd))
    _check(None, rc, "adi_create_dist")
    return hd, rc


def adi_create_dist_ex(nx, ny, h, dt, c, method, batch, unique_id, rank, nranks, mode):
    """adi_create_dist with the decomposition mode (ADI_DIST_HALO / ADI_DIST_TRANSPOSE)."""
    hd = ctypes.c_void_p()
    uid = None if unique_id is None else ctypes.create_string_buffer(bytes(unique_id), 128)
    rc = lib().adi_create_dist_ex(nx, ny, h, dt, c, method, batch, uid, rank, nranks, mode, ctypes.byref(hd))
    _check(None, rc, "adi_create_dist_ex")
    return hd, rc


def adi_check_guards(hd):
    """Guard words overwritten since allocation (needs ADI_GUARD_CHECK=1 at allocation)."""
    v = ctypes.c_longlong(0)
    _check(hd, lib().adi_check_guards(hd, ctypes.byref(v)), "adi_check_guards")
    return int(v.value)


def adi_dist_info(hd):
    """(mode, rows0, rows1, cols0, cols1): the owned rows (y) and columns (x) of a rank."""
    v = [ctypes.c_int(0) for _ in range(5)]
    _check(hd, lib().adi_dist_info(hd, *[ctypes.byref(x) for x in v]), "adi_dist_info")
    return tuple(int(x.value) for x in v)


def adi_create_dist_local(nx, ny, h, dt, c, method, batch, nranks, mode=0):
    """All ranks of a line-sharded grid in this process on the current device (loopback
    transport, include/adi.h); returns the list of handles."""
    hs = (ctypes.c_void_p * nranks)()
    rc = lib().adi_create_dist_local_ex(nx, ny, h, dt, c, method, batch, nranks, mode, hs)
    if rc < 0:
        raise AdiError(rc, f"adi_create_dist_local: {_STATUS.get(rc, rc)}")
    return [ctypes.c_void_p(x) for x in hs]


def adi_create_dist_local_ex(nx, ny, h, dt, c, method, batch, nranks, mode):
    return adi_create_dist_local(nx, ny, h, dt, c, method, batch, nranks, mode)


def adi_step_dist_local(handles, n):
    hs = (ctypes.c_void_p * len(handles))(*[h.value if isinstance(h, ctypes.c_void_p) else h for h in handles])
    _check(handles[0], lib().adi_step_dist_local(hs, len(handles), n), "adi_step_dist_local")


def adi_dist_bands(npos, nranks):
    """Band cuts of y positions [0, npos) over nranks (the library's plan)."""
    cuts = np.zeros(nranks + 1, dtype=np.int32)
    _check(None, lib().adi_dist_bands(npos, nranks, _ptr(cuts)), "adi_dist_bands")
    return [int(x) for x in cuts]


def adi_plan_halo(method):
    """Halo positions per band side of the band decomposition (the library's plan)."""
    v = ctypes.c_int(0)
    _check(None, lib().adi_plan_halo(method, ctypes.byref(v)), "adi_plan_halo")
    return int(v.value)


def adi_set_param(hd, key, value):
    return _check(hd, lib().adi_set_param(hd, key, float(value)), "adi_set_param")


def adi_set_stream(hd, stream_ptr):
    return _check(hd, lib().adi_set_stream(hd, ctypes.c_void_p(stream_ptr)), "adi_set_stream")


def adi_set_fields(hd, U, V, W):
    U, V, W = _host(U), _host(V), _host(W)
    return _check(hd, lib().adi_set_fields(hd, _ptr(U), _ptr(V), _ptr(W)), "adi_set_fields")


def _pinned_host(a, what):
    # async copies read/write the caller's buffer later: no temporary copies allowed
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]):
        raise ValueError(f"{what}: async transfers need C-contiguous float64 numpy arrays "
                         "(page-locked memory, e.g. torch.empty(...).pin_memory().numpy())")
    return a


def adi_set_fields_async(hd, U, V, W):
    """Enqueue the host->device copy of (U, V̄, W̄) on the handle's stream (buffers must
    stay valid and unmodified until the stream is synchronized)."""
    U, V, W = (_pinned_host(x, "adi_set_fields_async") for x in (U, V, W))
    return _check(hd, lib().adi_set_fields_async(hd, _ptr(U), _ptr(V), _ptr(W)), "adi_set_fields_async")


def adi_get_fields_async(hd, U, V, W):
    """Enqueue the device->host copy of the state into (U, V̄, W̄) on the handle's stream."""
    U, V, W = (_pinned_host(x, "adi_get_fields_async") for x in (U, V, W))
    return _check(hd, lib().adi_get_fields_async(hd, _ptr(U), _ptr(V), _ptr(W)), "adi_get_fields_async")


def adi_set_fields_device(hd, dU, dV, dW):
    return _check(hd, lib().adi_set_fields_device(hd, _ptr(dU), _ptr(dV), _ptr(dW)),
                  "adi_set_fields_device")


def adi_set_source(hd, phi=None, ix=-1, iy=-1, g=None):
    phi, g = _host(phi), _host(g)
    return _check(hd, lib().adi_set_source(hd, _ptr(phi), ix, iy, _ptr(g), 0 if g is None else g.size),
                  "adi_set_source")


def adi_set_point_sources(hd, ix, iy, g=None):
    ix, iy, g = _host(ix, np.int32), _host(iy, np.int32), _host(g)
    return _check(hd, lib().adi_set_point_sources(hd, _ptr(ix), _ptr(iy), _ptr(g),
                                                   0 if g is None else g.size), "adi_set_point_sources")


def adi_set_boundary(hd, edges=None, g=None):
    e = None if edges is None else np.concatenate([np.asarray(x, np.float64).ravel() for x in edges])
    g = _host(g)
    return _check(hd, lib().adi_set_boundary(hd, _ptr(e), _ptr(g), 0 if g is None else g.size),
                  "adi_set_boundary")


def adi_set_media(hd, kappa=None, rinv_v=None, rinv_w=None):
    """Heterogeneous media (f3): kappa (U layout), rho^-1 on the V̄ and W̄ layouts, as
    fp32 (other dtypes are rounded to fp32); all None returns to the scalar medium."""
    k, rv, rw = (_host(a, np.float32) for a in (kappa, rinv_v, rinv_w))
    return _check(hd, lib().adi_set_media(hd, _ptr(k), _ptr(rv), _ptr(rw)), "adi_set_media")


def adi_step(hd, n):
    return _check(hd, lib().adi_step(hd, int(n)), "adi_step")


def adi_step_begin(hd, n):
    return _check(hd, lib().adi_step_begin(hd, int(n)), "adi_step_begin")


def adi_step_rows(hd):
    return _check(hd, lib().adi_step_rows(hd), "adi_step_rows")


def adi_step_cols(hd):
    return _check(hd, lib().adi_step_cols(hd), "adi_step_cols")


def adi_step_end(hd):
    return _check(hd, lib().adi_step_end(hd), "adi_step_end")


def adi_set_band(hd, y0, y1):
    return _check(hd, lib().adi_set_band(hd, int(y0), int(y1)), "adi_set_band")


def adi_band_info(hd):
    v = [ctypes.c_int() for _ in range(4)]
    _check(hd, lib().adi_band_info(hd, *[ctypes.byref(x) for x in v]), "adi_band_info")
    return tuple(x.value for x in v)  # (y0, y1, halo, npos)


def adi_halo_bytes(hd, kind, side):
    n = ctypes.c_size_t()
    _check(hd, lib().adi_halo_bytes(hd, kind, side, ctypes.byref(n)), "adi_halo_bytes")
    return n.value


def adi_halo_pack(hd, kind, side, dev_buf):
    return _check(hd, lib().adi_halo_pack(hd, kind, side, _ptr(dev_buf)), "adi_halo_pack")


def adi_halo_unpack(hd, kind, side, dev_buf):
    return _check(hd, lib().adi_halo_unpack(hd, kind, side, _ptr(dev_buf)), "adi_halo_unpack")


def adi_get_fields(hd, U, V, W):
    return _check(hd, lib().adi_get_fields(hd, _ptr(U), _ptr(V), _ptr(W)), "adi_get_fields")


def adi_get_fields_device(hd, dU, dV, dW):
    return _check(hd, lib().adi_get_fields_device(hd, _ptr(dU), _ptr(dV), _ptr(dW)),
                  "adi_get_fields_device")


def adi_get_stats(hd):
    s = adi_stats()
    _check(hd, lib().adi_get_stats(hd, ctypes.byref(s)), "adi_get_stats")
    return {k: (list(getattr(s, k)) if isinstance(getattr(s, k), ctypes.Array) else getattr(s, k))
            for k, _ in adi_stats._fields_}


def adi_set_trace(hd, buf, cap: int, kind: int):
    """Tile trace of one kernel kind into a device tensor of >= 8 * cap int64 (None: off)."""
    _check(hd, lib().adi_set_trace(hd, _ptr(buf) if buf is not None else None, int(cap), int(kind)),
           "adi_set_trace")


def adi_get_last_sweeps(hd):
    """(rows, columns) sweeps used by the last step's stages."""
    kr, kc = ctypes.c_int(0), ctypes.c_int(0)
    _check(hd, lib().adi_get_last_sweeps(hd, ctypes.byref(kr), ctypes.byref(kc)), "adi_get_last_sweeps")
    return kr.value, kc.value


def adi_get_kernel_times(hd):
    """{kind: (ms, launches)} accumulated since the previous call (needs ADI_TIMING=1)."""
    n = len(KERNEL_KINDS)
    ms = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    _check(hd, lib().adi_get_kernel_times(hd, _ptr(ms), _ptr(cnt), n), "adi_get_kernel_times")
    return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(KERNEL_KINDS)}


def adi_last_error(hd):
    return lib().adi_last_error(hd).decode()


def adi_destroy(hd):
    lib().adi_destroy(hd)


def adi_version():
    return lib().adi_version().decode()


# ---- convenience wrapper ------------------------------------------------------
def shapes(method, nx, ny):
    if method == ADI_CFD_FULL:
        return (ny, nx), (ny, nx), (ny, nx)
    if method == ADI_CFD:
        return (ny, nx), (ny - 2, nx), (ny, nx - 2)
    return (ny + 1, nx + 1), (ny - 1, nx), (ny, nx - 1)


class AdiSolver:
    """One ADI handle (optionally a batch of independent grids)."""

    def __init__(self, nx, ny, h, dt, c, method, *, batch=1, K=8, rho=1.0, check_finite=False,
                 stream=None):
        self.nx, self.ny, self.h, self.dt, self.c, self.method, self.batch = nx, ny, h, dt, c, method, batch
        self.handle, self.create_status = adi_create_batch(nx, ny, h, dt, c, method, batch)
        adi_set_param(self.handle, ADI_K_SWEEPS, K)
        adi_set_param(self.handle, ADI_RHO, rho)
        adi_set_param(self.handle, ADI_CHECK_FINITE, 1 if check_finite else 0)
        if stream is not None:
            adi_set_stream(self.handle, stream)
        self.su, self.sv, self.sw = shapes(method, nx, ny)

    @classmethod
    def adopt(cls, handle, nx, ny, h, dt, c, method, *, batch=1, K=8, rho=1.0, stream=None, status=0):
        """Wrap a handle made elsewhere (adi_create_dist, adi_create_dist_local)."""
        self = cls.__new__(cls)
        self.nx, self.ny, self.h, self.dt, self.c, self.method, self.batch = nx, ny, h, dt, c, method, batch
        self.handle, self.create_status = handle, status
        adi_set_param(self.handle, ADI_K_SWEEPS, K)
        adi_set_param(self.handle, ADI_RHO, rho)
        if stream is not None:
            adi_set_stream(self.handle, stream)
        self.su, self.sv, self.sw = shapes(method, nx, ny)
        return self

    def close(self):
        if self.handle:
            adi_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_param(self, key, value):
        adi_set_param(self.handle, key, value)

    def set_fields(self, U, V, W):
        if hasattr(U, "data_ptr"):
            adi_set_fields_device(self.handle, U, V, W)
        else:
            adi_set_fields(self.handle, U, V, W)

    def set_source(self, phi=None, point=None, g=None):
        ix, iy = (-1, -1) if point is None else point
        adi_set_source(self.handle, phi, ix, iy, g)

    def set_point_sources(self, ix, iy, g=None):
        adi_set_point_sources(self.handle, ix, iy, g)

    def set_boundary(self, edges=None, g=None):
        adi_set_boundary(self.handle, edges, g)

    def set_media(self, kappa=None, rinv_v=None, rinv_w=None):
        return adi_set_media(self.handle, kappa, rinv_v, rinv_w)

    def step(self, n=1):
        return adi_step(self.handle, n)

    def get_fields(self):
        B = (self.batch,) if self.batch > 1 else ()
        U = np.empty(B + self.su)
        V = np.empty(B + self.sv)
        W = np.empty(B + self.sw)
        adi_get_fields(self.handle, U, V, W)
        return U, V, W

    def get_fields_device(self, U, V, W):
        adi_get_fields_device(self.handle, U, V, W)

    def stats(self):
        return adi_get_stats(self.handle)

    def kernel_times(self):
        return adi_get_kernel_times(self.handle)

    @classmethod
    def from_problem(cls, p, **kw):
        """Build a solver from an ``adi_inputs.Problem`` (test/bench helper)."""
        s = cls(p.nx, p.ny, p.h, p.dt, p.c, p.method, K=p.K, rho=p.rho, **kw)
        s.set_fields(p.U, p.V, p.W)
        s.set_source(p.phi, p.src, p.gf)
        s.set_boundary(p.edges, p.gb)
        if getattr(p, "kappa", None) is not None:
            s.set_media(p.kappa, p.rinv_v, p.rinv_w)
        return s
