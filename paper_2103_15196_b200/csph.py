"""Thin ctypes binding of ``include/csph.h`` (argument marshalling only).

Every step of the CSPH-TVD path runs in the CUDA kernels of ``libcsph.so``.
There is no CPU fallback: if the library is missing or no CUDA device is
present, the calls raise ``CsphError``.
"""
from __future__ import annotations

import ctypes
import math
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.path.join(_HERE, "libcsph.so")

CSPH_OK, CSPH_EINVAL, CSPH_ENOSTATE, CSPH_ENOMEM, CSPH_ECUDA, CSPH_ENCCL = 0, -1, -2, -3, -4, -5
CSPH_ENEGDEPTH, CSPH_ENONFINITE, CSPH_EDRY = -6, -7, -8
CSPH_PATH_FUSED, CSPH_PATH_STAGED = 0, 1

# every symbol include/csph.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "csph_default_params", "csph_create", "csph_set_state", "csph_set_state_rows", "csph_step",
    "csph_get_state", "csph_get_state_rows", "csph_get_time", "csph_get_dt_log",
    "csph_get_maxima", "csph_set_stream", "csph_strip_rows", "csph_destroy", "csph_strerror",
    "csph_last_error", "csph_nccl_id_bytes", "csph_make_nccl_id", "csph_create_dist",
    "csph_create_multi", "csph_create_multi_rows", "csph_create_dist_rows", "csph_balance_rows",
    "csph_last_launch_count", "csph_profile", "csph_get_profile",
    "csph_selftest_math", "csph_get_tile_stats", "csph_reset_tile_stats",
    "csph_set_fields", "csph_set_fields_rows", "csph_row_weights", "csph_rebalance_rows",
    "csph_ipc_blob_bytes", "csph_ipc_export", "csph_ipc_link", "csph_save_begin",
    "csph_save_wait",
]


class csph_params(ctypes.Structure):
    _fields_ = [
        ("g", ctypes.c_double), ("K", ctypes.c_double), ("eps_dry", ctypes.c_double),
        ("dt_max", ctypes.c_double), ("neg_tol", ctypes.c_double),
        ("n_manning", ctypes.c_double), ("A_J", ctypes.c_double), ("m_grass", ctypes.c_int),
        ("C_J", ctypes.c_double), ("C_Sh", ctypes.c_double), ("d50", ctypes.c_double),
        ("q_plus", ctypes.c_double), ("q_minus", ctypes.c_double), ("precision", ctypes.c_int),
        ("device", ctypes.c_int), ("path", ctypes.c_int), ("tile_rows", ctypes.c_int),
        ("hgs", ctypes.c_int), ("aj_mode", ctypes.c_int), ("s_rel", ctypes.c_double),
        ("open_bc", ctypes.c_int), ("graphs", ctypes.c_int), ("h_bed_min", ctypes.c_double),
        ("m_real", ctypes.c_double), ("halo_push", ctypes.c_int),
    ]


class CsphError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"csph error {code}: {msg}")
        self.code = code


_lib = None
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.POINTER(ctypes.c_int)
_vp = ctypes.c_void_p


def lib():
    """Load libcsph.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(SO_PATH):
            raise CsphError(CSPH_ECUDA, f"{SO_PATH} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(SO_PATH)
        L.csph_default_params.argtypes = [ctypes.POINTER(csph_params)]
        L.csph_default_params.restype = None
        L.csph_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.POINTER(csph_params)]
        L.csph_create.restype = _vp
        L.csph_create_dist.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                       ctypes.POINTER(csph_params), ctypes.c_int, ctypes.c_int,
                                       ctypes.c_int, ctypes.c_void_p]
        L.csph_create_dist.restype = _vp
        L.csph_create_multi.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                        ctypes.POINTER(csph_params), ctypes.c_int, _I]
        L.csph_create_multi.restype = _vp
        L.csph_create_dist_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            ctypes.POINTER(csph_params), ctypes.c_int,
                                            ctypes.c_int, _I, ctypes.c_int, ctypes.c_void_p]
        L.csph_create_dist_rows.restype = _vp
        L.csph_create_multi_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                             ctypes.POINTER(csph_params), ctypes.c_int, _I, _I]
        L.csph_create_multi_rows.restype = _vp
        L.csph_balance_rows.argtypes = [ctypes.c_int, ctypes.c_int, _D, _I]
        L.csph_set_state.argtypes = [_vp, _D, _D, _D, _D, _D]
        L.csph_set_state_rows.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _D, _D, _D, _D, _D]
        L.csph_step.argtypes = [_vp, ctypes.c_int]
        L.csph_set_fields.argtypes = [_vp, _D, _D, _D]
        L.csph_set_fields_rows.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _D, _D, _D]
        L.csph_get_state.argtypes = [_vp, _D, _D, _D, _D]
        L.csph_get_state_rows.argtypes = [_vp, ctypes.c_int, ctypes.c_int, _D, _D, _D, _D]
        L.csph_save_begin.argtypes = [_vp, _D, _D, _D, _D]
        L.csph_save_wait.argtypes = [_vp]
        L.csph_get_time.argtypes = [_vp, _D, ctypes.POINTER(ctypes.c_longlong), _D]
        L.csph_get_dt_log.argtypes = [_vp, _D, _I, ctypes.c_int, _I]
        L.csph_get_maxima.argtypes = [_vp, _D]
        L.csph_set_stream.argtypes = [_vp, _vp]
        L.csph_strip_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, _I, _I]
        L.csph_destroy.argtypes = [_vp]
        L.csph_destroy.restype = None
        L.csph_strerror.argtypes = [ctypes.c_int]
        L.csph_strerror.restype = ctypes.c_char_p
        L.csph_last_error.restype = ctypes.c_char_p
        L.csph_nccl_id_bytes.restype = ctypes.c_int
        L.csph_make_nccl_id.argtypes = [ctypes.c_void_p]
        L.csph_profile.argtypes = [_vp, ctypes.c_int]
        L.csph_get_profile.argtypes = [_vp, _D, ctypes.POINTER(ctypes.c_longlong)]
        L.csph_selftest_math.argtypes = [ctypes.c_longlong, ctypes.c_ulonglong,
                                         ctypes.POINTER(ctypes.c_longlong)]
        L.csph_get_tile_stats.argtypes = [_vp, ctypes.POINTER(ctypes.c_longlong)]
        L.csph_reset_tile_stats.argtypes = [_vp]
        L.csph_last_launch_count.argtypes = [_vp]
        L.csph_last_launch_count.restype = ctypes.c_longlong
        L.csph_row_weights.argtypes = [_vp, _D]
        L.csph_rebalance_rows.argtypes = [_vp, _I]
        L.csph_ipc_blob_bytes.restype = ctypes.c_int
        L.csph_ipc_export.argtypes = [_vp, ctypes.c_void_p]
        L.csph_ipc_link.argtypes = [_vp, ctypes.c_char_p, ctypes.c_int]
        _lib = L
    return _lib


def csph_last_error() -> str:
    return lib().csph_last_error().decode()


def csph_strerror(code: int) -> str:
    return lib().csph_strerror(code).decode()


def _check(code: int, what: str) -> int:
    if code != CSPH_OK:
        raise CsphError(code, f"{what}: {csph_last_error()}")
    return code


def _arr(a, shape):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.shape != shape:
        raise ValueError(f"expected shape {shape}, got {a.shape}")
    return a


def _out(a, shape):
    """An output array the library writes in place: no conversion copy is allowed."""
    if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous
            and a.flags.writeable and a.shape == shape):
        raise ValueError(f"expected a writable C-contiguous float64 array of shape {shape}")
    return a


def _p(a):
    return None if a is None else a.ctypes.data_as(_D)


def csph_default_params(**overrides) -> csph_params:
    p = csph_params()
    lib().csph_default_params(ctypes.byref(p))
    for k, v in overrides.items():
        setattr(p, k, v)
    return p


def csph_strip_rows(ny: int, nranks: int, rank: int):
    j0, j1 = ctypes.c_int(), ctypes.c_int()
    _check(lib().csph_strip_rows(ny, nranks, rank, ctypes.byref(j0), ctypes.byref(j1)), "csph_strip_rows")
    return j0.value, j1.value


def csph_balance_rows(ny: int, nranks: int, w) -> list:
    """Load-balanced partition bounds[0..nranks] of ny rows with per-row costs w."""
    import numpy as np
    w = np.ascontiguousarray(w, dtype=np.float64)
    assert w.shape == (ny,)
    b = (ctypes.c_int * (nranks + 1))()
    _check(lib().csph_balance_rows(ny, nranks, w.ctypes.data_as(_D), b), "csph_balance_rows")
    return list(b)


def csph_selftest_math(n: int, seed: int = 1) -> int:
    bad = ctypes.c_longlong()
    _check(lib().csph_selftest_math(n, seed, ctypes.byref(bad)), "csph_selftest_math")
    return bad.value


def csph_nccl_id_bytes() -> int:
    return lib().csph_nccl_id_bytes()


def csph_make_nccl_id() -> bytes:
    buf = ctypes.create_string_buffer(csph_nccl_id_bytes())
    _check(lib().csph_make_nccl_id(buf), "csph_make_nccl_id")
    return buf.raw


class Csph:
    """Owning wrapper of a csph_t* handle; methods mirror the C-ABI calls."""

    def __init__(self, handle, nx: int, ny: int, dx: float, params: csph_params):
        if not handle:
            raise CsphError(CSPH_ECUDA, f"csph_create failed: {csph_last_error()}")
        self.h = handle
        self.nx, self.ny, self.dx, self.params = nx, ny, dx, params

    def __del__(self):
        self.destroy()

    def destroy(self):
        if getattr(self, "h", None):
            lib().csph_destroy(self.h)
            self.h = None

    def set_state(self, h, hu, hv, b, psi=None):
        shp = (self.ny, self.nx)
        a = [_arr(x, shp) for x in (h, hu, hv, b)]
        ps = None if psi is None else _arr(np.broadcast_to(psi, shp), shp)
        return _check(lib().csph_set_state(self.h, *[_p(x) for x in a], _p(ps)), "csph_set_state")

    def set_state_rows(self, j_begin, j_end, h, hu, hv, b, psi=None):
        shp = (j_end - j_begin, self.nx)
        a = [_arr(x, shp) for x in (h, hu, hv, b)]
        ps = None if psi is None else _arr(np.broadcast_to(psi, shp), shp)
        return _check(lib().csph_set_state_rows(self.h, j_begin, j_end, *[_p(x) for x in a], _p(ps)),
                      "csph_set_state_rows")

    def set_fields(self, n_manning=None, beta=None, src=None):
        shp = (self.ny, self.nx)
        a = [None if x is None else _arr(np.broadcast_to(x, shp), shp) for x in (n_manning, beta, src)]
        return _check(lib().csph_set_fields(self.h, *[_p(x) for x in a]), "csph_set_fields")

    def set_fields_rows(self, j_begin, j_end, n_manning=None, beta=None, src=None):
        shp = (j_end - j_begin, self.nx)
        a = [None if x is None else _arr(np.broadcast_to(x, shp), shp) for x in (n_manning, beta, src)]
        return _check(lib().csph_set_fields_rows(self.h, j_begin, j_end, *[_p(x) for x in a]),
                      "csph_set_fields_rows")

    def step(self, nsteps: int, check: bool = True) -> int:
        code = lib().csph_step(self.h, nsteps)
        return _check(code, "csph_step") if check else code

    def get_state(self):
        out = [np.empty((self.ny, self.nx)) for _ in range(4)]
        _check(lib().csph_get_state(self.h, *[_p(x) for x in out]), "csph_get_state")
        return tuple(out)

    def get_state_rows(self, j_begin, j_end):
        out = [np.empty((j_end - j_begin, self.nx)) for _ in range(4)]
        _check(lib().csph_get_state_rows(self.h, j_begin, j_end, *[_p(x) for x in out]),
               "csph_get_state_rows")
        return tuple(out)

    def save_begin(self, h, hu, hv, b):
        """Asynchronous Save into the caller's [ny][nx] float64 arrays (C-contiguous; pinned
        for overlap, e.g. torch pin_memory().numpy()); they must stay alive until save_wait."""
        outs = [x if x is None else _out(x, (self.ny, self.nx)) for x in (h, hu, hv, b)]
        _check(lib().csph_save_begin(self.h, *[_p(x) for x in outs]), "csph_save_begin")

    def save_wait(self):
        _check(lib().csph_save_wait(self.h), "csph_save_wait")

    def get_time(self):
        t, n, d = ctypes.c_double(), ctypes.c_longlong(), ctypes.c_double()
        _check(lib().csph_get_time(self.h, ctypes.byref(t), ctypes.byref(n), ctypes.byref(d)),
               "csph_get_time")
        return t.value, n.value, d.value

    def get_dt_log(self, cap: int):
        dt = np.zeros(max(cap, 1))
        lim = np.zeros(max(cap, 1), dtype=np.int32)
        n = ctypes.c_int()
        _check(lib().csph_get_dt_log(self.h, _p(dt), lim.ctypes.data_as(_I), cap, ctypes.byref(n)),
               "csph_get_dt_log")
        return dt[: n.value].copy(), lim[: n.value].copy()

    def get_maxima(self):
        M = np.zeros(3)
        _check(lib().csph_get_maxima(self.h, _p(M)), "csph_get_maxima")
        return M

    def set_stream(self, stream_ptr: int):
        return _check(lib().csph_set_stream(self.h, ctypes.c_void_p(stream_ptr)), "csph_set_stream")

    def profile(self, enable: bool = True):
        return _check(lib().csph_profile(self.h, int(enable)), "csph_profile")

    def get_profile(self):
        ms, n = ctypes.c_double(), ctypes.c_longlong()
        _check(lib().csph_get_profile(self.h, ctypes.byref(ms), ctypes.byref(n)), "csph_get_profile")
        return ms.value, n.value

    def tile_stats(self):
        c = (ctypes.c_longlong * 3)()
        _check(lib().csph_get_tile_stats(self.h, c), "csph_get_tile_stats")
        return tuple(c)

    def reset_tile_stats(self):
        return _check(lib().csph_reset_tile_stats(self.h), "csph_reset_tile_stats")

    def last_launch_count(self) -> int:
        return lib().csph_last_launch_count(self.h)

    def row_weights(self, w=None):
        """Per-row cost weights of the current state (csph_row_weights) into w (ny doubles)."""
        if w is None:
            w = np.zeros(self.ny)
        w = np.ascontiguousarray(w, dtype=np.float64)
        assert w.shape == (self.ny,)
        _check(lib().csph_row_weights(self.h, _p(w)), "csph_row_weights")
        return w

    def ipc_export(self) -> bytes:
        """This DIST rank's CUDA IPC blob (csph_ipc_export) for the neighbours' csph_ipc_link."""
        buf = ctypes.create_string_buffer(lib().csph_ipc_blob_bytes())
        _check(lib().csph_ipc_export(self.h, buf), "csph_ipc_export")
        return buf.raw

    def ipc_link(self, blobs: list[bytes] | None):
        """Map every rank's buffers (csph_ipc_link: halo push and peer combine); all ranks'
        blobs in rank order, or None to drop the links."""
        if blobs is None:
            return _check(lib().csph_ipc_link(self.h, None, 0), "csph_ipc_link")
        return _check(lib().csph_ipc_link(self.h, b"".join(blobs), len(blobs)), "csph_ipc_link")

    def rebalance_rows(self, bounds):
        """Move to new strip bounds (collective for DIST; csph_rebalance_rows)."""
        b = (ctypes.c_int * len(bounds))(*bounds)
        return _check(lib().csph_rebalance_rows(self.h, b), "csph_rebalance_rows")


def _params(params: csph_params | dict | None) -> csph_params:
    if isinstance(params, csph_params):
        return params
    return csph_default_params(**(params or {}))


def csph_create(nx: int, ny: int, dx: float, params=None) -> Csph:
    p = _params(params)
    return Csph(lib().csph_create(nx, ny, dx, ctypes.byref(p)), nx, ny, dx, p)


def csph_create_multi(nx: int, ny: int, dx: float, params, devices) -> Csph:
    p = _params(params)
    arr = (ctypes.c_int * len(devices))(*devices)
    return Csph(lib().csph_create_multi(nx, ny, dx, ctypes.byref(p), len(devices), arr), nx, ny, dx, p)


def csph_create_multi_rows(nx: int, ny: int, dx: float, params, devices, bounds) -> Csph:
    p = _params(params)
    arr = (ctypes.c_int * len(devices))(*devices)
    b = (ctypes.c_int * len(bounds))(*bounds)
    return Csph(lib().csph_create_multi_rows(nx, ny, dx, ctypes.byref(p), len(devices), arr, b),
                nx, ny, dx, p)


def csph_create_dist_rows(nx: int, ny: int, dx: float, params, rank: int, nranks: int, bounds,
                          local_device: int, nccl_id: bytes) -> Csph:
    p = _params(params)
    buf = ctypes.create_string_buffer(nccl_id, len(nccl_id))
    b = (ctypes.c_int * len(bounds))(*bounds)
    return Csph(lib().csph_create_dist_rows(nx, ny, dx, ctypes.byref(p), rank, nranks, b,
                                            local_device, buf), nx, ny, dx, p)


def csph_create_dist(nx: int, ny: int, dx: float, params, rank: int, nranks: int,
                     local_device: int, nccl_id: bytes) -> Csph:
    p = _params(params)
    buf = ctypes.create_string_buffer(nccl_id, len(nccl_id))
    return Csph(lib().csph_create_dist(nx, ny, dx, ctypes.byref(p), rank, nranks, local_device, buf),
                nx, ny, dx, p)


def params_from(physics: dict | None = None, **kw) -> csph_params:
    """Default params with the physics dict of a synth.Config applied."""
    d = dict(physics or {})
    d.update(kw)
    if "dt_max" in d and d["dt_max"] is None:
        d["dt_max"] = math.inf
    return csph_default_params(**d)
