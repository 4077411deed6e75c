"""CPU oracle for the CSPH-TVD step -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper over ``oracle/csph_oracle.c``: a plain single-threaded C
implementation of the reading R of the paper's method.
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this module.  The
product package ``paper_2103_15196_b200`` never imports it.

Parity-unpinned: fidelity of R to the authors'
unpublished discretization; Exner morphodynamics beyond the invariants.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libcsph_oracle.so")
# the same source in IEEE binary32: the reference of the NEXT-2 fp32 mode
_SO32 = os.path.join(_HERE, "libcsph_oracle32.so")

OK, EINVAL, ENOSTATE, ENOMEM, ENEGDEPTH, ENONFINITE, EDRY = 0, -1, -2, -3, -6, -7, -8
GHOST = 3


def build(force: bool = False) -> str:
    """Compile the oracle with IEEE-strict flags (no FMA contraction), in binary64 and, with
    -DORC_FP32, in binary32 (SSE scalar float arithmetic: every operation rounded to
    float, no excess precision on x86-64)."""
    src = os.path.join(_HERE, "csph_oracle.c")
    hdr = os.path.join(_HERE, "csph_oracle.h")
    for so, extra in ((_SO, []), (_SO32, ["-DORC_FP32"])):
        t = max(os.path.getmtime(src), os.path.getmtime(hdr))
        if force or not os.path.exists(so) or os.path.getmtime(so) < t:
            subprocess.check_call([
                "gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fno-fast-math",
                "-fexcess-precision=standard", "-Wall", "-shared", "-fPIC", "-o", so, src,
                "-lm"] + extra)
    return _SO


class _Params(ctypes.Structure):
    _fields_ = [
        ("g", ctypes.c_double), ("K", ctypes.c_double), ("eps_dry", ctypes.c_double),
        ("dt_max", ctypes.c_double), ("neg_tol", ctypes.c_double),
        ("n_manning", ctypes.c_double), ("A_J", ctypes.c_double), ("m_grass", ctypes.c_int),
        ("C_J", ctypes.c_double), ("C_Sh", ctypes.c_double), ("d50", ctypes.c_double),
        ("q_plus", ctypes.c_double), ("q_minus", ctypes.c_double),
        ("aj_mode", ctypes.c_int), ("s_rel", ctypes.c_double), ("h_bed_min", ctypes.c_double),
        ("m_real", ctypes.c_double),
    ]


@dataclass
class Params:
    g: float = 9.81
    K: float = 0.25
    eps_dry: float = 1e-6
    dt_max: float = math.inf
    neg_tol: float = 1e-12
    n_manning: float = 0.0
    A_J: float = 0.0
    m_grass: int = 2
    C_J: float = 0.0
    C_Sh: float = 0.0
    d50: float = 1e-3
    q_plus: float = 0.0
    q_minus: float = 0.0
    aj_mode: int = 0
    s_rel: float = 2.65
    h_bed_min: float = -1.0  # reading #31 cut-off depth; < 0: d50
    m_real: float = -1.0     # NEXT-4 real Grass exponent (pinned pow); < 0: m_grass

    def to_c(self) -> _Params:
        return _Params(self.g, self.K, self.eps_dry, self.dt_max, self.neg_tol,
                       self.n_manning, self.A_J, self.m_grass, self.C_J, self.C_Sh,
                       self.d50, self.q_plus, self.q_minus, self.aj_mode, self.s_rel,
                       self.h_bed_min, self.m_real)


_libs = {}
_D = ctypes.POINTER(ctypes.c_double)


def lib(precision: int = 64):
    """The oracle library: binary64 (default, R itself) or binary32 (precision=32)."""
    if precision not in _libs:
        build()
        L = ctypes.CDLL(_SO if precision == 64 else _SO32)
        vp = ctypes.c_void_p
        L.orc_create.restype = vp
        L.orc_create.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.POINTER(_Params)]
        L.orc_destroy.argtypes = [vp]
        L.orc_set_walls.argtypes = [vp] + [ctypes.c_int] * 4
        L.orc_set_state.argtypes = [vp, _D, _D, _D, _D, _D]
        L.orc_set_state_padded.argtypes = [vp, _D, _D, _D, _D, _D]
        L.orc_get_state.argtypes = [vp, _D, _D, _D, _D]
        L.orc_set_fields.argtypes = [vp, _D, _D, _D]
        L.orc_get_state_padded.argtypes = [vp, _D, _D, _D, _D]
        L.orc_reduce_M.argtypes = [vp, _D]
        L.orc_tau_from_M.argtypes = [vp, _D, _D, ctypes.POINTER(ctypes.c_int)]
        L.orc_step_tau.argtypes = [vp, ctypes.c_double]
        L.orc_step.argtypes = [vp, ctypes.c_int, _D, ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int)]
        L.orc_get_time.argtypes = [vp, _D, ctypes.POINTER(ctypes.c_longlong), _D]
        L.orc_get_debug.argtypes = [vp, ctypes.c_char_p, _D]
        L.orc_grass.argtypes = [ctypes.c_double] * 3 + [_D] * 3
        L.orc_grass_m.argtypes = [ctypes.c_double, ctypes.c_int] + [ctypes.c_double] * 2 + [_D] * 3
        L.orc_aj_eq4.restype = ctypes.c_double
        L.orc_aj_eq4.argtypes = [ctypes.c_double] * 5
        L.orc_slope_flux.restype = ctypes.c_double
        L.orc_slope_flux.argtypes = [ctypes.c_double] * 4
        L.orc_pow_pinned.restype = ctypes.c_double
        L.orc_pow_pinned.argtypes = [ctypes.c_double] * 2
        L.orc_icbrt.restype = ctypes.c_double
        L.orc_icbrt.argtypes = [ctypes.c_double]
        L.orc_gamma.restype = ctypes.c_double
        L.orc_gamma.argtypes = [ctypes.POINTER(_Params)] + [ctypes.c_double] * 3
        L.orc_minmod.restype = ctypes.c_double
        L.orc_minmod.argtypes = [ctypes.c_double] * 2
        L.orc_hll_face.argtypes = [ctypes.c_double] * 9 + [ctypes.c_int] * 2 + [_D]
        L.orc_shamov_gate.argtypes = [ctypes.c_double] * 4
        L.orc_bed_mobile.argtypes = [ctypes.c_double] * 2
        _libs[precision] = L
    return _libs[precision]


def _ptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


class OracleError(RuntimeError):
    def __init__(self, code: int, what: str):
        super().__init__(f"{what}: oracle status {code}")
        self.code = code


class Oracle:
    """One walled (or partially given-ghost) domain of nx x ny cells."""

    def __init__(self, nx: int, ny: int, dx: float, params: Params | None = None,
                 precision: int = 64):
        self.nx, self.ny, self.dx = nx, ny, dx
        self.params = params or Params()
        self._cp = self.params.to_c()
        self._L = lib(precision)
        self._h = self._L.orc_create(nx, ny, dx, ctypes.byref(self._cp))
        if not self._h:
            raise OracleError(EINVAL, "orc_create")

    def __del__(self):
        h = getattr(self, "_h", None)
        if h:
            self._L.orc_destroy(h)
            self._h = None

    @property
    def padded_shape(self):
        return (self.ny + 2 * GHOST, self.nx + 2 * GHOST)

    def set_walls(self, xlo=True, xhi=True, ylo=True, yhi=True):
        """Per side: True/1 wall, 2 open (zero-gradient), False/0 caller-supplied ghosts."""
        st = self._L.orc_set_walls(self._h, int(xlo), int(xhi), int(ylo), int(yhi))
        if st != OK:
            raise OracleError(st, "orc_set_walls")

    def set_state(self, h, hu, hv, b, psi=None) -> int:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (h, hu, hv, b)]
        for a in arrs:
            assert a.shape == (self.ny, self.nx), a.shape
        p = None
        if psi is not None:
            psi = np.ascontiguousarray(np.broadcast_to(psi, (self.ny, self.nx)), dtype=np.float64)
            p = _ptr(psi)
        return self._L.orc_set_state(self._h, *[_ptr(a) for a in arrs], p)

    def set_fields(self, n_manning=None, beta=None, src=None) -> int:
        arrs = []
        for a in (n_manning, beta, src):
            if a is None:
                arrs.append(None)
            else:
                a = np.ascontiguousarray(np.broadcast_to(a, (self.ny, self.nx)), dtype=np.float64)
                arrs.append(a)
        self._fields = arrs  # keep alive during the call
        return self._L.orc_set_fields(self._h, *[None if a is None else _ptr(a) for a in arrs])

    def set_state_padded(self, H, Qx, Qy, b, W) -> int:
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in (H, Qx, Qy, b, W)]
        for a in arrs:
            assert a.shape == self.padded_shape
        return self._L.orc_set_state_padded(self._h, *[_ptr(a) for a in arrs])

    def get_state(self):
        out = [np.empty((self.ny, self.nx)) for _ in range(4)]
        st = self._L.orc_get_state(self._h, *[_ptr(a) for a in out])
        if st != OK:
            raise OracleError(st, "orc_get_state")
        return tuple(out)

    def get_state_padded(self):
        out = [np.empty(self.padded_shape) for _ in range(4)]
        st = self._L.orc_get_state_padded(self._h, *[_ptr(a) for a in out])
        if st != OK:
            raise OracleError(st, "orc_get_state_padded")
        return tuple(out)

    def reduce_M(self):
        M = np.zeros(3)
        self._L.orc_reduce_M(self._h, _ptr(M))
        return M

    def tau_from_M(self, M):
        M = np.ascontiguousarray(M, dtype=np.float64)
        tau = ctypes.c_double(0.0)
        lim = ctypes.c_int(-1)
        st = self._L.orc_tau_from_M(self._h, _ptr(M), ctypes.byref(tau), ctypes.byref(lim))
        return st, tau.value, lim.value

    def step_tau(self, tau: float) -> int:
        return self._L.orc_step_tau(self._h, tau)

    def step(self, nsteps: int):
        """Returns (status, dt_log, limiter_log) for the steps actually done."""
        dt = np.zeros(max(nsteps, 1))
        lim = np.zeros(max(nsteps, 1), dtype=np.int32)
        n = ctypes.c_int(0)
        st = self._L.orc_step(self._h, nsteps, _ptr(dt),
                            lim.ctypes.data_as(ctypes.POINTER(ctypes.c_int)), ctypes.byref(n))
        return st, dt[: n.value].copy(), lim[: n.value].copy()

    def time(self):
        t = ctypes.c_double(0.0)
        s = ctypes.c_longlong(0)
        d = ctypes.c_double(0.0)
        self._L.orc_get_time(self._h, ctypes.byref(t), ctypes.byref(s), ctypes.byref(d))
        return t.value, s.value, d.value

    def debug(self, name: str) -> np.ndarray:
        out = np.empty(self.padded_shape)
        st = self._L.orc_get_debug(self._h, name.encode(), _ptr(out))
        if st != OK:
            raise OracleError(st, f"orc_get_debug({name})")
        return out

    def debug_interior(self, name: str) -> np.ndarray:
        return self.debug(name)[GHOST:-GHOST, GHOST:-GHOST]


# ---- closed-form pieces (the same C functions the step uses) ---------------

def grass(A_J, vx, vy):
    jx, jy, ja = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().orc_grass(A_J, vx, vy, ctypes.byref(jx), ctypes.byref(jy), ctypes.byref(ja))
    return jx.value, jy.value, ja.value


def grass_m(A, m, vx, vy):
    jx, jy, ja = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    lib().orc_grass_m(A, m, vx, vy, ctypes.byref(jx), ctypes.byref(jy), ctypes.byref(ja))
    return jx.value, jy.value, ja.value


def aj_eq4(g, n_manning, s_rel, H, d50):
    return lib().orc_aj_eq4(g, n_manning, s_rel, H, d50)


def slope_flux(J0n, J0abs, C_J, db_dn):
    return lib().orc_slope_flux(J0n, J0abs, C_J, db_dn)


def icbrt(x):
    return lib().orc_icbrt(x)


def pow_pinned(x, q):
    """The pinned x^q of DESIGN.md 3.12 (NEXT-4 real Grass exponent)."""
    return lib().orc_pow_pinned(x, q)


def gamma(params: Params, H, u, v):
    cp = params.to_c()
    return lib().orc_gamma(ctypes.byref(cp), H, u, v)


def minmod(a, b):
    return lib().orc_minmod(a, b)


def hll_face(g, qm, qp, wL=1, wR=1):
    out = np.zeros(3)
    lib().orc_hll_face(g, *qm, *qp, int(wL), int(wR), _ptr(out))
    return out


def shamov_gate(kappa, s2, H, C_Sh):
    return bool(lib().orc_shamov_gate(kappa, s2, H, C_Sh))


def bed_mobile(H, d50):
    """Reading #31: bedload only through a water column deeper than the grain."""
    return bool(lib().orc_bed_mobile(H, d50))


def tau_from_M(nx, ny, dx, params: Params, M):
    o = Oracle(nx, ny, dx, params)
    return o.tau_from_M(M)


def run(nx, ny, dx, params, h, hu, hv, b, psi=None, nsteps=1):
    """Convenience: create, set state, step; returns (state tuple, dt, lim, status)."""
    o = Oracle(nx, ny, dx, params)
    st = o.set_state(h, hu, hv, b, psi)
    if st != OK:
        raise OracleError(st, "set_state")
    st, dt, lim = o.step(nsteps)
    return o.get_state(), dt, lim, st
