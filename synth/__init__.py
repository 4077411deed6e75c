"""Seeded synthetic inputs.

Serves both sides (oracle runs and the CUDA path) with the same arrays.  It
contains none of the method's arithmetic: only initial states and the
physical parameters of each config.  The generator itself is ``synth/gen.c``
(counter-based splitmix64 hash, value noise, fBm), built by ``build()``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "libsynth.so")
_lib = None


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "gen.c")
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(src):
        subprocess.check_call(["gcc", "-O2", "-std=c99", "-ffp-contract=off", "-fopenmp",
                               "-Wall", "-shared", "-fPIC", "-o", _SO, src, "-lm"])
    return _SO


def _L():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_SO)
        D = ctypes.POINTER(ctypes.c_double)
        L.syn_fill.restype = ctypes.c_int
        L.syn_fill.argtypes = [ctypes.c_int, ctypes.c_int] + [ctypes.c_int64] * 4 + [D] * 5
        L.syn_hash_u.restype = ctypes.c_double
        L.syn_hash_u.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
        L.syn_fbm.restype = ctypes.c_double
        L.syn_fbm.argtypes = [ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_int64, ctypes.c_int64]
        _lib = L
    return _lib


@dataclass
class Config:
    """A workload: grid, cell size, physics parameters."""
    name: str
    cfg: int
    nx: int
    ny: int
    dx: float = 1.0
    variant: int = 0
    params: dict = field(default_factory=dict)

    @property
    def cells(self) -> int:
        return self.nx * self.ny


_PHYS_ON = dict(n_manning=0.03, A_J=0.001, C_J=2.0, C_Sh=4.0, d50=1e-3)


def config(name: str, n: int | None = None, ny: int | None = None) -> Config:
    """C1..C5 of DESIGN.md section 6, optionally rescaled to n x ny."""
    base = {
        "C1": Config("C1", 1, 200, 4, params=dict(n_manning=0.0, A_J=0.0, C_Sh=0.0)),
        "C1S": Config("C1S", 1, 200, 4, variant=1, params=dict(n_manning=0.0, A_J=0.0, C_Sh=0.0)),
        "C2": Config("C2", 2, 1024, 1024, params=dict(_PHYS_ON)),
        "C2N": Config("C2N", 2, 1024, 1024, variant=1, params=dict(_PHYS_ON)),
        "C3": Config("C3", 3, 4096, 4096, params=dict(_PHYS_ON, n_manning=0.025)),
        "C4": Config("C4", 4, 8192, 8192, params=dict(_PHYS_ON)),
        "C4D": Config("C4D", 4, 8192, 8192, variant=1, params=dict(_PHYS_ON)),
        "C5": Config("C5", 5, 16384, 16384, params=dict(_PHYS_ON)),
    }[name]
    if n is not None:
        base.nx = n
        base.ny = ny if ny is not None else n
    return base


def fill(c: Config, j0: int = 0, j1: int | None = None):
    """Initial state rows [j0, j1) of config c: (h, hu, hv, b, psi), each [rows][nx]."""
    j1 = c.ny if j1 is None else j1
    rows = j1 - j0
    out = [np.empty((rows, c.nx), dtype=np.float64) for _ in range(5)]
    D = ctypes.POINTER(ctypes.c_double)
    st = _L().syn_fill(c.cfg, c.variant, c.nx, c.ny, j0, j1,
                       *[a.ctypes.data_as(D) for a in out])
    if st != 0:
        raise ValueError(f"unknown config {c}")
    return tuple(out)


def hash_u(seed: int, i: int, j: int, o: int = 0) -> float:
    return _L().syn_hash_u(seed, i, j, o)


def fbm(seed: int, P0: int, octaves: int, i: int, j: int) -> float:
    return _L().syn_fbm(seed, P0, octaves, i, j)


def random_state(nx: int, ny: int, seed: int, wet_frac: float = 0.7, rough: float = 0.3,
                 vel: float = 0.8, psi_field: bool = True, film: float = 0.0):
    """Small random state with wet/dry islands (tests only): hash-based, so
    reproducible; values are kept away from branch thresholds only
    statistically."""
    rng = np.random.Generator(np.random.Philox(seed))
    b = rough * rng.standard_normal((ny, nx))
    eta0 = np.quantile(b, wet_frac)
    h = np.maximum(0.0, eta0 - b + 0.05 * rng.standard_normal((ny, nx)))
    h[h < 1e-3] = 0.0
    hu = np.where(h > 0, h * vel * rng.standard_normal((ny, nx)), 0.0)
    hv = np.where(h > 0, h * vel * rng.standard_normal((ny, nx)), 0.0)
    psi = 0.3 + 0.2 * rng.random((ny, nx)) if psi_field else np.full((ny, nx), 0.4)
    if film > 0.0:
        # thin films just above eps_dry = 1e-6 with random currents (wet/dry stress)
        f = rng.random((ny, nx)) < film
        hf = 1e-6 + 2e-6 * rng.random((ny, nx))
        h = np.where(f, hf, h)
        hu = np.where(f, hf * rng.standard_normal((ny, nx)), hu)
        hv = np.where(f, hf * rng.standard_normal((ny, nx)), hv)
    return h, hu, hv, b, psi
