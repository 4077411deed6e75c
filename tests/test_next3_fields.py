"""NEXT-3: the paper's spatial model inputs -- Manning n_M(x,y) and
absorption beta(x,y) -- and the water source term sigma of Eq.6 (P:105,
P:109) as sigma = s - beta H (reading #21, 3.11).  Oracle pins (closed
forms / invariants) on CPU; GPU parity vs the oracle under -m gpu."""
import math

import numpy as np
import pytest

import oracle
import synth

G = 9.81


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def lake(nx=12, ny=9, H=1.0):
    return (np.full((ny, nx), H), np.zeros((ny, nx)), np.zeros((ny, nx)), np.zeros((ny, nx)))


def test_rain_on_a_lake_closed_form():
    """Uniform rain s on a flat lake at rest: no fluxes, H' = H + tau s exactly."""
    s = 2e-4
    o = oracle.Oracle(12, 9, 1.0, oracle.Params())
    o.set_state(*lake())
    assert o.set_fields(src=np.full((9, 12), s)) == 0
    st, dt, _ = o.step(1)
    H, Qx, Qy, b = o.get_state()
    assert np.all(H == 1.0 + dt[0] * s)
    assert np.all(Qx == 0.0) and np.all(Qy == 0.0)


def test_absorption_closed_form():
    """Uniform absorption beta (implicit): H' = H / (1 + tau beta)."""
    beta = 0.05
    o = oracle.Oracle(12, 9, 1.0, oracle.Params())
    o.set_state(*lake(H=2.0))
    o.set_fields(beta=np.full((9, 12), beta))
    st, dt, _ = o.step(1)
    H = o.get_state()[0]
    assert np.all(H == 2.0 * (1.0 / (1.0 + dt[0] * beta)))


def test_uniform_manning_field_equals_scalar():
    """A constant n_M field gives bitwise the same run as the scalar parameter."""
    nx, ny = 30, 22
    f = synth.random_state(nx, ny, seed=8)
    p = oracle.Params(n_manning=0.03, A_J=0.01, C_J=2.0)
    a = oracle.Oracle(nx, ny, 1.0, p)
    a.set_state(*f)
    a.step(20)
    b = oracle.Oracle(nx, ny, 1.0, oracle.Params(n_manning=0.0, A_J=0.01, C_J=2.0))
    b.set_state(*f)
    b.set_fields(n_manning=np.full((ny, nx), 0.03))
    b.step(20)
    for x, y in zip(a.get_state(), b.get_state()):
        assert np.array_equal(x, y)


def test_friction_field_is_local():
    """Uniform current; n_M = 0.05 on the left half, 0 on the right: interior
    momentum decays by 1/(1 + tau gamma) only where n_M > 0 (closed form)."""
    nx, ny, H0, u0 = 40, 5, 1.5, 0.8
    n = np.zeros((ny, nx)); n[:, :nx // 2] = 0.05
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    o.set_state(np.full((ny, nx), H0), np.full((ny, nx), H0 * u0), np.zeros((ny, nx)),
                np.zeros((ny, nx)))
    o.set_fields(n_manning=n)
    st, dt, _ = o.step(1)
    Qx = o.get_state()[1]
    gam = G * 0.05 ** 2 * u0 / H0 ** (4.0 / 3.0)
    assert rel(Qx[2, 8], H0 * u0 / (1 + dt[0] * gam)) < 1e-12
    assert Qx[2, 30] == H0 * u0


def test_source_mass_balance():
    """Walls, beta = 0: sum H' = sum H + tau sum s (rounding level)."""
    nx, ny = 36, 28
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=12)
    src = np.where(np.arange(nx)[None, :] % 7 == 0, 1e-3, 0.0) * np.ones((ny, 1))
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params(n_manning=0.02))
    o.set_state(h, hu, hv, b, psi)
    o.set_fields(src=src)
    V0 = math.fsum(h.ravel())
    st, dt, _ = o.step(10)
    assert st == 0
    V1 = math.fsum(o.get_state()[0].ravel())
    assert abs(V1 - (V0 + math.fsum(dt) * math.fsum(src.ravel()))) / V0 < 1e-12


def test_point_source_wets_a_dry_bed():
    """A point inflow on a dry plain (P:188 Index_Q cells stay active): water
    appears at the source and spreads, and the volume equals the inflow."""
    nx, ny = 21, 21
    src = np.zeros((ny, nx)); src[10, 10] = 0.05
    h = np.zeros((ny, nx)); h[0, 0] = 1e-2  # one wet cell so tau is finite
    z = np.zeros((ny, nx))
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    o.set_state(h, z, z, z)
    o.set_fields(src=src)
    st, dt, _ = o.step(30)
    assert st == 0
    H = o.get_state()[0]
    assert H[10, 10] > 1e-6 and H[10, 11] > 0.0
    assert rel(math.fsum(H.ravel()), 1e-2 + math.fsum(dt) * 0.05) < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("path", [0, 1])
def test_gpu_fields_parity(path):
    from paper_2103_15196_b200 import build, csph
    build.build()
    c = synth.config("C5", 260, 230)
    h, hu, hv, b, psi = synth.fill(c)
    rng = np.random.default_rng(3)
    n = 0.02 + 0.02 * rng.random((c.ny, c.nx))
    beta = np.where(rng.random((c.ny, c.nx)) < 0.3, 1e-3, 0.0)
    src = np.zeros((c.ny, c.nx)); src[40:44, 100:104] = 2e-3; src[200, 20] = 5e-3
    p = dict(c.params)
    ref = oracle.Oracle(c.nx, c.ny, 1.0, oracle.Params(**p))
    ref.set_state(h, hu, hv, b, psi)
    ref.set_fields(n, beta, src)
    st_r, dt_r, lim_r = ref.step(60)
    g = csph.csph_create(c.nx, c.ny, 1.0, csph.params_from(p, path=path))
    g.set_fields(n, beta, src)
    g.set_state(h, hu, hv, b, psi)
    assert g.step(60, check=False) == st_r
    dt, lim = g.get_dt_log(60)
    assert np.array_equal(dt, dt_r)
    for x, y in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(x, y)
