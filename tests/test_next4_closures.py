"""NEXT-4: the rest of the paper's sediment closures -- Eq.4's
depth-dependent A_J and a general (integer) Grass exponent m of Eq.3
(P:60-63).  Oracle pins (worked example, exact scalings, closed forms) on CPU;
GPU parity under -m gpu."""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import oracle
import synth

G = 9.81


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def test_eq4_worked_example():
    """Eq.4 at n_M = 0.02, s = 2.65, H = 1, d50 = 1e-3 (7.74e-5);
    closed form evaluated in 40-digit mpmath."""
    mp.mp.dps = 40
    exact = mp.mpf("0.05") * mp.mpf("0.02") ** 3 / (
        (mp.mpf("2.65") - 1) * mp.sqrt(mp.mpf("9.81")) * mp.mpf("1e-3"))
    a = oracle.aj_eq4(G, 0.02, 2.65, 1.0, 1e-3)
    assert rel(a, float(exact)) < 1e-14
    assert abs(a - 7.74e-5) < 5e-8


def test_eq4_exact_scalings():
    """A_J is cubic in n_M and proportional to H^(-1/2): doubling n gives 8x and
    quadrupling H halves it -- exactly, as powers of two."""
    a = oracle.aj_eq4(G, 0.03, 2.65, 1.3, 1e-3)
    assert oracle.aj_eq4(G, 0.06, 2.65, 1.3, 1e-3) == 8 * a
    assert oracle.aj_eq4(G, 0.03, 2.65, 4 * 1.3, 1e-3) == a / 2


def test_grass_general_exponent():
    """Eq.3 J0 = A v |v|^m: m = 2 is bitwise the hot-path formula; v = (3,4)
    gives |v| = 5, so m = 3 -> 125 A v and m = 0 -> A v."""
    assert oracle.grass_m(0.001, 2, 3.0, 4.0) == oracle.grass(0.001, 3.0, 4.0)
    jx, jy, ja = oracle.grass_m(0.001, 3, 3.0, 4.0)
    assert rel(jx, 0.375) < 1e-15 and rel(jy, 0.5) < 1e-15 and rel(ja, 0.625) < 1e-15
    assert oracle.grass_m(0.002, 0, 3.0, 4.0) == (0.006, 0.008, 0.01)


def test_eq4_channel_exner_walls():
    """W2 (walled uniform current) with Eq.4's A_J: the bed changes only at the
    walls, by -/+ tau W A_J(H) u~^3 / h (closed form), where the Manning n_M that
    sets A_J also slows the half-step velocity: u~ = u / (1 + (tau/2) gamma)."""
    nx, ny, K = 8, 3, 0.25
    p = oracle.Params(K=K, n_manning=0.0, aj_mode=1, s_rel=2.65, d50=1e-3, C_J=0.0)
    o = oracle.Oracle(nx, ny, 1.0, p)
    one = np.ones((ny, nx)); z = np.zeros((ny, nx))
    o.set_state(one, one, z, z, 0.4)
    o.set_fields(n_manning=np.full((ny, nx), 0.02))
    st, dt, _ = o.step(1)
    b = o.get_state()[3]
    A = oracle.aj_eq4(G, 0.02, 2.65, 1.0, 1e-3)
    gam = G * 0.02 ** 2 * 1.0 / 1.0
    ut = 1.0 / (1.0 + 0.5 * dt[0] * gam)
    db = dt[0] * (1 / 0.6) * A * ut ** 3
    assert np.allclose(b[:, 0], -db, rtol=1e-12, atol=0)
    assert np.allclose(b[:, -1], db, rtol=1e-12, atol=0)
    assert np.all(b[:, 1:-1] == 0.0)


def test_grass_m3_dt_term():
    """Eq.7's D = max|J0|/(1-psi) with m = 3: single moving cell, |J0| = A |v|^4."""
    p = oracle.Params(K=0.5, A_J=100.0, m_grass=3)
    o = oracle.Oracle(3, 3, 1.0, p)
    h = np.zeros((3, 3)); h[1, 1] = 1.0
    hu = np.zeros((3, 3)); hu[1, 1] = 0.5
    z = np.zeros((3, 3))
    o.set_state(h, hu, z, z, 0.4)
    M = o.reduce_M()
    assert rel(M[2], 100.0 * 0.5 ** 4 / 0.6) < 1e-15
    st, tau, lim = o.tau_from_M(M)
    assert lim == 2 and rel(tau, 0.5 * 1.0 / (2 * M[2])) < 1e-15


@pytest.mark.gpu
@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("case", ["eq4_field", "eq4_scalar", "m3", "m0"])
def test_gpu_closure_parity(path, case):
    from paper_2103_15196_b200 import build, csph
    build.build()
    c = synth.config("C3", 200, 170)
    h, hu, hv, b, psi = synth.fill(c)
    p = dict(c.params)
    nfield = None
    if case.startswith("eq4"):
        p.update(aj_mode=1, s_rel=2.65, A_J=0.0)
        if case == "eq4_field":
            nfield = 0.02 + 0.02 * np.random.default_rng(2).random((c.ny, c.nx))
    else:
        p.update(m_grass=3 if case == "m3" else 0)
    ref = oracle.Oracle(c.nx, c.ny, 1.0, oracle.Params(**p))
    ref.set_state(h, hu, hv, b, psi)
    if nfield is not None:
        ref.set_fields(n_manning=nfield)
    st_r, dt_r, _ = ref.step(60)
    g = csph.csph_create(c.nx, c.ny, 1.0, csph.params_from(p, path=path))
    if nfield is not None:
        g.set_fields(n_manning=nfield)
    g.set_state(h, hu, hv, b, psi)
    assert g.step(60, check=False) == st_r
    dt, _ = g.get_dt_log(60)
    assert np.array_equal(dt, dt_r)
    for x, y in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(x, y)
