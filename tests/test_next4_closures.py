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


def test_pinned_pow_vs_mpmath():
    """The pinned x^q of DESIGN.md 3.12 (NEXT-4 real Grass exponent, "m is a constant
    coefficient"): within 1e-13 (relative) of 40-digit mpmath over the range Eq.3 meets
    (s2 = |v|^2 in [1e-30, 1e4], q = m/2 in [0, 4]); exact special cases x^0 = 1, 0^q = 0,
    and powers of two to integer powers."""
    mp.mp.dps = 40
    rng = np.random.default_rng(3103)
    worst = 0.0
    for _ in range(4000):
        x = float(10.0 ** rng.uniform(-30, 4))
        q = float(rng.uniform(0.0, 4.0))
        y = oracle.pow_pinned(x, q)
        worst = max(worst, float(abs(mp.mpf(y) / mp.mpf(x) ** mp.mpf(q) - 1)))
    assert worst < 1e-13, worst
    assert oracle.pow_pinned(0.7, 0.0) == 1.0 and oracle.pow_pinned(0.0, 0.0) == 1.0
    assert oracle.pow_pinned(0.0, 1.25) == 0.0
    for e in range(-20, 21, 3):
        assert rel(oracle.pow_pinned(2.0 ** e, 1.5), 2.0 ** (1.5 * e)) < 1e-15


def test_grass_real_exponent_closed_form():
    """Eq.3 with m = 2.5: J0 = A v |v|^2.5; v = (3, 4), |v| = 5 -> |v|^2.5 = 25 sqrt 5, and the
    Eq.7 bed term A |v|^3.5 / (1 - psi) of a single moving cell (40-digit closed forms)."""
    mp.mp.dps = 40
    A = 0.002
    o = oracle.Oracle(3, 3, 1.0, oracle.Params(K=0.5, A_J=A, m_real=2.5))
    h = np.zeros((3, 3)); h[1, 1] = 1.0
    hu = np.zeros((3, 3)); hu[1, 1] = 3.0
    hv = np.zeros((3, 3)); hv[1, 1] = 4.0
    assert o.set_state(h, hu, hv, np.zeros((3, 3)), 0.4) == 0
    M = o.reduce_M()
    exact = mp.mpf(A) * mp.mpf(5) ** mp.mpf("3.5") / (1 - mp.mpf("0.4"))
    assert rel(M[2], float(exact)) < 1e-13
    # the integer path and the real path agree to the pow's accuracy at an integer m
    o3 = oracle.Oracle(3, 3, 1.0, oracle.Params(K=0.5, A_J=A, m_grass=3))
    o3r = oracle.Oracle(3, 3, 1.0, oracle.Params(K=0.5, A_J=A, m_real=3.0))
    for oo in (o3, o3r):
        oo.set_state(h, hu, hv, np.zeros((3, 3)), 0.4)
    assert rel(o3r.reduce_M()[2], o3.reduce_M()[2]) < 1e-14


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
@pytest.mark.parametrize("case", ["eq4_field", "eq4_scalar", "m3", "m0", "m2.5", "m1.7_eq4"])
def test_gpu_closure_parity(path, case):
    from paper_2103_15196_b200 import build, csph
    build.build()
    c = synth.config("C3", 200, 170)
    h, hu, hv, b, psi = synth.fill(c)
    p = dict(c.params)
    nfield = None
    if case.startswith("eq4") or case.endswith("eq4"):
        p.update(aj_mode=1, s_rel=2.65, A_J=0.0)
        if case == "eq4_field":
            nfield = 0.02 + 0.02 * np.random.default_rng(2).random((c.ny, c.nx))
    if case.startswith("m2.5") or case.startswith("m1.7"):
        p.update(m_real=float(case[1:4]))  # real exponent, pinned pow
    elif case in ("m3", "m0"):
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


# ---------------------------------------------------------------- open boundaries

def test_open_boundaries_keep_a_uniform_current():
    """Zero-gradient (open) ghosts (NEXT-4): a uniform current in a
    frictionless channel open at both ends is an exact steady state -- every face
    sees the same two states -- while walls would reflect it."""
    nx, ny = 30, 5
    H0, u0 = 1.2, 0.7
    h = np.full((ny, nx), H0); hu = np.full((ny, nx), H0 * u0); z = np.zeros((ny, nx))
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    o.set_walls(2, 2, 1, 1)
    o.set_state(h, hu, z, z)
    o.step(25)
    H, Qx, Qy, b = o.get_state()
    assert np.all(H == H0) and np.all(Qx == H0 * u0) and np.all(Qy == 0.0)
    w = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    w.set_state(h, hu, z, z)
    w.step(25)
    assert not np.all(w.get_state()[0] == H0)


def test_open_boundary_drains_a_dam_break():
    """A dam break with an open x-high edge: identical to the walled run until the
    front reaches the edge, then water leaves -- the volume never increases and
    ends well below its start."""
    nx, ny = 40, 4
    h = np.zeros((ny, nx)); h[:, :20] = 1.0
    z = np.zeros((ny, nx))
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    o.set_walls(1, 2, 1, 1)
    o.set_state(h, z, z, z)
    w = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    w.set_state(h, z, z, z)
    o.step(5); w.step(5)
    for a, b in zip(o.get_state(), w.get_state()):
        assert np.array_equal(a, b)  # the front is still far from the edge
    V = [math.fsum(o.get_state()[0].ravel())]
    for _ in range(60):
        st, _, _ = o.step(10)
        assert st == 0
        V.append(math.fsum(o.get_state()[0].ravel()))
    assert V[-1] < 0.7 * V[0]
    assert all(b <= a * (1 + 1e-14) for a, b in zip(V, V[1:]))


def test_open_boundaries_keep_lake_at_rest():
    """Well-balance with open edges: a dyadic lake at rest stays bitwise at rest."""
    c = synth.config("C2", 64, 48)
    h, hu, hv, b, psi = synth.fill(c)
    o = oracle.Oracle(c.nx, c.ny, 1.0, oracle.Params(**c.params))
    o.set_walls(2, 2, 2, 2)
    o.set_state(h, hu, hv, b, psi)
    o.step(200)
    H, Qx, Qy, bn = o.get_state()
    assert np.array_equal(H, h) and np.all(Qx == 0.0) and np.array_equal(bn, b)


@pytest.mark.gpu
@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("mask", [2, 5, 15])
def test_gpu_open_boundary_parity(path, mask):
    from paper_2103_15196_b200 import build, csph
    build.build()
    c = synth.config("C4", 190, 210)
    h, hu, hv, b, psi = synth.fill(c)
    sides = [2 if mask & (1 << k) else 1 for k in range(4)]
    ref = oracle.Oracle(c.nx, c.ny, 1.0, oracle.Params(**c.params))
    ref.set_walls(*sides)
    ref.set_state(h, hu, hv, b, psi)
    st_r, dt_r, _ = ref.step(80)
    g = csph.csph_create(c.nx, c.ny, 1.0, csph.params_from(c.params, path=path, open_bc=mask))
    g.set_state(h, hu, hv, b, psi)
    assert g.step(80, check=False) == st_r
    dt, _ = g.get_dt_log(80)
    assert np.array_equal(dt, dt_r)
    for x, y in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(x, y)


@pytest.mark.gpu
def test_gpu_open_boundary_strips():
    """Open y edges with the strip decomposition (3 strips on one GPU)."""
    from paper_2103_15196_b200 import build, csph
    build.build()
    c = synth.config("C5", 160, 150)
    f = synth.fill(c)
    p = csph.params_from(c.params, open_bc=12)
    a = csph.csph_create(c.nx, c.ny, 1.0, p)
    a.set_state(*f); a.step(40)
    m = csph.csph_create_multi(c.nx, c.ny, 1.0, p, [0, 0, 0])
    m.set_state(*f); m.step(40)
    for x, y in zip(a.get_state(), m.get_state()):
        assert np.array_equal(x, y)
