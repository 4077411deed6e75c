"""Pins of the CPU oracle against what the paper and the mathematics fix.

Each test names the passage it checks (P:n = PAPER.md line n) and the kind of
pin (worked example / closed form / invariant / analytic solution).  None of
the expected values comes from the oracle itself or from the CUDA path.
The oracle is R of DESIGN.md section 3.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import synth

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
G = 9.81


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


# ---------------------------------------------------------------- closures

def test_grass_worked_example(orc):
    """Eq.3 at A=0.001, m=2; odd in v (closed form)."""
    gg = GOLD["grass"]
    jx, jy, ja = orc.grass(gg["A_J"], *gg["v"])
    assert rel(jx, gg["J0"][0]) < 2e-16 and rel(jy, gg["J0"][1]) < 2e-16
    assert rel(ja, gg["J0_abs"]) < 2e-16
    mx, my, ma = orc.grass(gg["A_J"], -3.0, -4.0)
    assert (mx, my, ma) == (-jx, -jy, ja)
    assert orc.grass(0.001, 0.0, 0.0) == (0.0, 0.0, 0.0)


def test_shamov_gate_threshold(orc):
    """Eq.5: v_k = C_Sh d50^(1/3) H^(1/6); transport iff |v| > v_k."""
    s = GOLD["shamov"]
    kappa = (s["C_Sh"] ** 2) ** 3 * s["d50"] ** 2
    vk = s["v_k"]
    for H in (1.0,):
        assert not orc.shamov_gate(kappa, (vk * 0.999) ** 2, H, s["C_Sh"])
        assert orc.shamov_gate(kappa, (vk * 1.001) ** 2, H, s["C_Sh"])
    # H^(1/6) dependence: at H = 64, v_k doubles
    assert not orc.shamov_gate(kappa, (2 * vk * 0.999) ** 2, 64.0, s["C_Sh"])
    assert orc.shamov_gate(kappa, (2 * vk * 1.001) ** 2, 64.0, s["C_Sh"])
    # C_Sh = 0 disables the gate
    assert orc.shamov_gate(0.0, 0.0, 1.0, 0.0)


def test_slope_flux_worked_example(orc):
    """Eq.2, vector reading: J = J0 - C_J |J0| grad b."""
    s = GOLD["slope_flux"]
    J = orc.slope_flux(s["J0"][0], math.hypot(*s["J0"]), s["C_J"], s["grad_b"][0])
    assert rel(J, s["J"][0]) < 1e-15


def test_manning_worked_example(orc):
    """Friction term of Eq.6, Manning with n_M: gamma*v = g n^2 |v| v / H^(4/3)."""
    m = GOLD["manning"]
    p = orc.Params(n_manning=m["n_M"])
    gam = orc.gamma(p, m["H"], *m["v"])
    assert rel(gam * m["v"][0], m["gamma_v"]) < 1e-14
    # H^(4/3) closed form at H = 8: 16
    assert rel(orc.gamma(p, 8.0, 1.0, 0.0), G * 4e-4 / 16.0) < 1e-15
    assert orc.gamma(orc.Params(n_manning=0.0), 1.0, 1.0, 0.0) == 0.0


def test_icbrt_pinned_recipe(orc):
    """The pinned x^(-1/3) recipe of DESIGN.md 3.10 vs 50-digit mpmath."""
    mp.mp.dps = 50
    xs = np.concatenate([np.logspace(-6, 4, 2000), [1.0, 8.0, 27.0, 1e-6, 0.125]])
    worst = 0.0
    for x in xs:
        y = orc.icbrt(float(x))
        exact = mp.mpf(float(x)) ** (mp.mpf(-1) / 3)
        worst = max(worst, float(abs(mp.mpf(y) / exact - 1)))
    assert worst < 4.5e-16  # within ~2 ulp


def test_minmod_cases(orc):
    """TVD limiter, minmod: ramp keeps the centred slope, extremum clips."""
    q = [1.0, 2.0, 3.0]
    s = orc.minmod(q[1] - q[0], q[2] - q[1])
    assert q[1] - 0.5 * s == 1.5 and q[1] + 0.5 * s == 2.5
    assert orc.minmod(2.0, -2.0) == 0.0
    assert orc.minmod(0.0, 1.0) == 0.0
    assert orc.minmod(-1.0, -3.0) == -1.0
    assert orc.minmod(4.0, 1.0) == 1.0


def test_hll_special_cases(orc):
    """HLL (Harten-Lax-van Leer): symmetric rest -> 0; supercritical -> upwind."""
    z = orc.hll_face(G, (1.0, 1.0, 0.0, 0.0), (1.0, 1.0, 0.0, 0.0))
    assert np.all(z == 0.0)
    # both sides u = -10 > c: S_R < 0 -> F_R exactly
    F = orc.hll_face(G, (1.0, 1.0, -10.0, 0.5), (1.0, 1.0, -10.0, 0.5))
    assert F[0] == -10.0 and F[1] == 100.0 and F[2] == -5.0
    F = orc.hll_face(G, (2.0, 1.0, 12.0, 0.0), (1.5, 0.5, 12.0, 0.0))
    # S_L >= 0 -> F_L with the hydrostatic H*- = eta- - max(b-, b+) = 2 - 1 = 1
    assert F[0] == 12.0 and F[1] == 144.0
    # dry right side: mass flux of the Ritter onset (a+2c)/3 at a = 0 -> 2c/3
    F = orc.hll_face(G, (1.0, 1.0, 0.0, 0.0), (0.0, 0.0, 0.0, 0.0), 1, 0)
    assert rel(F[0], 2 * math.sqrt(G) / 3) < 1e-15
    # both cells dry -> 0
    assert np.all(orc.hll_face(G, (1.0, 1.0, 1.0, 0.0), (1.0, 1.0, 1.0, 0.0), 0, 0) == 0.0)


def _single_cell_tau(orc, H, u, v, K, A_J, psi, dt_max=math.inf):
    p = orc.Params(K=K, A_J=A_J, dt_max=dt_max)
    o = orc.Oracle(3, 3, 1.0, p)
    h = np.zeros((3, 3)); h[1, 1] = H
    hu = np.zeros((3, 3)); hu[1, 1] = H * u
    hv = np.zeros((3, 3)); hv[1, 1] = H * v
    assert o.set_state(h, hu, hv, np.zeros((3, 3)), psi) == 0
    M = o.reduce_M()
    return M, o.tau_from_M(M)


def test_eq7_worked_examples(orc):
    """Eq.7: moving single cell and rest state (closed form)."""
    e = GOLD["eq7_moving"]
    M, (st, tau, lim) = _single_cell_tau(orc, e["H"], e["v"][0], e["v"][1], e["K"], e["A_J"], e["psi"])
    assert st == 0
    t1 = 1.0 / (2 * math.sqrt(M[0])); t2 = 1.0 / M[1]; t3 = 1.0 / (2 * M[2])
    assert rel(t1, e["terms"][0]) < 1e-15 and rel(t2, e["terms"][1]) < 1e-15
    assert rel(t3, e["terms"][2]) < 1e-14
    assert rel(tau, e["tau"]) < 1e-15 and lim == e["limiter"]
    r = GOLD["eq7_rest"]
    M, (st, tau, lim) = _single_cell_tau(orc, 1.0, 0.0, 0.0, r["K"], 0.001, 0.4)
    assert st == 0 and rel(tau, r["tau"]) < 1e-15 and lim == 1
    # supercritical flow (|v| > sqrt(gH)): the particle term h/(2 v_p) binds, limiter 0.
    # H = 0.1, v = 3: t1 = 1/6 < t2 = 1/(3 + sqrt(0.981)) -> tau = K/6 exactly as written
    M, (st, tau, lim) = _single_cell_tau(orc, 0.1, 3.0, 0.0, 0.25, 0.0, 0.4)
    assert st == 0 and lim == 0 and rel(tau, 0.25 / 6.0) < 1e-15
    # dt_max cap -> limiter 3
    M, (st, tau, lim) = _single_cell_tau(orc, 1.0, 0.0, 0.0, 0.5, 0.0, 0.4, dt_max=0.01)
    assert st == 0 and tau == 0.01 and lim == 3
    # all dry, no cap -> EDRY; NaN maxima -> ENONFINITE
    o = orc.Oracle(3, 3, 1.0, orc.Params())
    z = np.zeros((3, 3))
    o.set_state(z, z, z, z)
    assert o.tau_from_M(o.reduce_M())[0] == orc.EDRY
    assert o.tau_from_M(np.array([np.nan, 1.0, 0.0]))[0] == orc.ENONFINITE


# --------------------------------------------------------- worked steps of R

def test_W1_first_step_of_C1(orc):
    """Closed-form first step of the C1 dam, derived by hand
    from R: a = tau0 g/8 etc.  Every other cell bitwise unchanged."""
    mp.mp.dps = 40
    K = mp.mpf("0.25"); g = mp.mpf("9.81"); c = mp.sqrt(g)
    tau0 = K / c
    a = tau0 * g / 8
    exp = {
        "tau0": tau0,
        "FH_99_100": (a + 2 * c) / 3,
        "FH_98_99": c * a / (a + 2 * c),
        "FQ_99_100": a * (a + 2 * c) / 3,
        "FQ_98_99": -c * c * a / (a + 2 * c),
        "H98": 1 - K * K / (K + 16),
        "H100": K * (K + 16) / 24,
    }
    c1 = synth.config("C1")
    h, hu, hv, b, psi = synth.fill(c1)
    o = orc.Oracle(c1.nx, c1.ny, 1.0, orc.Params(K=0.25, **c1.params))
    assert o.set_state(h, hu, hv, b, psi) == 0
    st, dt, lim = o.step(1)
    assert st == 0 and lim[0] == 1
    assert rel(dt[0], float(exp["tau0"])) < 1e-15
    FH = o.debug_interior("FH"); FQ = o.debug_interior("FQx")
    assert rel(FH[0, 100], float(exp["FH_99_100"])) < 1e-14
    assert rel(FH[0, 99], float(exp["FH_98_99"])) < 1e-14
    assert rel(FQ[0, 100], float(exp["FQ_99_100"])) < 1e-14
    assert rel(FQ[0, 99], float(exp["FQ_98_99"])) < 1e-14
    H, Qx, Qy, bn = o.get_state()
    lam = exp["tau0"]
    assert rel(H[0, 98], float(exp["H98"])) < 1e-14
    assert rel(H[0, 100], float(exp["H100"])) < 1e-14
    # H'99 = 1 - lam (F_99|100 - F_98|99); Q'99 = tau g/4 - lam (FQ_99|100 - FQ_98|99)
    H99 = 1 - lam * (exp["FH_99_100"] - exp["FH_98_99"])
    Q99 = tau0 * g / 4 - lam * (exp["FQ_99_100"] - exp["FQ_98_99"])
    assert rel(H[0, 99], float(H99)) < 1e-14 and rel(Qx[0, 99], float(Q99)) < 1e-14
    changed = np.nonzero((H[0] != h[0]) | (Qx[0] != 0.0))[0]
    assert list(changed) == [98, 99, 100]
    assert np.all(Qy == 0.0) and np.all(bn == 0.0)
    for j in range(1, 4):
        assert np.array_equal(H[j], H[0]) and np.array_equal(Qx[j], Qx[0])
    st, dt, lim = o.step(1)
    assert rel(dt[0], 0.0796646204805423) < 1e-13 and lim[0] == 1


def test_W2_exner_sign_and_walls(orc):
    """Uniform current in a walled channel: Eq.1 erosion at
    the upstream wall and deposition at the downstream wall, tau0 W J / h."""
    K = 0.25
    nx, ny = 8, 3
    o = orc.Oracle(nx, ny, 1.0, orc.Params(K=K, A_J=0.001, C_J=2.0))
    one = np.ones((ny, nx)); z = np.zeros((ny, nx))
    o.set_state(one, one, z, z, 0.4)
    st, dt, lim = o.step(1)
    tau0 = K * min(0.5, 1.0 / (1.0 + math.sqrt(G)), 300.0)
    assert st == 0 and rel(dt[0], tau0) < 1e-15 and lim[0] == 1
    H, Qx, Qy, b = o.get_state()
    db = tau0 * (1 / 0.6) * 0.001
    assert np.all(np.abs(b[:, 0] + db) < 1e-14 * db * 1e3)
    assert np.allclose(b[:, 0], -db, rtol=1e-13, atol=0)
    assert np.allclose(b[:, -1], db, rtol=1e-13, atol=0)
    assert np.all(b[:, 1:-1] == 0.0)
    assert math.fsum((0.6 * b).ravel()) == 0.0
    FJ = o.debug_interior("FJ")
    assert rel(FJ[0, 3], 0.001) < 1e-15


def test_uniform_surface_slope_force(orc):
    """K2/K4: uniform surface slope s on a wet flat patch gives
    Phi_x = -g H s and u~ = -g s tau/2 (closed form)."""
    nx, ny = 16, 5
    s = 1e-3
    x = np.arange(nx, dtype=float)
    h = np.broadcast_to(2.0 + s * x, (ny, nx)).copy()
    z = np.zeros((ny, nx))
    o = orc.Oracle(nx, ny, 1.0, orc.Params())
    o.set_state(h, z, z, z)
    st, dt, _ = o.step(1)
    tau = dt[0]
    phix = o.debug_interior("phix"); ut = o.debug_interior("ut")
    i = 7
    assert rel(phix[2, i], -G * h[2, i] * s) < 1e-12
    assert rel(ut[2, i], -G * s * tau / 2) < 1e-12
    assert np.all(o.debug_interior("phiy") == 0.0)


def test_friction_uniform_flow(orc):
    """Semi-implicit Manning (reading #19): in a uniform current the interior
    momentum after one step is Q/(1 + tau gamma) exactly (closed form)."""
    nx, ny = 24, 5
    n = 0.05
    H0, u0 = 1.5, 0.8
    o = orc.Oracle(nx, ny, 1.0, orc.Params(n_manning=n))
    h = np.full((ny, nx), H0); hu = np.full((ny, nx), H0 * u0); z = np.zeros((ny, nx))
    o.set_state(h, hu, z, z)
    st, dt, _ = o.step(1)
    tau = dt[0]
    gam = G * n * n * u0 / H0 ** (4.0 / 3.0)
    H, Qx, Qy, b = o.get_state()
    assert rel(Qx[2, 12], H0 * u0 / (1 + tau * gam)) < 1e-12
    assert H[2, 12] == H0


def test_slope_term_at_bed_kink(orc):
    """Eq.2 slope term: flat surface, uniform velocity, bed kink at
    column k.  Only the kink cell sees Delta J = -C_J |J0| (s_E - s_W)/h."""
    nx, ny = 20, 3
    k = 10
    s = 0.01
    u0, eta0, A, CJ = 1.0, 2.0, 0.001, 2.0
    x = np.arange(nx, dtype=float)
    bed = np.where(x > k, s * (x - k), 0.0)
    b = np.broadcast_to(bed, (ny, nx)).copy()
    h = eta0 - b
    hu = h * u0
    z = np.zeros((ny, nx))
    o = orc.Oracle(nx, ny, 1.0, orc.Params(A_J=A, C_J=CJ))
    o.set_state(h, hu, z, b, 0.4)
    st, dt, _ = o.step(1)
    tau = dt[0]
    H, Qx, Qy, bn = o.get_state()
    J0 = A * u0 ** 3
    dJ = -(CJ * J0) * (s - 0.0)
    expect = bed[k] - tau * (1 / 0.6) * dJ
    assert rel(bn[1, k], expect) < 1e-12
    for i in (5, 6, 14, 15):
        assert abs(bn[1, i] - bed[i]) <= 1e-15


def test_gate_freezes_bed(orc):
    """Eq.5 gate: with |v| < v_k everywhere the bed does not move;
    above it, it does (invariant)."""
    nx, ny = 12, 4
    one = np.ones((ny, nx)); z = np.zeros((ny, nx))
    b = 0.01 * np.arange(nx, dtype=float)[None, :].repeat(ny, 0)
    for u0, moves in ((0.45, False), (0.6, True)):
        o = orc.Oracle(nx, ny, 1.0, orc.Params(A_J=0.001, C_J=2.0, C_Sh=5.0, d50=1e-3))
        o.set_state(1.0 - b, (1.0 - b) * u0, z, b, 0.4)
        o.step(3)
        bn = o.get_state()[3]
        assert np.array_equal(bn, b) != moves


# -------------------------------------------------------------- invariants

def test_lake_at_rest_dyadic_bitwise(orc):
    """Well-balance: dyadic terrain (C2 recipe), H+b = eta0 exactly; 1000
    steps keep H, b bitwise and Q == 0, islands included."""
    c = synth.config("C2", 96, 80)
    h, hu, hv, b, psi = synth.fill(c)
    assert 0.2 < (h > 0).mean() < 0.9
    o = orc.Oracle(c.nx, c.ny, 1.0, orc.Params(**c.params))
    o.set_state(h, hu, hv, b, psi)
    st, dt, lim = o.step(1000)
    assert st == 0 and len(dt) == 1000
    H, Qx, Qy, bn = o.get_state()
    assert np.array_equal(H, h) and np.array_equal(bn, b)
    assert np.all(Qx == 0.0) and np.all(Qy == 0.0)


def test_lake_at_rest_nondyadic(orc):
    """Well-balance on non-dyadic terrain: max|v| <= 1e-12 m/s after 300 steps."""
    c = synth.config("C2N", 64, 64)
    h, hu, hv, b, psi = synth.fill(c)
    o = orc.Oracle(c.nx, c.ny, 1.0, orc.Params(**c.params))
    o.set_state(h, hu, hv, b, psi)
    st, dt, lim = o.step(300)
    assert st == 0
    H, Qx, Qy, bn = o.get_state()
    wet = H > 1e-3
    v = np.hypot(Qx[wet] / H[wet], Qy[wet] / H[wet])
    assert v.max() <= 1e-12


def test_conservation_water_and_bed(orc):
    """Eq.1/Eq.6 conservative form with walls, sigma = q = 0: sum H and
    sum (1-psi) b are conserved to 1e-13 relative per 100 steps."""
    nx, ny = 48, 40
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=11)
    p = orc.Params(n_manning=0.03, A_J=0.01, C_J=2.0, C_Sh=0.0)
    o = orc.Oracle(nx, ny, 1.0, p)
    assert o.set_state(h, hu, hv, b, psi) == 0
    st, dt, _ = o.step(100)
    assert st == 0
    H, Qx, Qy, bn = o.get_state()
    V0, V1 = math.fsum(h.ravel()), math.fsum(H.ravel())
    B0 = math.fsum(((1 - psi) * b).ravel()); B1 = math.fsum(((1 - psi) * bn).ravel())
    scaleB = math.fsum((np.abs((1 - psi) * b)).ravel())
    assert abs(V1 - V0) / V0 <= 1e-13
    assert abs(B1 - B0) / scaleB <= 1e-13
    assert not np.array_equal(bn, b)  # the bed really moved


def test_wall_faces_carry_no_mass(orc):
    """Mirror ghosts (reading #14): mass, tangential momentum and sediment
    fluxes are exactly 0 on every wall face (mirror symmetry invariant)."""
    nx, ny = 20, 14
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=5)
    o = orc.Oracle(nx, ny, 1.0, orc.Params(n_manning=0.02, A_J=0.01, C_J=2.0))
    o.set_state(h, hu, hv, b, psi)
    o.step(3)
    FH, FQy, FJ = o.debug("FH"), o.debug("FQy"), o.debug("FJ")
    GH, GQx, GJ = o.debug("GH"), o.debug("GQx"), o.debug("GJ")
    g = 3
    for A in (FH, FQy, FJ):
        assert np.all(A[g:g + ny, g] == 0.0) and np.all(A[g:g + ny, g + nx] == 0.0)
    for A in (GH, GQx, GJ):
        assert np.all(A[g, g:g + nx] == 0.0) and np.all(A[g + ny, g:g + nx] == 0.0)


def test_b_frozen_without_transport(orc):
    """A_J = 0 (C1) -> b bitwise constant (Eq.1 with J = q = 0)."""
    nx, ny = 30, 20
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=3)
    o = orc.Oracle(nx, ny, 1.0, orc.Params(n_manning=0.03, A_J=0.0, C_J=2.0))
    o.set_state(h, hu, hv, b, psi)
    st, _, _ = o.step(50)
    assert st == 0
    assert np.array_equal(o.get_state()[3], b)


def test_y_uniformity_C1(orc):
    """C1 (200x4): all 4 rows bitwise identical after 100 steps."""
    c = synth.config("C1")
    h, hu, hv, b, psi = synth.fill(c)
    o = orc.Oracle(c.nx, c.ny, 1.0, orc.Params(**c.params))
    o.set_state(h, hu, hv, b, psi)
    st, dt, _ = o.step(100)
    assert st == 0
    for F in o.get_state():
        for j in range(1, 4):
            assert np.array_equal(F[j], F[0])


def test_mirror_and_transpose_symmetry(orc):
    """Flip x (Qx negated) mirrors the output; transposing x<->y (Qx<->Qy)
    transposes it -- bitwise (catches a swapped index or sign)."""
    nx, ny = 22, 17
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=9)
    p = orc.Params(n_manning=0.03, A_J=0.01, C_J=2.0, C_Sh=4.0, d50=1e-3)
    base, dt0, _, st = orc.run(nx, ny, 1.0, p, h, hu, hv, b, psi, nsteps=20)
    assert st == 0
    fl, dt1, _, _ = orc.run(nx, ny, 1.0, p, h[:, ::-1], -hu[:, ::-1], hv[:, ::-1], b[:, ::-1], psi[:, ::-1], nsteps=20)
    assert np.array_equal(dt0, dt1)
    for k, (A, B) in enumerate(zip(base, fl)):
        sgn = -1.0 if k == 1 else 1.0
        assert np.array_equal(A, sgn * B[:, ::-1])
    tr, dt2, _, _ = orc.run(ny, nx, 1.0, p, h.T, hv.T, hu.T, b.T, psi.T, nsteps=20)
    assert np.array_equal(dt0, dt2)
    assert np.array_equal(base[0], tr[0].T) and np.array_equal(base[3], tr[3].T)
    assert np.array_equal(base[1], tr[2].T) and np.array_equal(base[2], tr[1].T)


def test_particle_confinement(orc):
    """Eq.7's factor 2: a particle moves at most h/2 per step, |tau u~| <= h/2."""
    c = synth.config("C3", 96)
    h, hu, hv, b, psi = synth.fill(c)
    o = orc.Oracle(c.nx, c.ny, 1.0, orc.Params(**c.params))
    o.set_state(h, hu, hv, b, psi)
    for _ in range(40):
        st, dt, _ = o.step(1)
        assert st == 0
        ut, vt = o.debug_interior("ut"), o.debug_interior("vt")
        assert np.max(np.abs(ut)) * dt[0] <= 0.5 and np.max(np.abs(vt)) * dt[0] <= 0.5


def test_checkpoint_resume_bitwise(orc):
    """get_state/set_state is a bit-exact checkpoint: 30+30 steps == 60 steps."""
    nx, ny = 26, 19
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=21)
    p = orc.Params(n_manning=0.03, A_J=0.01, C_J=2.0)
    full, dtf, _, _ = orc.run(nx, ny, 1.0, p, h, hu, hv, b, psi, nsteps=60)
    o = orc.Oracle(nx, ny, 1.0, p)
    o.set_state(h, hu, hv, b, psi)
    _, d1, _ = o.step(30)
    mid = o.get_state()
    o2 = orc.Oracle(nx, ny, 1.0, p)
    o2.set_state(*mid, psi)
    _, d2, _ = o2.step(30)
    assert np.array_equal(np.concatenate([d1, d2]), dtf)
    for A, B in zip(full, o2.get_state()):
        assert np.array_equal(A, B)


def test_given_ghost_window_matches_full_domain(orc):
    """A window with its 3 ghost layers supplied (not mirrored) reproduces the
    full-domain step on its interior: R has stencil radius 3."""
    nx, ny = 40, 36
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=4)
    p = orc.Params(n_manning=0.03, A_J=0.01, C_J=2.0, C_Sh=4.0, d50=1e-3)
    o = orc.Oracle(nx, ny, 1.0, p)
    o.set_state(h, hu, hv, b, psi)
    M = o.reduce_M()
    st, tau, _ = o.tau_from_M(M)
    Hp, Qxp, Qyp, bp = o.get_state_padded()
    Wp = o.debug("W")
    o.step_tau(tau)
    ref = o.get_state()
    x0, y0, wx, wy = 11, 9, 17, 13
    sl = (slice(y0, y0 + wy + 6), slice(x0, x0 + wx + 6))  # padded coords
    w = orc.Oracle(wx, wy, 1.0, p)
    w.set_walls(False, False, False, False)
    w.set_state_padded(Hp[sl], Qxp[sl], Qyp[sl], bp[sl], Wp[sl])
    assert w.step_tau(tau) == 0
    for A, B in zip(ref, w.get_state()):
        assert np.array_equal(A[y0:y0 + wy, x0:x0 + wx], B)


def test_negative_depth_flag(orc):
    """Positivity guard (reading #27): an over-large step drives H
    below -neg_tol and the status is ENEGDEPTH with the state kept."""
    nx, ny = 10, 3
    h = np.zeros((ny, nx)); h[:, :5] = 1.0
    hu = np.zeros((ny, nx)); hu[:, 4] = 5.0
    z = np.zeros((ny, nx))
    o = orc.Oracle(nx, ny, 1.0, orc.Params())
    o.set_state(h, hu, z, z)
    assert o.step_tau(2.0) == orc.ENEGDEPTH


# ------------------------------------------------------- analytic solutions

def _run_to(orc, o, T):
    t = 0.0
    while t < T:
        st, tau, _ = o.tau_from_M(o.reduce_M())
        assert st == 0
        tau = min(tau, T - t)
        assert o.step_tau(tau) == 0
        t += tau


def _ritter_err(orc, nx, T=12.0):
    H0, L, x0 = 1.0, 200.0, 100.0
    dx = L / nx
    x = (np.arange(nx) + 0.5) * dx
    h = np.where(x < x0, H0, 0.0)[None, :].repeat(4, 0)
    z = np.zeros_like(h)
    o = orc.Oracle(nx, 4, dx, orc.Params(K=0.25))
    o.set_state(h, z, z, z, 0.4)
    _run_to(orc, o, T)
    H = o.get_state()[0]
    c0 = math.sqrt(G * H0)
    xs = (np.arange(nx * 16) + 0.5) * dx / 16
    xi = (xs - x0) / T
    he = np.where(xi <= -c0, H0, np.where(xi < 2 * c0, (2 * c0 - xi) ** 2 / (9 * G), 0.0))
    he = he.reshape(nx, 16).mean(1)
    return np.abs(H[0] - he).sum() / he.sum(), H


def test_ritter_dry_dam_break(orc):
    """Ritter (1892) dry-bed dam break: L1 <= 2e-2 at 200 cells, observed
    order >= 0.8 over 200/400 cells, no overshoot above H0."""
    e200, H = _ritter_err(orc, 200)
    e400, _ = _ritter_err(orc, 400)
    assert e200 <= 2e-2
    assert math.log2(e200 / e400) >= 0.8
    assert H.max() <= 1.0 * (1 + 1e-3)


def test_stoker_wet_dam_break(orc):
    """Stoker wet dam break H_L = 1, H_R = 0.1: plateau h_m = 0.3961748 within 1 %."""
    nx, L, x0, T = 400, 200.0, 100.0, 10.0
    dx = L / nx
    x = (np.arange(nx) + 0.5) * dx
    h = np.where(x < x0, 1.0, 0.1)[None, :].repeat(4, 0)
    z = np.zeros_like(h)
    o = orc.Oracle(nx, 4, dx, orc.Params(K=0.25))
    o.set_state(h, z, z, z, 0.4)
    _run_to(orc, o, T)
    H = o.get_state()[0][0]
    hm, um, s = 0.3961748, 2.3213550, 3.1051337
    xi = (x - x0) / T
    sel = (xi > um - math.sqrt(G * hm) + 0.3) & (xi < s - 0.3)
    assert abs(H[sel].mean() - hm) / hm < 1e-2


def test_seiche_second_order(orc):
    """Linear seiche eta = H0 + a cos(pi x / L) cos(omega t): R is second
    order for smooth linear flow (observed order >= 1.8 against the exact
    cell averages)."""
    H0, Lx, T = 1.0, 100.0, 10.0
    errs = []
    for nx in (50, 100, 200):
        dx = Lx / nx
        x = (np.arange(nx) + 0.5) * dx
        a = 1e-4
        h = (H0 + a * np.cos(math.pi * x / Lx))[None, :].repeat(4, 0)
        z = np.zeros_like(h)
        o = orc.Oracle(nx, 4, dx, orc.Params(K=0.25))
        o.set_state(h, z, z, z, 0.4)
        _run_to(orc, o, T)
        om = math.pi / Lx * math.sqrt(G * H0)
        ex = H0 + a * (np.sin(math.pi * (x + dx / 2) / Lx) - np.sin(math.pi * (x - dx / 2) / Lx)) \
            / (math.pi * dx / Lx) * math.cos(om * T)
        errs.append(np.abs(o.get_state()[0][0] - ex).mean())
    assert math.log2(errs[0] / errs[1]) >= 1.8 and math.log2(errs[1] / errs[2]) >= 1.8


def test_positivity_on_dam_configs(orc):
    """Eq.7 at K = 0.25 keeps H >= -neg_tol on the C3/C4 recipes (200 steps)."""
    for name in ("C3", "C4"):
        c = synth.config(name, 64)
        h, hu, hv, b, psi = synth.fill(c)
        o = orc.Oracle(c.nx, c.ny, 1.0, orc.Params(**c.params))
        o.set_state(h, hu, hv, b, psi)
        st, dt, _ = o.step(200)
        assert st == 0 and len(dt) == 200


def test_eq7_bed_diffusion_limits(orc):
    """Eq.7 third term: with a large A_J the bed-diffusion bound
    h^2/(2D), D = max|J0|/(1-psi), sets tau (closed form, limiter 2)."""
    H, u, K, A, psi = 1.0, 0.5, 0.5, 10.0, 0.4
    M, (st, tau, lim) = _single_cell_tau(orc, H, u, 0.0, K, A, psi)
    D = A * u ** 3 / (1 - psi)
    assert st == 0 and lim == 2
    assert rel(tau, K * 1.0 / (2 * D)) < 1e-15


def test_wet_threshold_is_strict(orc):
    """K1's wet test is strict, w = H > eps (P:188 listing `H > Eps`; SURVEY 8(c.1) step 1,
    reading #15): a grid whose every cell holds exactly eps of water is all dry -- no
    Eq.7 term, so EDRY without a cap -- and a cell at eps beside a wet one is a dry cell
    (no velocity, no force) while a cell at the next double above eps is wet."""
    eps = 1e-6
    o = orc.Oracle(4, 3, 1.0, orc.Params(eps_dry=eps))
    e = np.full((3, 4), eps)
    assert o.set_state(e, 0.5 * e, 0 * e, 0 * e) == 0
    assert np.all(o.reduce_M() == 0.0)
    st, _, _ = o.step(1)
    assert st == orc.EDRY
    up = np.nextafter(eps, 1.0)
    o = orc.Oracle(4, 3, 1.0, orc.Params(eps_dry=eps))
    h = np.full((3, 4), eps); h[1, 2] = up
    assert o.set_state(h, 0 * h, 0 * h, 0 * h) == 0
    M = o.reduce_M()
    assert M[1] == math.sqrt(G * up)  # only the cell above eps counts (|v| = 0)
    o.step(1)
    w = o.debug_interior("w")
    assert w[1, 2] == 1.0 and np.sum(w) == 1.0


def test_dry_cells_hold_no_momentum(orc):
    """Type invariant (reading #28): after every step, H <= eps implies
    hu = hv = +0 exactly, including cells that just dried."""
    nx, ny = 40, 32
    h, hu, hv, b, psi = synth.random_state(nx, ny, seed=17, wet_frac=0.5, vel=2.0, film=0.3)
    o = orc.Oracle(nx, ny, 1.0, orc.Params(n_manning=0.02))
    o.set_state(h, hu, hv, b, psi)
    dried = 0
    prev = h
    for _ in range(30):
        st, _, _ = o.step(1)
        assert st == 0
        H, Qx, Qy, _ = o.get_state()
        dry = H <= 1e-6
        assert np.all(Qx[dry] == 0.0) and np.all(Qy[dry] == 0.0)
        dried += int(np.sum(dry & (prev > 1e-6)))
        prev = H
    assert dried > 0  # the case really occurs


def test_ledge_force_is_hydrostatic(orc):
    """K2 face force at a bed step (hydrostatic reconstruction):
    water on a ledge (b=1, H=0.2) above a lower pool (b=0, H=0.5) is pushed
    over the edge by its own pressure g H^2/2 only, not by the drop height:
    Phi_x = g 0.2^2/(4h) on both cells of the step face, 0 elsewhere."""
    nx, ny, k = 12, 3, 6
    x = np.arange(nx)
    b = np.where(x < k, 1.0, 0.0)[None, :].repeat(ny, 0)
    h = np.where(x < k, 0.2, 0.5)[None, :].repeat(ny, 0)
    z = np.zeros((ny, nx))
    o = orc.Oracle(nx, ny, 1.0, orc.Params())
    o.set_state(h, z, z, b)
    o.step(1)
    phix = o.debug_interior("phix")
    f = G * 0.2 ** 2 / 4.0
    assert rel(phix[1, k - 1], f) < 1e-14 and rel(phix[1, k], f) < 1e-14
    other = np.delete(phix[1], [k - 1, k])
    assert np.all(other == 0.0)
    assert np.all(o.debug_interior("phiy") == 0.0)


def test_film_cutoff_reading31(orc):
    """Reading #31: bedload needs a water column deeper than the grain.
    A uniform 2 m/s current over a sloping bed between walls (Shamov gate off, so Eq.3 alone
    decides): with H = d50/2 the bed does not move and Eq.7's bed term is absent (M3 = 0);
    with H = 4 d50 the wall ends erode/deposit and M3 = A_J |v|^3 / (1 - psi)."""
    d50, A, psi = 1e-3, 1e-3, 0.4
    assert orc.bed_mobile(2 * d50, d50) and not orc.bed_mobile(d50, d50)
    nx, ny = 16, 3
    x = np.arange(nx)
    b = (0.01 * (nx - x))[None, :].repeat(ny, 0).astype(float)
    for Hd, moves in ((0.5 * d50, False), (4 * d50, True)):
        h = np.full((ny, nx), Hd)
        hu = 2.0 * h
        z = np.zeros((ny, nx))
        p = orc.Params(A_J=A, C_J=2.0, C_Sh=0.0, d50=d50, eps_dry=1e-6)
        o = orc.Oracle(nx, ny, 1.0, p)
        assert o.set_state(h, hu, z, b, np.full((ny, nx), psi)) == 0
        M = o.reduce_M()
        if moves:
            assert rel(M[2], A * 8.0 / (1 - psi)) < 1e-14
        else:
            assert M[2] == 0.0
        st, _, _ = o.step(1)
        assert st == 0
        moved = np.any(o.get_state()[3] != b)
        assert moved == moves
    # h_bed_min (csph_params / orc_params): an explicit cut-off depth, and 0 = the literal
    # Eq.5 under which the same film carries bedload
    for hb, moves in ((0.25 * d50, True), (0.0, True), (0.75 * d50, False)):
        h = np.full((ny, nx), 0.5 * d50)
        z = np.zeros((ny, nx))
        p = orc.Params(A_J=A, C_J=2.0, C_Sh=0.0, d50=d50, eps_dry=1e-6, h_bed_min=hb)
        o = orc.Oracle(nx, ny, 1.0, p)
        assert o.set_state(h, 2.0 * h, z, b, np.full((ny, nx), psi)) == 0
        assert (o.reduce_M()[2] > 0.0) == moves
        assert o.step(1)[0] == 0
        assert np.any(o.get_state()[3] != b) == moves
