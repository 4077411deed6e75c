"""Pins added for the survivors of the systematic oracle mutation sweep
(tools/mutate_oracle_sweep.py, profiles/r02_oracle_sweep.txt): every mutant that is not a
threshold-equivalent boundary change now fails one of these.

  * Eq.7 with h != 1 and its limiter ties (reading #25: ties to the lower index);
  * the sediment donor tie (reading #25: u~_L + u~_R = 0 exactly -> the average of the two
    sides' J0 and |J0|), with the Eq.2 slope term at h != 1;
  * Eq.1's q+ - q- bed source in closed form;
  * Eq.3 with a real exponent m = 0 (|v|^0 = 1), which must not fall back to m_grass;
  * the pinned pow on subnormal arguments; the binary32 oracle's x^(-1/3);
  * Eq.5's "exceeds" at equality; HLL's S_L >= 0 -> F_L at S_L = 0 (reading #25)."""
import math

import mpmath as mp
import numpy as np
import pytest

import oracle

G = 9.81
GH = oracle.GHOST


def test_eq7_t3_uses_h_squared():
    """tau = K min(h/(2 sqrt M1), h/M2, h^2/(2 M3)) (Eq.7) on a 2.5 m grid, the bed term
    limiting: t3 = 6.25 / (2 * 0.5) = 6.25 exactly, tau = 0.25 * 6.25."""
    o = oracle.Oracle(4, 4, 2.5, oracle.Params(K=0.25))
    st, tau, lim = o.tau_from_M([1e-4, 1e-2, 0.5])  # t1 = 125, t2 = 250
    assert st == 0 and lim == 2 and tau == 0.25 * 6.25


@pytest.mark.parametrize("M,lim", [
    ([1.0, 2.0, 0.5], 0),     # h = 2: t1 = 1 = t2 < t3 = 4       -> lower index 0
    ([0.25, 0.5, 1.0], 0),    # t1 = 2 = t3 = 2 < t2 = 4           -> 0   (sqrt(0.25) = 0.5 exact)
    ([0.0625, 1.0, 1.0], 1),  # t1 = 4, t2 = 2 = t3 = 2            -> 1
])
def test_eq7_limiter_ties_go_to_lower_index(M, lim):
    o = oracle.Oracle(4, 4, 2.0, oracle.Params(K=0.5))
    st, tau, l = o.tau_from_M(M)
    assert st == 0 and l == lim
    t = [2.0 / (2 * math.sqrt(M[0])), 2.0 / M[1], 4.0 / (2 * M[2])]
    assert tau == 0.5 * min(t)


def test_eq7_dt_max_tie_keeps_the_eq7_limiter():
    o = oracle.Oracle(4, 4, 2.0, oracle.Params(K=0.5, dt_max=0.5))
    st, tau, l = o.tau_from_M([1.0, 1.0, 1e-9])  # t1 = 1, t2 = 2: K t1 = 0.5 = dt_max
    assert st == 0 and tau == 0.5 and l == 0
    o = oracle.Oracle(4, 4, 2.0, oracle.Params(K=0.5, dt_max=0.25))
    assert o.tau_from_M([1.0, 1.0, 1e-9])[1:] == (0.25, 3)


def _step_debug(nx, ny, dx, prm, h, hu, hv, b, psi=0.4):
    o = oracle.Oracle(nx, ny, dx, oracle.Params(**prm))
    assert o.set_state(h, hu, hv, b, psi) == 0
    st, dt, _ = o.step(1)
    assert st == 0
    return o, dt[0]


def test_sediment_tie_averages_abs_J0_with_slope_term():
    """x-faces of a lake at rest in x (eta constant along x, Qx = 0) carrying a flow in y:
    every x-face has u~_L = u~_R = +0 (the hydrostatic face forces vanish, reading #29), so
    the donor test ties and Eq.2's face flux is J_n = 0.5 (J0x_L + J0x_R) - C_J 0.5 (|J0|_L +
    |J0|_R) (b_R - b_L)/h with J0x = 0 (reading #25), on a 2.5 m grid."""
    nx, ny, dx = 6, 4, 2.5
    b = np.tile(np.array([0.0, 0.1, 0.25, 0.3, 0.45, 0.5]), (ny, 1))
    h = 1.2 - b
    hv = h * np.tile(np.array([0.5, 0.7, 0.9, 1.1, 0.8, 0.6]), (ny, 1))
    prm = dict(A_J=0.01, C_J=2.0, C_Sh=0.0, n_manning=0.0)
    o, tau = _step_debug(nx, ny, dx, prm, h, np.zeros_like(h), hv, b)
    ut = o.debug_interior("ut")
    assert np.all(ut == 0.0)
    Ja = o.debug_interior("J0a")
    FJ = o.debug_interior("FJ")  # FJ[j, i] is the face (i-1 | i)
    for j in range(ny):
        for i in range(1, nx):
            ja = 0.5 * (Ja[j, i - 1] + Ja[j, i])
            want = -(2.0 * ja) * ((b[j, i] - b[j, i - 1]) / dx)
            assert Ja[j, i - 1] != Ja[j, i]
            assert abs(FJ[j, i] - want) <= 1e-15 * abs(want), (j, i, FJ[j, i], want)


def test_sediment_tie_averages_J0n():
    """A state mirror-symmetric about the face (2 | 3) (H, b even; Qx odd; Qy different on the
    two sides, no friction so Qy does not enter u~): u~_L = -u~_R exactly, the donor test ties,
    and J_n = 0.5 (J0x_L + J0x_R) != 0 because |v~| differs (reading #25); b_R = b_L."""
    nx, ny = 6, 3
    hrow = np.array([0.8, 1.0, 1.1, 1.1, 1.0, 0.8])
    brow = np.array([0.3, 0.2, 0.1, 0.1, 0.2, 0.3])
    qrow = np.array([0.1, 0.3, 0.4, -0.4, -0.3, -0.1])
    h, b, hu = (np.tile(r, (ny, 1)) for r in (hrow, brow, qrow))
    hv = np.tile(np.array([0.2, 0.3, 0.5, 0.1, 0.0, -0.2]), (ny, 1))
    prm = dict(A_J=0.01, C_J=2.0, C_Sh=0.0, n_manning=0.0)
    o, _ = _step_debug(nx, ny, 1.0, prm, h, hu, hv, b)
    ut, J0x, FJ = (o.debug_interior(k) for k in ("ut", "J0x", "FJ"))
    for j in range(ny):
        assert ut[j, 2] == -ut[j, 3] and ut[j, 2] != 0.0
        want = 0.5 * (J0x[j, 2] + J0x[j, 3])
        assert want != 0.0 and FJ[j, 3] == want


def test_eq1_bed_source_closed_form():
    """Eq.1 with q+ - q- != 0 on a lake at rest over a flat bed: no flux moves, so
    after n steps b = b0 + sum(tau_k) (q+ - q-) / (1 - psi)."""
    nx, ny, psi = 5, 4, 0.4
    qp, qm = 2e-4, 5e-5
    o = oracle.Oracle(nx, ny, 1.0, oracle.Params(q_plus=qp, q_minus=qm, A_J=0.001))
    h = np.full((ny, nx), 0.7)
    assert o.set_state(h, np.zeros_like(h), np.zeros_like(h), np.full((ny, nx), 0.2), psi) == 0
    st, dt, _ = o.step(5)
    assert st == 0
    db = o.get_state()[3] - 0.2
    want = float(sum(mp.mpf(t) for t in dt) * (mp.mpf(qp) - mp.mpf(qm)) / (1 - mp.mpf(psi)))
    assert np.all(np.abs(db - want) <= 1e-12 * want), (db, want)


def test_grass_real_exponent_zero():
    """Eq.3 with a real exponent m = 0: |v|^0 = 1, J0 = A v~ -- the integer m_grass (3 here)
    must not be used."""
    nx, ny = 5, 4
    rs = np.random.RandomState(7)
    h = rs.uniform(0.5, 1.0, (ny, nx))
    hu, hv = h * rs.uniform(-1, 1, (ny, nx)), h * rs.uniform(-1, 1, (ny, nx))
    A = 0.003
    prm = dict(A_J=A, m_grass=3, m_real=0.0, C_Sh=0.0, h_bed_min=1e-9)
    o, _ = _step_debug(nx, ny, 1.0, prm, h, hu, hv, np.zeros((ny, nx)))
    ut, vt, J0x, J0y, J0a = (o.debug_interior(k) for k in ("ut", "vt", "J0x", "J0y", "J0a"))
    assert np.array_equal(J0x, A * ut) and np.array_equal(J0y, A * vt)
    assert np.array_equal(J0a, A * np.sqrt(ut * ut + vt * vt))


def test_pow_pinned_subnormal_arguments():
    """The pinned x^q on subnormal x (its exponent-extraction branch)."""
    mp.mp.dps = 40
    for x in (4.9e-324, 1e-320, 3.3e-315, 2.2e-310, 2.0e-308):
        for q in (0.5, 1.1, 1.5, 0.25):
            y = oracle.pow_pinned(x, q)
            ref = mp.mpf(x) ** mp.mpf(q)
            if ref < mp.mpf(2) ** -1021:
                continue  # below the pinned pow's range (it returns 0 there)
            assert abs(mp.mpf(y) / ref - 1) < 1e-13, (x, q, y, ref)


def test_binary32_oracle_icbrt():
    """The fp32 mode's x^(-1/3) (binary32 oracle): within 2 binary32 ulps of
    the exact value over the depths R takes it of (1e-6 .. 1e3 m)."""
    L = oracle.lib(32)
    xs = np.float32(np.logspace(-6, 3, 2000))
    for x in xs:
        y = np.float32(L.orc_icbrt(float(x)))
        ref = float(mp.mpf(float(x)) ** (-mp.mpf(1) / 3))
        ulp = float(np.spacing(np.float32(ref)))
        assert abs(float(y) - ref) <= 2 * ulp, (x, y, ref)


def test_shamov_gate_is_strict():
    """Eq.5: bedload when the flow *exceeds* the threshold: s2^3 > kappa H, so at
    equality (s2 = 1, kappa H = 0.5 * 2 = 1) there is none."""
    assert not oracle.shamov_gate(0.5, 1.0, 2.0, 4.0)
    assert oracle.shamov_gate(0.5, 1.0 + 2 ** -40, 2.0, 4.0)


def test_hll_sl_zero_takes_the_left_flux():
    """Reading #25: S_L >= 0 -> F = F(q-) exactly, at S_L = 0 (u = sqrt(g H) on both sides)."""
    seen_diff = False
    for H in (1.0, 0.37, 2.3, 0.9, 0.1507, 0.2055):
        u = math.sqrt(G * H)
        for ut in (0.0, 0.4, -0.7):
            F = oracle.hll_face(G, (H, H, u, ut), (H, H, u, ut))
            m = H * u
            assert F[0] == m and F[1] == m * u and F[2] == m * ut
            SR = u + math.sqrt(G * H)
            seen_diff |= ((SR * m) * (1.0 / SR) != m) or ((SR * (m * u)) * (1.0 / SR) != m * u)
    assert seen_diff


def test_hll_sr_zero_takes_the_right_flux():
    """Reading #25: else S_R <= 0 -> F = F(q+) exactly, at S_R = 0 (u = -sqrt(g H) on both
    sides, so S_L < 0 = S_R)."""
    seen_diff = False
    for H in (1.0, 0.37, 2.3, 0.9, 0.1507, 0.2055):
        u = -math.sqrt(G * H)
        for ut in (0.0, 0.4, -0.7):
            F = oracle.hll_face(G, (H, H, u, ut), (H, H, u, ut))
            m = H * u
            assert F[0] == m and F[1] == m * u and F[2] == m * ut
            SL = u - math.sqrt(G * H)
            # the HLL average at S_R = 0: (-S_L F(q+)) / (0 - S_L)
            seen_diff |= ((-SL * m) * (1.0 / -SL) != m) or ((-SL * (m * u)) * (1.0 / -SL) != m * u)
    assert seen_diff


def test_pow_pinned_range_edges():
    """x^q closed forms at the edges of the pinned pow's range: 0^q = 0 for
    q > 0 (also where q log2 of the scaled zero would stay in range), x^1 = x at the smallest
    and largest binary exponents it returns (2^-1021, 2^1023)."""
    assert oracle.pow_pinned(0.0, 0.5) == 0.0 and oracle.pow_pinned(0.0, 0.1) == 0.0
    for e in (-1021, -1000, 1000, 1023):
        assert oracle.pow_pinned(2.0 ** e, 1.0) == 2.0 ** e
