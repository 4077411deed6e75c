"""Brute-force pin of the oracle: SURVEY.md 8(c.3) "Implementation of R".

The fp64 oracle (oracle/csph_oracle.c) against an independent 50-digit transcription of
DESIGN.md section 3 (tests/brute_r.py) for one and two steps on random 4x3 .. 6x5 grids
with *moving* water: non-zero velocities, wet, dry and film cells, bed steps, a psi
field, friction and bedload on.  With the water moving, H_half != H_n, so these cases
fix the time levels PAPER.md:224-238 assigns to K4-K7: K5's
forces on eta_half at the centre cell too, K7's reconstruction of the n-level H, the
Shamov gate and the film cut-off on the n-level H, and H_half = H_n on dry cells.
Two families place a threshold on purpose between a cell's H_n and H_half (the Shamov
gate via C_Sh, the film cut-off via d50), so that the gate's time level decides the
result.  Random inputs that put any branch of R within 1e-9 (relative) of its threshold
are redrawn: there a correct fp64 evaluation may legitimately branch the other way.

Pass: after each step the dt and limiter agree (tau to 1e-14 relative) and the state
agrees within 1e-13 in the parity metric of DESIGN.md 3.10.
"""
import math

import mpmath as mp
import numpy as np
import pytest

from brute_r import BruteR

G = 9.81
TOL = 1e-13
MARGIN = 1e-9


def _params(**kw):
    p = dict(g=G, K=0.25, eps_dry=1e-6, dt_max=math.inf, neg_tol=1e-12, n_manning=0.03,
             A_J=0.02, m_grass=2, C_J=2.0, C_Sh=4.0, d50=1e-3, q_plus=0.0, q_minus=0.0,
             aj_mode=0, s_rel=2.65, h_bed_min=-1.0, m_real=-1.0)
    p.update(kw)
    return p


def _random_case(seed, films=False, bc=None, fields=False, closures=False, spacing=False):
    """A tiny grid with moving water.  Cells are wet (H in [0.15, 1.2]), dry (H = 0) or,
    with films, thin films 0 < H < eps; velocities up to 1.2 m/s in any direction; the
    bed has steps of up to 0.5 m; psi in [0.3, 0.45]."""
    rs = np.random.RandomState(seed)
    nx, ny = int(rs.randint(4, 7)), int(rs.randint(3, 6))
    kind = rs.choice(3, size=(ny, nx), p=[0.62, 0.2, 0.18])
    eps = 1e-2 if films else 1e-6
    H = np.where(kind == 0, rs.uniform(0.15, 1.2, (ny, nx)), 0.0)
    if films:
        H = np.where(kind == 2, rs.uniform(0.1 * eps, 0.9 * eps, (ny, nx)), H)
    u = rs.uniform(-1.2, 1.2, (ny, nx))
    v = rs.uniform(-1.2, 1.2, (ny, nx))
    wet = H > eps
    Qx = np.where(wet, H * u, 0.0)
    Qy = np.where(wet, H * v, 0.0)
    b = rs.uniform(0.0, 0.5, (ny, nx)) * (rs.uniform(size=(ny, nx)) < 0.7)
    psi = rs.uniform(0.3, 0.45, (ny, nx))
    prm = _params(eps_dry=eps, K=float(rs.uniform(0.12, 0.3)))
    if closures:  # NEXT-4: Eq.4 A_J at the local depth and an odd Grass exponent
        prm.update(aj_mode=1, m_grass=int(rs.choice([1, 3, 4])), d50=2e-4)
        if rs.uniform() < 0.5:  # a real exponent through the pinned pow
            prm.update(m_real=float(rs.uniform(1.2, 3.8)))
    if spacing:  # h != 1 (lambda = tau/h, Eq.7's h and h^2, the Eq.2 slope) and Eq.1's q+/q-
        prm.update(_dx=float(rs.uniform(0.4, 3.0)), q_plus=float(rs.uniform(0.0, 2e-4)),
                   q_minus=float(rs.uniform(0.0, 1e-4)))
    if bc is None:
        bc = (1, 1, 1, 1)
    fl = {}
    if fields:
        fl = dict(n_field=rs.uniform(0.0, 0.05, (ny, nx)) * (rs.uniform(size=(ny, nx)) < 0.8),
                  beta=rs.uniform(0.0, 0.2, (ny, nx)), src=rs.uniform(0.0, 0.01, (ny, nx)))
    return nx, ny, prm, (H, Qx, Qy, b, psi), bc, fl


def _dx(prm):
    """Grid spacing of a case (the "spacing" family draws one != 1; "_dx" is not a param)."""
    return prm.get("_dx", 1.0), {k: v for k, v in prm.items() if k != "_dx"}


def _oracle(orc, nx, ny, prm, st, bc, fl):
    dx, prm = _dx(prm)
    o = orc.Oracle(nx, ny, dx, orc.Params(**prm))
    o.set_walls(*bc)
    assert o.set_state(*st) == 0
    if fl:
        assert o.set_fields(fl["n_field"], fl["beta"], fl["src"]) == 0
    return o


def _brute(nx, ny, prm, st, bc, fl):
    H, Qx, Qy, b, psi = (a.tolist() for a in st)
    kw = {k: v.tolist() for k, v in fl.items()}
    dx, prm = _dx(prm)
    return BruteR(nx, ny, dx, prm, H, Qx, Qy, b, psi, bc=bc, **kw)


def _err(state_o, state_b):
    """DESIGN.md 3.10 parity metric, the brute force as the reference."""
    ref = [np.array([[float(x) for x in row] for row in F]) for F in state_b]
    sh = max(np.max(np.abs(ref[0])), 1e-300)
    sq = max(np.max(np.abs(ref[1])), np.max(np.abs(ref[2])), sh * math.sqrt(G * sh))
    sb = max(np.max(np.abs(ref[3])), sh)
    scales = (sh, sq, sq, sb)
    # differences in 50 digits: the fp64 value is exact as an mpf
    errs = []
    for F, R, s in zip(state_o, state_b, scales):
        d = max(abs(mp.mpf(float(F[j, i])) - R[j][i]) for j in range(F.shape[0])
                for i in range(F.shape[1]))
        errs.append(float(d) / s)
    return errs


def _run_pair(orc, case, nsteps):
    nx, ny, prm, st, bc, fl = case
    o = _oracle(orc, nx, ny, prm, st, bc, fl)
    br = _brute(nx, ny, prm, st, bc, fl)
    out = []
    for _ in range(nsteps):
        stat, dt, lim = o.step(1)
        tau, blim = br.step()
        out.append((stat, dt, lim, tau, blim, _err(o.get_state(), br.state())))
    return br, out


def _accept(br):
    return br.mg.min_rel >= MARGIN


def _check(out):
    for k, (stat, dt, lim, tau, blim, errs) in enumerate(out):
        assert stat == 0, (k, stat)
        assert int(lim[0]) == blim, (k, lim, blim)
        assert abs(dt[0] - float(tau)) <= 1e-14 * float(tau), (k, dt[0], float(tau))
        assert max(errs) <= TOL, (k, errs)


def _cases(kind, n, **kw):
    """Accepted cases of a family: seeds are drawn until n have every branch of R at
    least MARGIN away from its threshold over both steps."""
    got, seed = [], 1000 * (1 + ["moving", "films", "open", "fields", "closures",
                                 "spacing"].index(kind))
    while len(got) < n:
        seed += 1
        case = _random_case(seed, **kw)
        br = _brute(*case[:4], case[4], case[5])
        try:
            br.step(); br.step()
        except ValueError:
            continue
        if _accept(br):
            got.append(case)
    return got


@pytest.mark.parametrize("kind,kw", [
    ("moving", {}),
    ("films", {"films": True}),
    ("open", {"bc": (2, 1, 1, 2)}),
    ("fields", {"fields": True}),
    ("closures", {"closures": True}),
    ("spacing", {"spacing": True}),
])
def test_oracle_matches_bruteforce_R(orc, kind, kw):
    """Two steps of R on random tiny grids with moving water."""
    for case in _cases(kind, 4, **kw):
        br, out = _run_pair(orc, case, 2)
        _check(out)
        # the cases exercise what they claim: water moves, so H_half != H_n somewhere
        assert any(float(x) != 0.0 for row in br.state()[1] for x in row)


def _threshold_case(orc, seed, which):
    """A moving-water case whose Shamov gate (which = 'gate': C_Sh chosen) or film cut-off
    (which = 'film': h_bed_min chosen, no gate) puts the threshold of one wet cell between its
    H_n and H_half, so the time level of H in Eq.5 / reading #31 decides whether that cell
    carries bedload (n-level H)."""
    case = _random_case(seed)
    nx, ny, prm, st, bc, fl = case
    br = _brute(nx, ny, prm, st, bc, fl)
    best = None
    for j in range(ny):
        for i in range(nx):
            H, Hh, ut, vt = br.probe(i, j)
            if H > prm["eps_dry"] and H > 0.3:
                gap = abs(Hh / H - 1)
                if gap > 1e-3 and (best is None or gap > best[0]):
                    best = (gap, H, Hh, ut * ut + vt * vt)
    if best is None:
        return None
    _, H, Hh, s2 = best
    mid = mp.sqrt(H * Hh)
    if which == "gate":
        kappa = s2 ** 3 / mid
        prm = dict(prm, C_Sh=float((kappa / mp.mpf(prm["d50"]) ** 2) ** (mp.mpf(1) / 6)))
    else:
        prm = dict(prm, C_Sh=0.0, h_bed_min=float(mid))
    return nx, ny, prm, st, bc, fl


@pytest.mark.parametrize("which", ["gate", "film"])
def test_time_level_of_the_bedload_gates(orc, which):
    """Eq.5 gate and reading #31's cut-off read the n-level H: with the
    threshold of one cell placed between H_n and H_half, the oracle follows R."""
    done, seed = 0, 7000 if which == "gate" else 8000
    while done < 3:
        seed += 1
        case = _threshold_case(orc, seed, which)
        if case is None:
            continue
        br = _brute(*case[:4], case[4], case[5])
        try:
            br.step(); br.step()
        except ValueError:
            continue
        if not _accept(br):
            continue
        _, out = _run_pair(orc, case, 2)
        _check(out)
        done += 1


def test_W1_two_steps_bruteforce(orc):
    """SURVEY 8(c.3) W1 continued: the C1 dam (H = 1 | 0, flat dry bed, no friction or
    transport) for two steps on a 24 x 3 channel -- the front moves 6 cells in 2 steps,
    so the walls 12 cells away play no part and the cells near the dam are those of the
    200 x 4 C1 grid.  In the second step H_half != H (the water moves)."""
    nx, ny = 24, 3
    H = np.zeros((ny, nx)); H[:, :12] = 1.0
    z = np.zeros((ny, nx))
    prm = _params(n_manning=0.0, A_J=0.0, C_Sh=0.0, C_J=0.0)
    case = (nx, ny, prm, (H, z, z, z, np.full((ny, nx), 0.4)), (1, 1, 1, 1), {})
    br, out = _run_pair(orc, case, 2)
    _check(out)
    # step 1 reproduces the hand-derived W1 values: tau0 = K/sqrt(g)
    assert abs(out[0][1][0] - 0.0798188571017626) < 1e-16
    assert abs(out[1][1][0] - 0.0796646204805423) < 1e-15
