"""GPU parity: the CUDA path (through the C-ABI) vs the CPU oracle on the same
seeded inputs.  Bar (north_star): err_F <= 1e-9 after 100
fp64 steps, identical step count, bitwise-identical dt sequence.  Under the
arithmetic contract the fields are in fact bitwise equal,
which is asserted as well."""
import math
import os

import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
G = 9.81
PATHS = {"fused": 0, "staged": 1}


@pytest.fixture(scope="module")
def cs():
    from paper_2103_15196_b200 import build, csph
    build.build()
    return csph


def parity_err(gpu, ref):
    h, hu, hv, b = ref
    sh = np.max(np.abs(h))
    sq = max(np.max(np.abs(hu)), np.max(np.abs(hv)), sh * math.sqrt(G * sh))
    sb = max(np.max(np.abs(b)), sh)
    scales = [sh, sq, sq, sb]
    return [float(np.max(np.abs(g - r)) / s) for g, r, s in zip(gpu, ref, scales)]


def run_both(cs, c, steps, path, fields=None):
    h, hu, hv, b, psi = fields if fields is not None else synth.fill(c)
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    assert ref.set_state(h, hu, hv, b, psi) == 0
    st_ref, dt_ref, lim_ref = ref.step(steps)
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, path=PATHS[path]))
    g.set_state(h, hu, hv, b, psi)
    st = g.step(steps, check=False)
    dt, lim = g.get_dt_log(steps)
    out = g.get_state()
    tg = g.get_time()
    g.destroy()
    return (st, dt, lim, out, tg), (st_ref, dt_ref, lim_ref, ref.get_state(), ref.time())


def assert_parity(gpu, ref, tol=1e-9, bitwise=True):
    st, dt, lim, out, tg = gpu
    st_r, dt_r, lim_r, out_r, tr = ref
    assert st == st_r
    assert len(dt) == len(dt_r) and np.array_equal(dt, dt_r), "dt sequence differs"
    assert np.array_equal(lim, lim_r)
    errs = parity_err(out, out_r)
    assert max(errs) <= tol, errs
    assert tg[1] == tr[1] and tg[0] == tr[0] and tg[2] == tr[2]  # steps, time = sum of tau, last tau
    if bitwise:
        for a, r in zip(out, out_r):
            assert np.array_equal(a, r)


@pytest.mark.parametrize("path", list(PATHS))
def test_C1_dam_break_100_steps(cs, path):
    c = synth.config("C1")
    gpu, ref = run_both(cs, c, 100, path)
    assert_parity(gpu, ref)


@pytest.mark.parametrize("path", list(PATHS))
def test_C2_lake_at_rest_100_steps(cs, path):
    c = synth.config("C2", 256)
    gpu, ref = run_both(cs, c, 100, path)
    assert_parity(gpu, ref)
    h, hu, hv, b, psi = synth.fill(c)
    assert np.array_equal(gpu[3][0], h) and np.all(gpu[3][1] == 0.0)


@pytest.mark.parametrize("path", list(PATHS))
@pytest.mark.parametrize("name,n,ny", [("C3", 256, 200), ("C4", 192, 256), ("C5", 300, 260)])
def test_dam_and_flood_configs_100_steps(cs, path, name, n, ny):
    """Several tiles and ragged tails (sizes not multiples of the tile)."""
    c = synth.config(name, n, ny)
    gpu, ref = run_both(cs, c, 100, path)
    assert_parity(gpu, ref)


@pytest.mark.parametrize("path", list(PATHS))
def test_random_wet_dry_films(cs, path):
    """Thin films, random currents, heterogeneous psi, all physics on."""
    c = synth.Config("rand", 0, 131, 77, params=dict(n_manning=0.03, A_J=0.01, C_J=2.0,
                                                    C_Sh=4.0, d50=1e-3))
    f = synth.random_state(c.nx, c.ny, seed=5, wet_frac=0.6, vel=1.0, film=0.2)
    gpu, ref = run_both(cs, c, 60, path, fields=f)
    assert_parity(gpu, ref)


@pytest.mark.parametrize("path", list(PATHS))
def test_minimum_grid_3x3(cs, path):
    c = synth.Config("tiny", 0, 3, 3, params={})
    h = np.array([[1.0, 0.5, 0.0], [0.2, 0.0, 0.0], [1.0, 1.0, 1.0]])
    z = np.zeros((3, 3))
    gpu, ref = run_both(cs, c, 10, path, fields=(h, z, z, z, np.full((3, 3), 0.4)))
    assert_parity(gpu, ref)


@pytest.mark.parametrize("path", list(PATHS))
def test_all_dry_is_EDRY(cs, path):
    z = np.zeros((8, 8))
    g = cs.csph_create(8, 8, 1.0, cs.csph_default_params(path=PATHS[path]))
    g.set_state(z, z, z, z, None)
    assert g.step(1, check=False) == cs.CSPH_EDRY
    assert g.get_time()[1] == 0


def test_input_validation(cs):
    g = cs.csph_create(8, 8, 1.0)
    z = np.zeros((8, 8))
    bad = z.copy(); bad[2, 3] = np.nan
    with pytest.raises(cs.CsphError) as e:
        g.set_state(bad, z, z, z)
    assert e.value.code == cs.CSPH_EINVAL
    with pytest.raises(cs.CsphError):
        g.set_state(z - 1.0, z, z, z)
    with pytest.raises(cs.CsphError):
        g.set_state(z, z, z, z, np.full((8, 8), 1.0))
    with pytest.raises(cs.CsphError) as e:
        cs.csph_create(8, 8, 1.0).step(1)
    assert e.value.code == cs.CSPH_ENOSTATE


def test_checkpoint_resume_bitwise(cs):
    c = synth.config("C3", 128)
    h, hu, hv, b, psi = synth.fill(c)
    p = cs.params_from(c.params)
    a = cs.csph_create(c.nx, c.ny, 1.0, p)
    a.set_state(h, hu, hv, b, psi)
    a.step(40)
    full = a.get_state()
    x = cs.csph_create(c.nx, c.ny, 1.0, p)
    x.set_state(h, hu, hv, b, psi)
    x.step(25)
    mid = x.get_state()
    y = cs.csph_create(c.nx, c.ny, 1.0, p)
    y.set_state(*mid, psi)
    y.step(15)
    for u, v in zip(full, y.get_state()):
        assert np.array_equal(u, v)


def test_staged_and_fused_agree_on_dt_and_state(cs):
    c = synth.config("C5", 512)
    h, hu, hv, b, psi = synth.fill(c)
    outs = []
    for path in PATHS.values():
        g = cs.csph_create(c.nx, c.ny, 1.0, cs.params_from(c.params, path=path))
        g.set_state(h, hu, hv, b, psi)
        g.step(30)
        outs.append((g.get_dt_log(30)[0], g.get_state()))
    assert np.array_equal(outs[0][0], outs[1][0])
    for u, v in zip(outs[0][1], outs[1][1]):
        assert np.array_equal(u, v)


def test_branch_free_rcp_sqrt_match_ieee(cs):
    """the kernels' branch-free reciprocal and square root are
    bitwise IEEE-correct on 2^28 hashed inputs (exponents -300..300)."""
    assert cs.csph_selftest_math(1 << 28, 7) == 0


@pytest.mark.parametrize("name,n,ny,steps", [("C5", 700, 650, 80), ("C3", 480, 500, 120),
                                             ("C4", 600, 520, 80)])
def test_hgs_tile_skipping_is_exact(cs, name, n, ny, steps):
    """NEXT-1 HGS: skipping tiles whose neighbourhood
    was dry changes nothing -- state and dt log bitwise equal with it off."""
    c = synth.config(name, n, ny)
    f = synth.fill(c)
    res = []
    for hgs in (1, 0):
        g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, hgs=hgs))
        g.set_state(*f)
        g.step(steps)
        res.append((g.get_dt_log(steps)[0], g.get_state()))
        g.destroy()
    assert np.array_equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)


def test_dam_breach_moving_fronts_vs_oracle(cs):
    """C4D (the C4 valley with its dam breached over 1536 m at t = 0): the reservoir floods
    the valley floor, so wet/dry fronts sweep through HGS tiles, the launch order's costs go
    stale every step and fronts cross strip edges -- single grid and 3 pushing strips, 300
    steps, bitwise the CPU oracle (state and dt log); the wet area grows by > 3 % of the grid."""
    import oracle
    c = synth.config("C4D", 192, 192)
    f = synth.fill(c)
    steps = 300
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    assert ref.set_state(*f) == 0
    st, dt0, lim0 = ref.step(steps)
    assert st == 0
    rs = ref.get_state()
    assert (rs[0] > 1e-6).mean() > (f[0] > 1e-6).mean() + 0.03
    for g in (cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, tile_rows=16)),
              cs.csph_create_multi_rows(c.nx, c.ny, c.dx, cs.params_from(c.params, tile_rows=16),
                                        [0] * 3, [0, 50, 120, 192])):
        g.set_state(*f)
        g.step(steps)
        dt, lim = g.get_dt_log(steps)
        assert np.array_equal(dt, dt0) and np.array_equal(lim, lim0)
        for a, r in zip(g.get_state(), rs):
            assert np.array_equal(a, r)
        g.destroy()


def test_tile_launch_order_is_exact(cs):
    """The launch order: tiles run costliest first, by the previous step's
    costs, through the one-CTA counting sort -- here with more tiles than one sort chunk
    (137 x 183 tiles of 16 rows > 24576), a single grid and 3 strips: bitwise the same
    state and dt log as HGS off (natural order, every tile marched)."""
    c = synth.config("C5", 16384, 2920)
    f = synth.fill(c)
    steps = 6
    res = []
    for hgs, ns in ((0, 1), (1, 1), (1, 3)):
        p = cs.params_from(c.params, hgs=hgs, tile_rows=16)
        if ns == 1:
            g = cs.csph_create(c.nx, c.ny, c.dx, p)
        else:
            g = cs.csph_create_multi(c.nx, c.ny, c.dx, p, [0] * ns)
        g.set_state(*f)
        g.step(steps)
        res.append((g.get_dt_log(steps)[0], g.get_state()))
        g.destroy()
    for r in res[1:]:
        assert np.array_equal(res[0][0], r[0])
        for a, b in zip(res[0][1], r[1]):
            assert np.array_equal(a, b)


def test_hgs_with_bed_source_term(cs):
    """q+ - q- != 0 changes b in dry cells too: HGS must keep copying (never skip)."""
    c = synth.config("C5", 400, 380)
    f = synth.fill(c)
    p = dict(c.params, q_plus=1e-5, q_minus=0.0)
    c2 = synth.Config("C5q", 5, c.nx, c.ny, params=p)
    gpu, ref = run_both(cs, c2, 40, "fused", fields=f)
    assert_parity(gpu, ref)


def _radial_dam(nx, ny, ci, cj, r=9.0):
    """Flat-bed circular dam (C1-style, radius r cells around cell (ci, cj)): the front
    crosses tile edges in every direction and at the corners."""
    jj, ii = np.mgrid[0:ny, 0:nx]
    h = np.where((ii - ci) ** 2 + (jj - cj) ** 2 < r * r, 1.0, 0.0)
    z = np.zeros((ny, nx))
    b = 0.01 * np.sin(0.3 * ii) * np.cos(0.2 * jj)
    return h, z.copy(), z.copy(), b, np.full((ny, nx), 0.4)


@pytest.mark.parametrize("strips", [1, 2, 3])
def test_hgs_band_rule_narrow_tiles(cs, strips):
    """HGS band-mask rule with 16-row tiles, a 1-column last tile column
    (nx = 241 = 2 x 120 + 1) and strips whose last tile has 1-2 rows: a radial front
    crossing tile edges, corners and strip edges must give the HGS-off result bitwise."""
    nx, ny, steps = 241, 131, 150
    f = _radial_dam(nx, ny, 120, 64)
    phys = dict(n_manning=0.03, A_J=1e-3, C_J=2.0, C_Sh=4.0, d50=1e-3)
    res = []
    for hgs in (1, 0):
        p = cs.params_from(phys, hgs=hgs, tile_rows=16)
        g = (cs.csph_create(nx, ny, 1.0, p) if strips == 1
             else cs.csph_create_multi(nx, ny, 1.0, p, [0] * strips))
        g.set_state(*f)
        g.step(steps)
        res.append((g.get_dt_log(steps)[0], g.get_state(), g.tile_stats() if strips == 1 else None))
        g.destroy()
    assert np.array_equal(res[0][0], res[1][0])
    for a, b in zip(res[0][1], res[1][1]):
        assert np.array_equal(a, b)
    if strips == 1:
        assert res[0][2][2] > 0  # tiles were actually skipped


def test_cuda_graph_replay_is_exact(cs):
    """csph_step replays step pairs from CUDA graphs (one per starting buffer parity).
    Odd and even step counts, a re-upload of the state between calls (graph rebuild) and
    both paths: bitwise equal to plain launches (params.graphs = 0) and to the oracle."""
    c = synth.config("C5", 300, 260)
    f = synth.fill(c)
    f2 = synth.fill(synth.config("C3", 300, 260))
    plan = [3, 4, 1, 2]
    for path in (0, 1):
        res = []
        for nog, default_stream in ((False, False), (True, False), (False, True)):
            g = cs.csph_create(c.nx, c.ny, c.dx,
                               cs.params_from(c.params, path=path, graphs=0 if nog else 1))
            if default_stream:  # what bench.py does: torch's (legacy default) stream
                g.set_stream(0)
            g.set_state(*f)
            for n in plan:
                g.step(n)
            a = (g.get_dt_log(sum(plan))[0], g.get_state(), g.last_launch_count())
            g.set_state(*f2)  # rebuilds the graphs (W and the state changed)
            g.step(5)
            res.append((a, g.get_dt_log(5)[0], g.get_state()))
            g.destroy()
        (a0, d0, s0) = res[0]
        for (a1, d1, s1) in res[1:]:
            assert np.array_equal(a0[0], a1[0]) and np.array_equal(d0, d1)
            for x, y in zip(a0[1] + s0, a1[1] + s1):
                assert np.array_equal(x, y)
            assert a0[2] == a1[2]  # kernels launched by the last call (graph or not)
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    ref.set_state(*f)
    st, dt_ref, _ = ref.step(sum(plan))
    assert np.array_equal(dt_ref, a0[0])
    for x, y in zip(ref.get_state(), a0[1]):
        assert np.array_equal(x, y)


def test_tilings_are_bitwise_identical(cs):
    """The CTA tile height (= HGS tile) is a pure performance parameter: the automatic
    state-driven choice and fixed 16..192-row tilings give the same dt log and state."""
    c = synth.config("C3", 700, 600)
    f = synth.fill(c)
    out = []
    for ty in (0, 16, 32, 64, 128, 192):
        g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, tile_rows=ty))
        g.set_state(*f)
        g.step(60)
        out.append((g.get_dt_log(60)[0], g.get_state()))
        g.destroy()
    for dt, st in out[1:]:
        assert np.array_equal(dt, out[0][0])
        for a, b in zip(st, out[0][1]):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("seed", range(int(os.environ.get("CSPH_RAND_SEEDS", "16"))))
def test_randomised_configs_bitwise(cs, seed):
    """Randomised parity net: grid size, terrain/flow config, every physics switch (friction,
    transport, Shamov gate, slope term, Grass exponent, Eq.4 A_J, Exner sources), Courant
    number, dry threshold, open edges, HGS, tile height, path and grid spacing -- status, dt
    log and state bitwise equal to the oracle after 30 steps."""
    rng = np.random.default_rng(1000 + seed)
    nx, ny = int(rng.integers(12, 300)), int(rng.integers(12, 260))
    name = ["C2", "C3", "C4", "C5"][int(rng.integers(0, 4))]
    c = synth.config(name, nx, ny)
    f = synth.fill(c)
    ph = dict(
        n_manning=float(rng.choice([0.0, rng.uniform(0.01, 0.05)])),
        A_J=float(rng.choice([0.0, rng.uniform(1e-4, 3e-3)])),
        C_J=float(rng.uniform(0.0, 3.0)),
        C_Sh=float(rng.choice([0.0, rng.uniform(2.0, 6.0)])),
        d50=float(rng.uniform(5e-4, 2e-3)),
        K=float(rng.uniform(0.1, 0.4)),
        eps_dry=float(rng.choice([1e-6, 1e-4])),
        m_grass=int(rng.choice([2, 2, 0, 1, 3, 4])),
        aj_mode=int(rng.choice([0, 0, 1])),
        q_plus=float(rng.choice([0.0, 0.0, 1e-6])),
        q_minus=float(rng.choice([0.0, 0.0, 5e-7])),
    )
    if ph["aj_mode"] == 1 and ph["n_manning"] == 0.0:
        ph["n_manning"] = 0.02
    open_bc = int(rng.integers(0, 16)) if rng.random() < 0.4 else 0
    walls = [2 if open_bc & m else 1 for m in (1, 2, 4, 8)]
    steps = 30
    # grid spacing: 1 m, or a non-unit h (lambda = tau/h, c_P = g/(4h), Eq.7's h and h^2, the
    # Eq.2 slope) from a generator of its own, so the other draws of a seed are unchanged
    dx = float(np.random.default_rng(5000 + seed).choice([1.0, 0.37, 2.5, 6.1]))
    ref = oracle.Oracle(nx, ny, dx, oracle.Params(**ph))
    ref.set_walls(*walls)
    assert ref.set_state(*f) == 0
    st_ref, dt_ref, lim_ref = ref.step(steps)
    kw = dict(path=int(rng.integers(0, 2)), hgs=int(rng.integers(0, 2)),
              tile_rows=int(rng.choice([0, 16, 40])), open_bc=open_bc)
    g = cs.csph_create(nx, ny, dx, cs.params_from(ph, **kw))
    g.set_state(*f)
    st = g.step(steps, check=False)
    dt, lim = g.get_dt_log(steps)
    out = g.get_state()
    tg = g.get_time()
    g.destroy()
    assert st == st_ref, (ph, kw, st, st_ref)
    assert tg == ref.time(), (tg, ref.time())  # steps done, sum of tau, last tau
    assert np.array_equal(dt, dt_ref) and np.array_equal(lim, lim_ref), (ph, kw)
    for a, r in zip(out, ref.get_state()):
        assert np.array_equal(a, r), (ph, kw, dx)


def _tie_states():
    """Two states whose x-faces have u~_L + u~_R = 0 exactly (the sediment donor tie, reading
    #25; the same constructions as tests/test_oracle_sweep_pins.py): a lake at rest along x
    carrying a flow in y over an x-sloping bed (u~ = +0 on both sides, |J0| averaged with the
    Eq.2 slope term), and a state mirror-symmetric about the face (2|3) with different y-flows
    on the two sides (u~_L = -u~_R, J0x averaged)."""
    ny = 4
    b = np.tile(np.array([0.0, 0.1, 0.25, 0.3, 0.45, 0.5]), (ny, 1))
    h = 1.2 - b
    hv = h * np.tile(np.array([0.5, 0.7, 0.9, 1.1, 0.8, 0.6]), (ny, 1))
    yield 2.5, (h, np.zeros_like(h), hv, b, np.full_like(h, 0.4))
    ny = 3
    rows = [np.array(r) for r in ([0.8, 1.0, 1.1, 1.1, 1.0, 0.8], [0.3, 0.2, 0.1, 0.1, 0.2, 0.3],
                                  [0.1, 0.3, 0.4, -0.4, -0.3, -0.1],
                                  [0.2, 0.3, 0.5, 0.1, 0.0, -0.2])]
    h, b, hu, hv = (np.tile(r, (ny, 1)) for r in rows)
    yield 1.0, (h, hu, hv, b, np.full_like(h, 0.4))


@pytest.mark.parametrize("path", ["fused", "staged"])
def test_sediment_donor_tie_bitwise(cs, path):
    """The donor tie of the sediment face flux on the GPU: 1 and 5 steps bitwise the oracle's
    (the first step ties exactly; a 0.25 average or a wrong side would change b')."""
    ph = dict(A_J=0.01, C_J=2.0, C_Sh=0.0, n_manning=0.0)
    for dx, f in _tie_states():
        ny, nx = f[0].shape
        for steps in (1, 5):
            ref = oracle.Oracle(nx, ny, dx, oracle.Params(**ph))
            assert ref.set_state(*f) == 0
            st, dt0, _ = ref.step(steps)
            assert st == 0
            g = cs.csph_create(nx, ny, dx, cs.params_from(ph, path=PATHS[path]))
            g.set_state(*f)
            g.step(steps)
            assert np.array_equal(g.get_dt_log(steps)[0], dt0)
            for a, r in zip(g.get_state(), ref.get_state()):
                assert np.array_equal(a, r)
            g.destroy()


@pytest.mark.parametrize("case", ["t1=t2", "t2=t3", "t3 at h=2"])
def test_eq7_limiters_on_device(cs, case):
    """Eq.7 ties on the device (reading #25: the lower limiter index wins), with g = 4 so that
    sqrt(gH) is exact: t1 = t2 for a uniform H = 1, u = 2 flow (|u| = c = 2: M1 = 4, M2 = 4,
    h/(2 sqrt M1) = h/M2 = 1/4); t2 = t3 < t1 for still water of depth 4 (c = 4: M2 = 4) beside
    a 1 m deep flow at u = 1 with A_J = 2, psi = 0 (M1 = 1, M3 = A |u|^3 = 2: t2 = t3 = 1/4,
    t1 = 1/2); and the bed term binding on a 2 m grid (H = 1, u = 1, A_J = 10: t1 = 1, t2 = 2/3,
    t3 = h^2/(2 M3) = 4/20).  The device's first tau and limiter equal the oracle's and the
    closed form."""
    n, dx, tau_want = 4, 1.0, 0.25 * 0.25
    if case == "t3 at h=2":
        h = np.ones((n, n)); hu = np.ones((n, n))
        ph = dict(g=4.0, K=0.25, A_J=10.0, C_J=0.0, C_Sh=0.0)
        lim_want, dx, tau_want = 2, 2.0, 0.25 * (4.0 / 20.0)
    elif case == "t1=t2":
        h = np.ones((n, n)); hu = 2.0 * h
        ph = dict(g=4.0, K=0.25, A_J=0.0)
        lim_want = 0
    else:
        h = np.ones((n, n)); h[:, : n // 2] = 4.0
        hu = np.zeros((n, n)); hu[:, n // 2:] = 1.0
        ph = dict(g=4.0, K=0.25, A_J=2.0, C_J=0.0, C_Sh=0.0)
        lim_want = 1
    f = (h, hu, np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n)))
    ref = oracle.Oracle(n, n, dx, oracle.Params(**ph))
    assert ref.set_state(*f) == 0
    st, dt0, lim0 = ref.step(1)
    assert st == 0 and lim0[0] == lim_want and dt0[0] == tau_want
    for path in (0, 1):
        g = cs.csph_create(n, n, dx, cs.params_from(ph, path=path))
        g.set_state(*f)
        g.step(1)
        dt, lim = g.get_dt_log(1)
        assert dt[0] == dt0[0] and lim[0] == lim_want, (path, dt, lim)
        g.destroy()
