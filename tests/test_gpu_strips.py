"""Row-strip decomposition on one GPU.

csph_create_multi puts several strips on the same device and moves the 3 halo
rows with cudaMemcpyPeerAsync; csph_create_dist with one rank exercises the NCCL
communicator and the allreduce-max of the Eq.7 maxima.  Max is exact and
order-free, so every decomposition must be bitwise equal to the single grid."""
import os

import numpy as np
import pytest

import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cs():
    from paper_2103_15196_b200 import build, csph
    build.build()
    return csph


def single(cs, c, f, steps, path):
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, path=path))
    g.set_state(*f)
    g.step(steps)
    return g.get_dt_log(steps)[0], g.get_state()


@pytest.mark.parametrize("push", [1, 0])
@pytest.mark.parametrize("path", [0, 1])
@pytest.mark.parametrize("nstrips", [2, 3, 5])
def test_multi_strips_bitwise(cs, nstrips, path, push):
    """2-5 strips on one device: halos pushed from inside the step kernel (halo_push = 1,
    fused path) or peer copies (halo_push = 0, and the staged path) -- bitwise the single grid."""
    c = synth.config("C4", 160, 203)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 60, path)
    g = cs.csph_create_multi(c.nx, c.ny, c.dx, cs.params_from(c.params, path=path, halo_push=push),
                             [0] * nstrips)
    g.set_state(*f)
    g.step(60)
    dt, _ = g.get_dt_log(60)
    assert np.array_equal(dt, dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)


def test_multi_strips_set_state_rows(cs):
    """Each strip can be fed from a row window covering its rows + halo."""
    c = synth.config("C5", 144, 150)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 30, 0)
    g = cs.csph_create_multi(c.nx, c.ny, c.dx, cs.params_from(c.params), [0, 0])
    g.set_state_rows(0, c.ny, *f)
    g.step(30)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)


def test_dist_single_rank_nccl(cs):
    """NCCL communicator of one rank: allreduce path, bitwise equal to single."""
    c = synth.config("C3", 128, 96)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 40, 0)
    nid = cs.csph_make_nccl_id()
    g = cs.csph_create_dist(c.nx, c.ny, c.dx, cs.params_from(c.params), 0, 1, 0, nid)
    g.set_state(*f)
    g.step(40)
    dt, _ = g.get_dt_log(40)
    assert np.array_equal(dt, dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)
    g.destroy()


@pytest.mark.parametrize("push", [1, 0])
@pytest.mark.parametrize("path", [0, 1])
def test_uneven_strips_bitwise(cs, path, push):
    """Caller-chosen (load-balanced) strip rows, csph_create_multi_rows: strips of 3, 17,
    150 and 33 rows are bitwise the single grid; bounds from csph_balance_rows too."""
    c = synth.config("C4", 160, 203)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 50, path)
    w = (f[0] > 1e-6).sum(axis=1) + 0.03 * c.nx
    for bounds in ([0, 3, 20, 170, 203], cs.csph_balance_rows(c.ny, 3, w)):
        g = cs.csph_create_multi_rows(c.nx, c.ny, c.dx,
                                      cs.params_from(c.params, path=path, halo_push=push),
                                      [0] * (len(bounds) - 1), bounds)
        g.set_state(*f)
        g.step(50)
        assert np.array_equal(g.get_dt_log(50)[0], dt0)
        for a, r in zip(g.get_state(), ref):
            assert np.array_equal(a, r)
        g.destroy()
    with pytest.raises(cs.CsphError):
        cs.csph_create_multi_rows(c.nx, c.ny, c.dx, cs.params_from(c.params), [0, 0], [0, 2, 203])


def test_dist_ipc_link_single_rank(cs):
    """The DIST halo push's link step (csph_ipc_export / csph_ipc_link) on one
    rank: the blob exports; a rank with no neighbours links nothing and steps whole (sort,
    fused kernel, ctrl per step: no edge split, no halo traffic), bitwise the single grid; a
    blob where no neighbour exists, or one for the wrong rank, is rejected."""
    c = synth.config("C5", 200, 96)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 40, 0)
    g = cs.csph_create_dist_rows(c.nx, c.ny, c.dx, cs.params_from(c.params, tile_rows=16),
                                 0, 1, [0, c.ny], 0, cs.csph_make_nccl_id())
    blob = g.ipc_export()
    assert len(blob) == cs.lib().csph_ipc_blob_bytes() and blob[:4] == b"HPSC"
    g.ipc_link([blob])
    with pytest.raises(cs.CsphError):
        g.ipc_link([blob, blob])  # one rank: one blob
    with pytest.raises(cs.CsphError):
        g.ipc_link([b"\0" * len(blob)])  # not a blob of this handle's geometry
    g.ipc_link(None)
    g.ipc_link([blob])
    g.set_state(*f)
    g.step(40)
    assert np.array_equal(g.get_dt_log(40)[0], dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)
    assert g.last_launch_count() == 40 * 3
    g.destroy()
    m = cs.csph_create_multi(c.nx, c.ny, c.dx, cs.params_from(c.params), [0, 0])
    with pytest.raises(cs.CsphError):
        m.ipc_export()  # DIST only
    m.destroy()


def test_dist_rows_single_rank(cs):
    """csph_create_dist_rows with one rank and bounds [0, ny]."""
    c = synth.config("C3", 128, 96)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 30, 0)
    g = cs.csph_create_dist_rows(c.nx, c.ny, c.dx, cs.params_from(c.params), 0, 1, [0, c.ny], 0,
                                 cs.csph_make_nccl_id())
    g.set_state(*f)
    g.step(30)
    assert np.array_equal(g.get_dt_log(30)[0], dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)
    g.destroy()


@pytest.mark.parametrize("tile_rows", [16, 40, 48, 64])
def test_dist_split_launches(cs, tile_rows):
    """The send/recv multi-GPU step (halo_push = 0: edge tile rows, NCCL halo on the comm
    stream, interior, allreduce) on one rank: 2..6 tile rows, ragged last tile
    row, HGS on -- bitwise the single grid."""
    c = synth.config("C5", 200, 96)
    f = synth.fill(c)
    dt0, ref = single(cs, c, f, 40, 0)
    g = cs.csph_create_dist_rows(c.nx, c.ny, c.dx,
                                 cs.params_from(c.params, tile_rows=tile_rows, halo_push=0),
                                 0, 1, [0, c.ny], 0, cs.csph_make_nccl_id())
    g.set_state(*f)
    g.step(40)
    assert np.array_equal(g.get_dt_log(40)[0], dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)
    # per step: ctrl + the edge tile rows, the interior and its tile-order sort (when there
    # is one); the last launch must hold >= 3 rows (a short last tile is merged with the
    # one before it)
    nty = -(-c.ny // tile_rows)
    hi = (nty - 1) * tile_rows
    if c.ny - hi < 3:
        hi -= tile_rows
    split = nty >= 3 and hi > tile_rows
    assert g.last_launch_count() == 40 * (1 + (4 if split else 1))
    g.destroy()


@pytest.mark.parametrize("up", [False, True])
@pytest.mark.parametrize("push", [1, 0])
@pytest.mark.parametrize("nstrips", [2, 4])
def test_front_crosses_strip_edges_hgs(cs, nstrips, push, up):
    """HGS across strip edges (ghost tile flags): a dam-break front starts
    in the first (up: the last) strip and runs into dry strips whose edge tiles were being
    skipped -- so both ghost-flag rows of a strip (facing the strip below and above) decide;
    with 16-row tiles and uneven strips the result is bitwise the single grid without HGS."""
    nx, ny = 150, 180
    jj, ii = np.mgrid[0:ny, 0:nx]
    if up:
        jj = ny - 1 - jj
    h = np.where(jj < 30, 1.5, 0.0)
    b = 0.4 - 0.002 * jj + 0.01 * np.sin(0.2 * ii)  # downhill, away from the dam
    z = np.zeros((ny, nx))
    f = (h, z.copy(), z.copy(), b, np.full((ny, nx), 0.4))
    phys = dict(n_manning=0.02, A_J=1e-3, C_J=2.0, C_Sh=4.0, d50=1e-3)
    steps = 500
    g = cs.csph_create(nx, ny, 1.0, cs.params_from(phys, hgs=0))
    g.set_state(*f)
    g.step(steps)
    dt0, ref = g.get_dt_log(steps)[0], g.get_state()
    g.destroy()
    bounds = [0, 37, 70, 131, 180] if nstrips == 4 else [0, 41, 180]
    g = cs.csph_create_multi_rows(nx, ny, 1.0, cs.params_from(phys, tile_rows=16, halo_push=push),
                                  [0] * nstrips, bounds)
    g.set_state(*f)
    g.step(steps)
    assert np.array_equal(g.get_dt_log(steps)[0], dt0)
    for a, r in zip(g.get_state(), ref):
        assert np.array_equal(a, r)
    # the front crossed the strip edges at rows 37/41 and 70 (up: 131 and 70)
    assert (ref[0][:104] if up else ref[0][76:]).max() > 0
    g.destroy()


@pytest.mark.parametrize("push", [1, 0])
@pytest.mark.parametrize("tile_rows", [16, 32])
def test_split_strips_short_last_tile_vs_oracle(cs, tile_rows, push):
    """Overlapped multi-strip steps (edge tile rows -> halo on the comm stream || interior,
    DESIGN.md 9) with strips whose last tile row has 1 or 2 rows (ny % ty in {1, 2}): the
    halo rows sent at the edge event must all be final.  Four strips of
    3 * ty + 1, 3 * ty + 2, 4 * ty + 1 rows and the rest, HGS on, compared element by
    element with the CPU oracle (and the dt log bitwise)."""
    import oracle
    c = synth.config("C4", 160, 14 * tile_rows + 7)
    f = synth.fill(c)
    b1 = 3 * tile_rows + 1
    b2 = b1 + 3 * tile_rows + 2
    b3 = b2 + 4 * tile_rows + 1
    bounds = [0, b1, b2, b3, c.ny]
    steps = 60
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    assert ref.set_state(*f) == 0
    st, dt0, lim0 = ref.step(steps)
    assert st == 0
    g = cs.csph_create_multi_rows(c.nx, c.ny, c.dx,
                                  cs.params_from(c.params, tile_rows=tile_rows, halo_push=push),
                                  [0] * 4, bounds)
    g.set_state(*f)
    g.step(steps)
    dt, lim = g.get_dt_log(steps)
    assert np.array_equal(dt, dt0) and np.array_equal(lim, lim0)
    for a, r in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(a, r)
    g.destroy()


@pytest.mark.parametrize("path", [0, 1])
def test_negative_depth_stops_every_strip(cs, path):
    """CSPH_ENEGDEPTH (reading #27) on the device: with K = 0.95 (beyond the
    unsplit scheme's positivity bound, reading #13) a random moving state drives a depth
    below -neg_tol at step 4.  Like the oracle, the GPU returns ENEGDEPTH after exactly that
    step with its state kept (bitwise the oracle's), and later calls neither advance nor
    clear the error.  The flag is combined across strips with the Eq.7 maxima:
    on 3 strips every strip stops after the same step."""
    import oracle
    nx, ny = 48, 40
    f = synth.random_state(nx, ny, seed=35, wet_frac=0.6, vel=4.0)
    prm = dict(K=0.95)
    ref = oracle.Oracle(nx, ny, 1.0, oracle.Params(**prm))
    ref.set_state(*f)
    st, dt0, _ = ref.step(20)
    assert st == oracle.ENEGDEPTH and len(dt0) == 4
    for g in (cs.csph_create(nx, ny, 1.0, cs.params_from(prm, path=path)),
              cs.csph_create_multi_rows(nx, ny, 1.0, cs.params_from(prm, path=path), [0] * 3,
                                        [0, 13, 27, ny])):
        g.set_state(*f)
        with pytest.raises(cs.CsphError) as e:
            g.step(20)
        assert e.value.code == cs.CSPH_ENEGDEPTH
        assert g.get_time()[1] == 4
        assert np.array_equal(g.get_dt_log(20)[0], dt0)
        for a, r in zip(g.get_state(), ref.get_state()):
            assert np.array_equal(a, r)
        assert g.step(3, check=False) == cs.CSPH_ENEGDEPTH
        assert g.get_time()[1] == 4
        g.destroy()


def test_nonfinite_maxima(cs):
    """CSPH_ENONFINITE: finite inputs whose Eq.7 term overflows (|v| = 1e200,
    s2 = inf) stop the first step, as in the oracle; nothing advances."""
    import oracle
    nx, ny = 8, 6
    h = np.ones((ny, nx)); hu = np.zeros((ny, nx)); hu[2, 3] = 1e200
    z = np.zeros((ny, nx))
    ref = oracle.Oracle(nx, ny, 1.0, oracle.Params())
    ref.set_state(h, hu, z, z)
    assert ref.step(1)[0] == oracle.ENONFINITE
    g = cs.csph_create(nx, ny, 1.0, cs.params_from({}))
    g.set_state(h, hu, z, z)
    assert g.step(2, check=False) == cs.CSPH_ENONFINITE
    assert g.get_time()[1] == 0
    for a, r in zip(g.get_state(), (h, hu, z, z)):
        assert np.array_equal(a, r)
    g.destroy()


@pytest.mark.parametrize("fields", [False, True])
def test_rebalance_multi_bitwise(cs, fields):
    """Re-partitioning during a run (csph_row_weights -> csph_balance_rows ->
    csph_rebalance_rows): 3 strips start on an even split, are re-balanced on the
    wet cells of the current state after 40 steps (state, psi field and NEXT-3 fields migrate;
    time, tau and dt log carry over), and step on -- bitwise the single grid, dt log included.
    With `fields`: n_M / beta / source fields, open edges, 16-row tiles."""
    c = synth.config("C5", 200, 183)
    f = synth.fill(c)
    prm = dict(c.params)
    kw = {}
    fl = None
    if fields:
        rng = np.random.default_rng(4)
        fl = dict(n_manning=0.02 + 0.02 * rng.random((c.ny, c.nx)),
                  beta=np.full((c.ny, c.nx), 1e-4), src=np.where(rng.random((c.ny, c.nx)) < 0.01, 1e-3, 0.0))
        prm.update(open_bc=5)
        kw = dict(tile_rows=16)
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(prm, **kw))
    g.set_state(*f)
    if fl:
        g.set_fields(**fl)
    g.step(100)
    dt0, ref = g.get_dt_log(100)[0], g.get_state()
    g.destroy()
    m = cs.csph_create_multi(c.nx, c.ny, c.dx, cs.params_from(prm, **kw), [0, 0, 0])
    m.set_state(*f)
    if fl:
        m.set_fields(**fl)
    m.step(40)
    w = m.row_weights()
    wet = (m.get_state()[0] > 1e-6).sum(axis=1) + 0.03 * c.nx
    assert np.array_equal(w, wet)
    bounds = cs.csph_balance_rows(c.ny, 3, w)
    assert bounds != [0, 61, 122, 183]
    m.rebalance_rows(bounds)
    assert m.get_time()[1] == 40
    m.step(60)
    assert np.array_equal(m.get_dt_log(100)[0], dt0)
    for a, r in zip(m.get_state(), ref):
        assert np.array_equal(a, r)
    # and back to an uneven split with a short last tile
    m.rebalance_rows([0, 3, 100, 183])
    m.destroy()


def test_rebalance_dist_single_rank(cs):
    """csph_rebalance_rows on a 1-rank NCCL handle (the DIST migration code path: a rank's rows
    to itself), mid-run, graphs on: bitwise the uninterrupted run."""
    c = synth.config("C3", 150, 130)
    f = synth.fill(c)
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params))
    g.set_state(*f)
    g.step(50)
    dt0, ref = g.get_dt_log(50)[0], g.get_state()
    g.destroy()
    d = cs.csph_create_dist_rows(c.nx, c.ny, c.dx, cs.params_from(c.params, tile_rows=32), 0, 1,
                                 [0, c.ny], 0, cs.csph_make_nccl_id())
    d.set_state(*f)
    d.step(20)
    d.rebalance_rows([0, c.ny])
    d.step(30)
    assert np.array_equal(d.get_dt_log(50)[0], dt0)
    for a, r in zip(d.get_state(), ref):
        assert np.array_equal(a, r)
    with pytest.raises(cs.CsphError):
        d.rebalance_rows([0, 2, c.ny])  # wrong rank count
    d.destroy()


@pytest.mark.parametrize("seed", range(int(os.environ.get("CSPH_STRIP_SEEDS", "8"))))
def test_randomised_strips_vs_oracle(cs, seed):
    """Randomised strip net: 2-6 strips with random bounds (>= 3 rows each),
    halo push or peer copies, automatic or fixed tile heights, HGS on/off, random config,
    grid spacing and physics switches, stepped in calls of 1-7 steps -- dt log and state
    bitwise the CPU oracle's after 40 steps."""
    import oracle
    rng = np.random.default_rng(7000 + seed)
    nx, ny = int(rng.integers(20, 220)), int(rng.integers(30, 240))
    name = ["C2", "C3", "C4", "C5"][int(rng.integers(0, 4))]
    c = synth.config(name, nx, ny)
    f = synth.fill(c)
    ph = dict(c.params, C_J=float(rng.uniform(0.0, 3.0)), K=float(rng.uniform(0.15, 0.35)),
              C_Sh=float(rng.choice([0.0, 4.0])), q_plus=float(rng.choice([0.0, 1e-6])))
    dx = float(rng.choice([1.0, 0.6, 3.0]))
    ns = int(rng.integers(2, 7))
    while True:
        cuts = sorted(rng.choice(np.arange(3, ny - 2), size=ns - 1, replace=False).tolist())
        bounds = [0] + cuts + [ny]
        if min(b - a for a, b in zip(bounds, bounds[1:])) >= 3:
            break
    kw = dict(halo_push=int(rng.integers(0, 2)), hgs=int(rng.integers(0, 2)),
              tile_rows=int(rng.choice([0, 0, 16, 24])))
    ref = oracle.Oracle(nx, ny, dx, oracle.Params(**ph))
    assert ref.set_state(*f) == 0
    st, dt0, lim0 = ref.step(40)
    g = cs.csph_create_multi_rows(nx, ny, dx, cs.params_from(ph, **kw), [0] * ns, bounds)
    g.set_state(*f)
    done, code = 0, 0
    while done < 40 and code == 0:  # steps in calls of 1-7: back to back and host-synchronised
        k = min(int(rng.integers(1, 8)), 40 - done)
        code = g.step(k, check=False)
        done += k
    assert code == st
    assert g.get_time() == ref.time()  # steps done, sum of tau, last tau
    dt, lim = g.get_dt_log(40)
    assert np.array_equal(dt, dt0) and np.array_equal(lim, lim0), (bounds, kw, dx)
    for a, r in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(a, r), (bounds, kw, dx)
    g.destroy()


def test_ghost_flag_rows_are_per_side(cs):
    """Each strip's two ghost-flag rows carry the facing tile row of the
    right neighbour: strip 1 (two 16-row tile rows, dry) sits between strip 0, whose dam-break
    front reaches its last row after a few steps (water then about to enter strip 1 from
    below), and strip 2, wet inside its first tile row but not at its ends (a slower tile
    whose flags have no BOT band).  Both transports; bitwise the single grid without HGS.
    Stepped one step per call, so that the three strips' kernels start together: a mutant
    writing strip 2's flags into strip 1's lower ghost row (racing with strip 0's correct
    write) then shows (profiles/r02_kernel_mutations.txt)."""
    nx, ny = 120, 128
    jj, ii = np.mgrid[0:ny, 0:nx]
    h = np.zeros((ny, nx))
    h[30:41, :] = 0.6  # strip 0's reservoir: its front reaches the strip edge after some steps
    h[81:95, :] = 0.8
    b = 0.5 - 0.004 * jj + 0.01 * np.sin(0.3 * ii)
    b[81:95, :] = 0.5 - 0.004 * 96  # strip 2's pool on a flat shelf between two bed walls,
    b[80, :] = b[95, :] = 2.0       # so its first tile row stays wet inside, dry at both ends
    z = np.zeros((ny, nx))
    f = (h, z.copy(), z.copy(), b, np.full((ny, nx), 0.4))
    phys = dict(n_manning=0.02, A_J=1e-3, C_J=1.0, C_Sh=0.0)
    steps = 120
    g = cs.csph_create(nx, ny, 1.0, cs.params_from(phys, hgs=0))
    g.set_state(*f)
    g.step(steps)
    dt0, ref = g.get_dt_log(steps)[0], g.get_state()
    g.destroy()
    assert ref[0][48:56].max() > 1e-3  # water entered strip 1's first tile row
    for push in (1, 0):
        g = cs.csph_create_multi_rows(nx, ny, 1.0, cs.params_from(phys, tile_rows=16,
                                                                  halo_push=push),
                                      [0] * 3, [0, 48, 80, ny])
        g.set_state(*f)
        for _ in range(steps):  # one step per call: the strips' kernels start together
            g.step(1)
        assert np.array_equal(g.get_dt_log(steps)[0], dt0), push
        for a, r in zip(g.get_state(), ref):
            assert np.array_equal(a, r), push
        g.destroy()
