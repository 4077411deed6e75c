"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(fused path, HGS on, default tiling), at north_star's 100 steps.

* C3 4096^2 (the third config, 16.7 M cells): the whole grid against the oracle over
  100 steps -- every cell and the dt log bitwise (about 2.5 min of oracle time).
* C4: SURVEY 8(d)'s oracle crop of the 8192^2 field, columns [3584, 4608) x rows
  [0, 2048) (the dam, the breach and the channel) as its own walled domain, 100 steps,
  whole crop and dt log bitwise.
* C5 16384^2 (the bench workload, 268 M cells): the oracle cannot run the whole grid in
  test time, so (a) tau_0 is computed by the oracle from the Eq.7 maxima of the initial
  state, reduced strip by strip (max is exact and order-free); (b) after
  k = 20 and k = 100 GPU steps, sampled 48 x 48 patches (wall corners, wet/dry fronts,
  random interior points) are recomputed by the oracle: the patch's dependency cone, a
  window of 48 + 6k cells with its 3 ghost layers taken from the real neighbours (walls
  mirrored by the oracle itself), stepped k times with the GPU's own tau log -- cells
  farther than 3k from the window edge are exact (stencil radius 3);
  (c) properties that hold at any size over 12 steps: HGS on == HGS off bitwise, exact
  volume bookkeeping of the walled domain, no negative depth."""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu
GH = oracle.GHOST


@pytest.fixture(scope="module")
def cs():
    from paper_2103_15196_b200 import build, csph
    build.build()
    return csph


def _whole_vs_oracle(cs, c, f, steps):
    ref = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    assert ref.set_state(*f) == 0
    st, dt_ref, lim_ref = ref.step(steps)
    assert st == 0 and len(dt_ref) == steps
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params))
    g.set_state(*f)
    g.step(steps)
    dt, lim = g.get_dt_log(steps)
    assert np.array_equal(dt, dt_ref) and np.array_equal(lim, lim_ref)
    for a, r in zip(g.get_state(), ref.get_state()):
        assert np.array_equal(a, r)
    g.destroy()


def test_C3_full_grid_100_steps_bitwise(cs):
    c = synth.config("C3")
    assert (c.nx, c.ny) == (4096, 4096)
    _whole_vs_oracle(cs, c, synth.fill(c), 100)


def test_C4_survey_crop_100_steps_bitwise(cs):
    """the crop i in [3584, 4608), j in [0, 2048) of the 8192^2 fields,
    run as its own walled domain (it holds the dam rows 1016-1023, the breach and the
    channel: moving wet/dry fronts)."""
    c8 = synth.config("C4")
    assert (c8.nx, c8.ny) == (8192, 8192)
    rows = synth.fill(c8, 0, 2048)
    f = tuple(np.ascontiguousarray(a[:, 3584:4608]) for a in rows)
    c = synth.Config("C4crop", 4, 1024, 2048, c8.dx, 0, dict(c8.params))
    h = f[0]
    assert (h[:1016] > 1e-6).any() and (h[1024:] > 1e-6).any()  # reservoir and channel
    _whole_vs_oracle(cs, c, f, 100)


def _window(a, i0, i1, j0, j1, fill):
    """Padded window of rows j0-3..j1+3, cols i0-3..i1+3; cells outside the grid get
    `fill` (they are wall ghosts, which the oracle mirrors itself)."""
    ny, nx = a.shape
    out = np.full((j1 - j0 + 2 * GH, i1 - i0 + 2 * GH), fill)
    ja, jb = max(0, j0 - GH), min(ny, j1 + GH)
    ia, ib = max(0, i0 - GH), min(nx, i1 + GH)
    out[ja - (j0 - GH):jb - (j0 - GH), ia - (i0 - GH):ib - (i0 - GH)] = a[ja:jb, ia:ib]
    return out


def _patches(wet, n, rng, size):
    ny, nx = wet.shape
    m = size
    ps = [(0, 0), (nx - m, 0), (0, ny - m), (nx - m, ny - m)]  # wall corners
    # wet/dry fronts: cells whose east neighbour differs
    fr = np.argwhere(wet[:, :-1] != wet[:, 1:])
    for k in rng.choice(len(fr), size=6, replace=False):
        j, i = fr[k]
        ps.append((int(np.clip(i - m // 2, 0, nx - m)), int(np.clip(j - m // 2, 0, ny - m))))
    for _ in range(n):
        ps.append((int(rng.integers(0, nx - m)), int(rng.integers(0, ny - m))))
    return ps


def test_C5_full_size_cones_vs_oracle(cs):
    c = synth.config("C5")
    assert (c.nx, c.ny) == (16384, 16384)
    P = oracle.Params(**c.params)
    f = synth.fill(c)
    h, hu, hv, b, psi = f
    # (a) tau_0 from the oracle's Eq.7 maxima of the initial state, strip by strip
    M = np.zeros(3)
    step = 1024
    for j0 in range(0, c.ny, step):
        j1 = min(c.ny, j0 + step)
        o = oracle.Oracle(c.nx, j1 - j0, c.dx, P)
        assert o.set_state(h[j0:j1], hu[j0:j1], hv[j0:j1], b[j0:j1], psi[j0:j1]) == 0
        M = np.maximum(M, o.reduce_M())
        del o
    st, tau0, lim0 = oracle.Oracle(8, 8, c.dx, P).tau_from_M(M)
    assert st == 0
    # the GPU, bench configuration
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params))
    g.set_state(*f)
    size = 48
    W = 1.0 / (1.0 - psi)
    rng = np.random.default_rng(2103)
    patches = _patches(h > P.eps_dry, 4, rng, size)
    done = 0
    for k in (20, 100):
        g.step(k - done)
        done = k
        dt, lim = g.get_dt_log(k)
        assert len(dt) == k and dt[0] == tau0 and lim[0] == lim0
        m = 3 * k  # the dependency cone of the patch after k steps
        for (pi, pj) in patches:
            i0, i1 = max(0, pi - m), min(c.nx, pi + size + m)
            j0, j1 = max(0, pj - m), min(c.ny, pj + size + m)
            o = oracle.Oracle(i1 - i0, j1 - j0, c.dx, P)
            o.set_walls(i0 == 0, i1 == c.nx, j0 == 0, j1 == c.ny)
            assert o.set_state_padded(*[_window(a, i0, i1, j0, j1, 0.0) for a in (h, hu, hv, b)],
                                      _window(W, i0, i1, j0, j1, 1.0)) == 0
            for tau in dt:
                assert o.step_tau(float(tau)) == 0
            ref = o.get_state()
            got = g.get_state_rows(pj, pj + size)
            for a, r in zip(got, ref):
                assert np.array_equal(a[:, pi:pi + size],
                                      r[pj - j0:pj - j0 + size, pi - i0:pi - i0 + size]), (k, pi, pj)
            del o
    g.destroy()


def test_C5_full_size_fp32_cones_vs_binary32_oracle(cs):
    """NEXT-2 at the bench's size: the fp32 mode on C5 16384^2 (the `bench.py --precision 32`
    configuration) against the binary32 oracle (reading #33) on the dependency cones of 48^2
    patches (wall corners, wet/dry fronts, random) after 20 and 100 steps, replaying the
    GPU's tau log -- bitwise."""
    c = synth.config("C5")
    P = oracle.Params(**c.params)
    f = synth.fill(c)
    h, hu, hv, b, psi = f
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, precision=32))
    g.set_state(*f)
    size = 48
    W = 1.0 / (1.0 - psi)  # rounded to binary32 by the oracle as by the library
    rng = np.random.default_rng(2104)
    patches = _patches(h > P.eps_dry, 4, rng, size)
    done = 0
    for k in (20, 100):
        g.step(k - done)
        done = k
        dt, _ = g.get_dt_log(k)
        assert len(dt) == k
        m = 3 * k
        for (pi, pj) in patches:
            i0, i1 = max(0, pi - m), min(c.nx, pi + size + m)
            j0, j1 = max(0, pj - m), min(c.ny, pj + size + m)
            o = oracle.Oracle(i1 - i0, j1 - j0, c.dx, P, precision=32)
            o.set_walls(i0 == 0, i1 == c.nx, j0 == 0, j1 == c.ny)
            assert o.set_state_padded(*[_window(a, i0, i1, j0, j1, 0.0) for a in (h, hu, hv, b)],
                                      _window(W, i0, i1, j0, j1, 1.0)) == 0
            for tau in dt:
                assert o.step_tau(float(tau)) == 0
            ref = o.get_state()
            got = g.get_state_rows(pj, pj + size)
            for a, r in zip(got, ref):
                assert np.array_equal(a[:, pi:pi + size],
                                      r[pj - j0:pj - j0 + size, pi - i0:pi - i0 + size]), (k, pi, pj)
            del o
    g.destroy()


def test_C5_full_size_hgs_and_conservation(cs):
    c = synth.config("C5")
    f = synth.fill(c)
    W = 1.0 / (1.0 - f[4])
    vol0 = float(np.sum(f[0]))
    sed0 = float(np.sum(f[3] / W))  # sum (1 - psi) b
    steps = 12
    gs = []
    for hgs in (1, 0):  # both handles resident (2 x 19 GB of HBM)
        g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, hgs=hgs))
        g.set_state(*f)
        g.step(steps)
        gs.append(g)
    del f
    assert np.array_equal(gs[0].get_dt_log(steps)[0], gs[1].get_dt_log(steps)[0])
    assert gs[0].tile_stats()[2] > 0  # HGS skipped tiles
    vol = sed = 0.0
    hmin = np.inf
    for j0 in range(0, c.ny, 2048):  # row chunks: bounded host memory
        a = gs[0].get_state_rows(j0, j0 + 2048)
        r = gs[1].get_state_rows(j0, j0 + 2048)
        for x, y in zip(a, r):
            assert np.array_equal(x, y), j0
        vol += float(np.sum(a[0]))
        sed += float(np.sum(a[3] / W[j0:j0 + 2048]))
        hmin = min(hmin, float(a[0].min()))
    for g in gs:
        g.destroy()
    assert hmin >= -1e-12
    # walls: no mass crosses the boundary; R's update is a flux difference, so the sums
    # change only by rounding (268 M cells, 12 steps)
    assert abs(vol - vol0) <= 1e-11 * vol0
    assert abs(sed - sed0) <= 1e-11 * abs(sed0)


def test_C5_full_size_long_run(cs):
    """The bench workload over 1200 steps (about 38 s of simulated flood; without reading
    #31 the bed blew up after ~800): no error status, tau > 0.01 s every
    step, volume and Sum (1 - psi) b kept to rounding, no depth below -neg_tol, no NaN."""
    c = synth.config("C5")
    f = synth.fill(c)
    W = 1.0 / (1.0 - f[4])
    vol0 = float(np.sum(f[0]))
    sed0 = float(np.sum(f[3] / W))
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params))
    g.set_state(*f)
    del f
    steps = 1200
    assert g.step(steps) == 0
    dt, lim = g.get_dt_log(steps)
    assert len(dt) == steps and np.all(np.isfinite(dt)) and np.all(dt > 0.01)
    t, n, _ = g.get_time()
    assert n == steps and t == pytest.approx(float(np.sum(dt)), rel=1e-12)
    vol = sed = 0.0
    for j0 in range(0, c.ny, 2048):
        h, hu, hv, b = g.get_state_rows(j0, j0 + 2048)
        assert np.all(np.isfinite(h)) and np.all(np.isfinite(hu)) and np.all(np.isfinite(b))
        assert h.min() >= -1e-12
        vol += float(np.sum(h))
        sed += float(np.sum(b / W[j0:j0 + 2048]))
    g.destroy()
    assert abs(vol - vol0) <= 1e-10 * vol0
    assert abs(sed - sed0) <= 1e-10 * abs(sed0)


def test_C5_literal_eq5_blow_up(cs):
    """Reading #31 / DESIGN.md 3.15 reproduced at full size: with the literal Eq.5
    (`h_bed_min = 0`, films of any depth carry bedload) the bench workload's bed at the
    downstream wall end of the channel runs away within ~1000 steps -- the step ends in an
    error, or tau collapses, or the bed moves by metres in one 100-step chunk.  The default
    cut-off (h_bed_min = d50) runs the same 1200 steps cleanly (test_C5_full_size_long_run)."""
    c = synth.config("C5")
    f = synth.fill(c)
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params, h_bed_min=0.0))
    g.set_state(*f)
    b0 = f[3][c.ny - 64:, :].copy()
    del f
    blew, why = False, ""
    for chunk in range(12):
        st = g.step(100, check=False)
        if st != 0:
            blew, why = True, f"status {st} in steps {100 * chunk}..{100 * chunk + 100}"
            break
        dt, _ = g.get_dt_log(100)
        if dt.min() < 1e-3:
            blew, why = True, f"tau {dt.min():.3g} s by step {100 * chunk + 100}"
            break
        b = g.get_state_rows(c.ny - 64, c.ny)[3]
        if not np.all(np.isfinite(b)) or np.max(np.abs(b - b0)) > 50.0:
            blew, why = True, f"|db| {np.nanmax(np.abs(b - b0)):.3g} m by step {100 * chunk + 100}"
            break
    g.destroy()
    assert blew, "the literal Eq.5 run stayed bounded for 1200 steps"
    print("literal Eq.5:", why)
