"""Asynchronous Save (csph_save_begin / csph_save_wait, the Save block with
CUDA streams separating the CPU<->GPU copies from the computation).

A Save delivers the state as of the step it was issued after, bitwise, while later steps run
on the step stream; the steps themselves are unaffected (bitwise the same as a run without
saves, and the oracle's)."""
import numpy as np
import pytest
import torch

import oracle
import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cs():
    from paper_2103_15196_b200 import build, csph
    build.build()
    return csph


def pinned(ny, nx):
    return [torch.empty((ny, nx), dtype=torch.float64).pin_memory().numpy() for _ in range(4)]


def make(cs, c, kind, **kw):
    p = cs.params_from(c.params, **kw)
    if kind == "multi":
        return cs.csph_create_multi(c.nx, c.ny, c.dx, p, [0, 0, 0])
    return cs.csph_create(c.nx, c.ny, c.dx, p)


@pytest.mark.parametrize("kind,prec", [("single", 64), ("multi", 64), ("single", 32)])
def test_save_overlaps_steps_and_is_exact(cs, kind, prec):
    c = synth.config("C3", 260, 200)
    f = synth.fill(c)
    ref = make(cs, c, kind, precision=prec)
    ref.set_state(*f)
    ref.step(20)
    s20 = ref.get_state()
    ref.step(20)
    s40 = ref.get_state()
    ref.step(20)
    s60 = ref.get_state()

    g = make(cs, c, kind, precision=prec)
    g.set_state(*f)
    a, b = pinned(c.ny, c.nx), pinned(c.ny, c.nx)
    g.step(20)
    g.save_begin(*a)        # the state after 20 steps ...
    g.step(20)              # ... while steps 21..40 run
    g.save_begin(*b)        # a second Save, ordered after the first on the device
    g.step(20)
    g.save_wait()
    for x, r in zip(a, s20):
        assert np.array_equal(x, r)
    for x, r in zip(b, s40):
        assert np.array_equal(x, r)
    for x, r in zip(g.get_state(), s60):  # the steps are unaffected
        assert np.array_equal(x, r)
    assert np.array_equal(g.get_dt_log(60)[0], ref.get_dt_log(60)[0])
    g.save_wait()  # nothing pending: returns at once
    g.destroy()
    ref.destroy()


def test_save_matches_oracle_and_partial_fields(cs):
    c = synth.config("C5", 300, 260)
    f = synth.fill(c)
    o = oracle.Oracle(c.nx, c.ny, c.dx, oracle.Params(**c.params))
    assert o.set_state(*f) == 0
    assert o.step(30)[0] == 0
    g = cs.csph_create(c.nx, c.ny, c.dx, cs.params_from(c.params))
    g.set_state(*f)
    g.step(30)
    h, hu, hv, b = pinned(c.ny, c.nx)
    g.save_begin(h, None, None, b)  # any field may be skipped
    g.step(5)
    g.save_wait()
    rh, _, _, rb = o.get_state()
    assert np.array_equal(h, rh) and np.array_equal(b, rb)


def test_save_errors(cs):
    g = cs.csph_create(32, 24, 1.0, cs.csph_default_params())
    x = np.zeros((24, 32))
    with pytest.raises(cs.CsphError):
        g.save_begin(x, x, x, x)  # no state yet
    g.save_wait()  # nothing pending
    with pytest.raises(ValueError):
        g.save_begin(np.zeros((24, 32), dtype=np.float32), None, None, None)
    g.destroy()
    assert cs.lib().csph_save_wait(None) == cs.CSPH_EINVAL
