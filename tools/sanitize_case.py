#!/usr/bin/env python3
"""Small runs of every kernel family for compute-sanitizer (tests/test_gpu_sanitizers.py).

    compute-sanitizer --tool memcheck python tools/sanitize_case.py --case fused

Cases (each a few steps on a small grid, so that racecheck's ~100x slowdown stays in
seconds): fused (hot-path specialisation, HGS on, CUDA-graph replay and a profiled plain
launch), general (the NEXT-3/4 instance: open edges, n_M/beta/src fields, Eq.4 A_J, m = 3),
staged (the K1..K8 kernels + mirrors), strips (3 uneven strips with 16-row tiles: halos pushed
by the step kernel, then overlapped edge / peer-copy halo / interior launches), fp32 (the NEXT-2 instance), tiles (every tile height
with a ragged last tile column and row).  Every case also checks its result against a
reference (the single grid or the fused path) so a sanitizer run is also a parity run.
No torch import: only the ctypes binding and numpy.
"""
from __future__ import annotations

import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from paper_2103_15196_b200 import csph  # noqa: E402


def run(g, f, steps, fields=None):
    g.set_state(*f)
    if fields:
        g.set_fields(**fields)
    g.step(steps)
    return g.get_dt_log(steps)[0], g.get_state()


def same(a, b):
    (da, sa), (db, sb) = a, b
    assert np.array_equal(da, db)
    for x, y in zip(sa, sb):
        assert np.array_equal(x, y)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", required=True)
    a = ap.parse_args()
    c = synth.config("C5", 250, 150)
    f = synth.fill(c)
    P = c.params
    if a.case == "fused":
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(P, tile_rows=32))
        r1 = run(g, f, 6)               # graph replay (pairs)
        g.profile(True)                 # plain launches with events
        g.set_state(*f)
        g.step(6)
        r2 = (g.get_dt_log(6)[0], g.get_state())
        same(r1, r2)
        g.destroy()
    elif a.case == "general":
        ny, nx = c.ny, c.nx
        rng = np.random.default_rng(5)
        fl = dict(n_manning=rng.uniform(0.0, 0.04, (ny, nx)), beta=np.full((ny, nx), 1e-4),
                  src=np.where(rng.random((ny, nx)) < 0.01, 1e-3, 0.0))
        prm = dict(P, open_bc=5, aj_mode=1, m_grass=3)
        g = csph.csph_create(nx, ny, c.dx, csph.params_from(prm, tile_rows=32))
        r1 = run(g, f, 5, fl)
        g.destroy()
        s = csph.csph_create(nx, ny, c.dx, csph.params_from(prm, path=csph.CSPH_PATH_STAGED))
        same(r1, run(s, f, 5, fl))
        s.destroy()
    elif a.case == "staged":
        s = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(P, path=csph.CSPH_PATH_STAGED))
        r1 = run(s, f, 4)
        s.destroy()
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(P))
        same(r1, run(g, f, 4))
        g.destroy()
    elif a.case == "strips":
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(P))
        r1 = run(g, f, 5)
        g.destroy()
        for push in (1, 0):  # halos pushed by the kernel / peer copies after the edge rows
            m = csph.csph_create_multi_rows(c.nx, c.ny, c.dx,
                                            csph.params_from(P, tile_rows=16, halo_push=push),
                                            [0, 0, 0], [0, 49, 98, c.ny])
            same(r1, run(m, f, 5))
            m.destroy()
    elif a.case == "fp32":
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(P, precision=32, tile_rows=32))
        d, st = run(g, f, 5)
        assert np.all(np.isfinite(st[0]))
        g.destroy()
    elif a.case == "tiles":
        c2 = synth.config("C5", 241, 83)  # 3 tile columns, the last 1 wide; ragged rows
        f2 = synth.fill(c2)
        ref = None
        for ty in (16, 32, 64, 128):
            g = csph.csph_create(c2.nx, c2.ny, c2.dx, csph.params_from(P, tile_rows=ty))
            r = run(g, f2, 3)
            g.destroy()
            if ref is None:
                ref = r
            else:
                same(ref, r)
    else:
        raise SystemExit(f"unknown case {a.case}")
    print("case ok:", a.case)


if __name__ == "__main__":
    main()
