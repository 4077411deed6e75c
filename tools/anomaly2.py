"""Intermittent slow strips (dev aid): after a full-grid handle, create/time/destroy the N=4
balanced C5 strips for several rounds; a slow strip is re-timed on the same handle."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
c = synth.config("C5")
f = synth.fill(c)
w = (f[0] > 1e-6).sum(axis=1) + 0.03 * c.nx
def timed(g, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.step(n); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n
g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params))
g.set_state(*f); g.step(3); print("full", round(timed(g), 3), flush=True); g.destroy()
for N in (4, 8):
    b = csph.csph_balance_rows(c.ny, N, w)
    for rnd in range(3):
        out = []
        for r in range(N):
            j0, j1 = b[r], b[r + 1]
            g = csph.csph_create(c.nx, j1 - j0, c.dx, csph.params_from(c.params))
            g.set_state(*[a[j0:j1] for a in f]); g.step(3); torch.cuda.synchronize()
            t1 = timed(g); t2 = timed(g)
            out.append((round(t1, 3), round(t2, 3)))
            g.destroy()
        print("N", N, "round", rnd, out, flush=True)
