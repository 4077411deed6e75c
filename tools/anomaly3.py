"""Intermittent slow strips (dev aid): like scaling_sim (a fresh fill per strip) but each strip
is timed three times on the same handle, to tell a transient stall from a slow handle."""
import os, sys
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, time, synth
from paper_2103_15196_b200 import csph
c = synth.config("C5")
def timed(g, n=10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    h0 = time.perf_counter()
    e0.record(); g.step(n); e1.record(); torch.cuda.synchronize()
    return round(e0.elapsed_time(e1) / n, 3), round((time.perf_counter() - h0) * 1e3 / n, 3)
for rnd in range(3):
    for N in (8,):
        b = [csph.csph_strip_rows(c.ny, N, r)[0] for r in range(N)] + [c.ny]
        out = []
        for r in range(N):
            f = synth.fill(c, b[r], b[r + 1])
            g = csph.csph_create(c.nx, b[r + 1] - b[r], c.dx, csph.params_from(c.params))
            g.set_state(*f); g.step(3); torch.cuda.synchronize()
            out.append([timed(g) for _ in range(3)])
            g.destroy()
        print("round", rnd, out, flush=True)
