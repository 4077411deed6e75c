"""Does re-balancing the row strips pay as the flood spreads?  (dev aid, one B200)

Runs the C5 16384^2 bench workload for T steps on one GPU, then predicts the N-GPU step time
from the state at step T for two partitions:
  * static   -- balanced on the INITIAL wet cells (what bench.py / a run without re-balancing
                keeps using),
  * rebalanced -- balanced on the wet cells of the state at step T (csph_row_weights ->
                csph_balance_rows, what csph_rebalance_rows would switch to),
each strip timed alone on the state at step T as a walled domain (as tools/scaling_sim.py).

    N=8 T=3000 python tools/rebalance_sim.py
"""
import os
import sys

os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_15196_b200 import csph  # noqa: E402

N = int(os.environ.get("N", "8"))
T = int(os.environ.get("T", "3000"))
steps = int(os.environ.get("STEPS", "10"))
c = synth.config("C5")
n = c.nx
f0 = synth.fill(c)
psi = f0[4]
w0 = (f0[0] > 1e-6).sum(axis=1) + 0.03 * n


def timed(g, k):
    g.step(4)  # even: the timed steps start at parity 0, whose pair graph is captured here
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.step(k); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / k


g = csph.csph_create(n, c.ny, c.dx, csph.params_from(c.params))
g.set_state(*f0)
del f0
g.step(T)
wT = g.row_weights()
state = g.get_state()
t_full = timed(g, steps)
g.destroy()
print(f"C5 at step {T}: whole grid {t_full:.3f} ms/step; wet fraction {(state[0] > 1e-6).mean():.3f}",
      flush=True)


def strip_ms(j0, j1):
    s = csph.csph_create(n, j1 - j0, c.dx, csph.params_from(c.params))
    s.set_state(*[a[j0:j1] for a in state], psi[j0:j1])
    t = timed(s, steps)
    s.destroy()
    return t


for kind, w in (("static", w0), ("rebalanced", wT)):
    b = csph.csph_balance_rows(c.ny, N, w)
    ts = [strip_ms(b[r], b[r + 1]) for r in range(N)]
    print(f"N={N} {kind:10s}: strips {[b[r + 1] - b[r] for r in range(N)]} ms "
          f"{[round(x, 3) for x in ts]} -> slowest {max(ts):.3f} ms, efficiency "
          f"{t_full / (N * max(ts)):.2f}", flush=True)
