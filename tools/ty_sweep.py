"""Fused-kernel time for several tile heights (dev aid, GPU): CFG (default C5) at N
(default: the config's size), tile heights from argv (0 = the library's auto rule)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2103_15196_b200 import csph
if len(sys.argv) > 1 and sys.argv[1].endswith(".so"):
    csph.SO_PATH = os.path.abspath(sys.argv.pop(1))
c = synth.config(os.environ.get("CFG", "C5"))
n = int(os.environ.get("N", str(c.nx)))
c = synth.config(c.name, n)
f = synth.fill(c)
for ty in [int(x) for x in (sys.argv[1:] or ["128", "256"])]:
    g = csph.csph_create(n, n, 1.0, csph.params_from(c.params, tile_rows=ty))
    g.set_state(*f)
    g.step(3); torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        g.profile(True); g.reset_tile_stats(); g.step(10); torch.cuda.synchronize()
        ms, k = g.get_profile(); best = min(best, ms / k)
    t = g.tile_stats()
    print(f"{c.name} TY {ty}: {best:.3f} ms {n*n/best/1e6:.2f} Gcell/s tiles marched {t[0]/sum(t):.3f}", flush=True)
    g.destroy()
