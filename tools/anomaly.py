"""Repeated timing of one C5 strip (dev aid): looks for intermittent slow runs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2103_15196_b200 import csph
c = synth.config("C5")
for (j0, j1) in [(10157 - 0, 11190), (12212, 15479), (0, 4001)]:
    f = synth.fill(c, j0, j1)
    for rep in range(4):
        g = csph.csph_create(c.nx, j1 - j0, c.dx, csph.params_from(c.params))
        g.set_state(*f)
        g.step(3); torch.cuda.synchronize()
        res = []
        for k in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); g.step(10); e1.record(); torch.cuda.synchronize()
            res.append(round(e0.elapsed_time(e1) / 10, 3))
        print(j0, j1, os.environ.get("CSPH_NO_GRAPHS", "graphs"), "rep", rep, res, g.tile_stats(), flush=True)
        g.destroy()
