"""C5 16384^2 as N load-balanced strips on ONE GPU (csph_create_multi_rows): step time and HGS
tile counts with the halo push (halo_push = 1) and with peer copies (0) (dev aid)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
c = synth.config("C5")
f = synth.fill(c)
w = (f[0] > 1e-6).sum(axis=1) + 0.03 * c.nx
for N, push in ((1, 1), (8, 1), (8, 0)):
    b = csph.csph_balance_rows(c.ny, N, w)
    g = csph.csph_create_multi_rows(c.nx, c.ny, c.dx, csph.params_from(c.params, halo_push=push),
                                    [0] * N, b)
    g.set_state(*f)
    g.step(4); torch.cuda.synchronize()
    g.reset_tile_stats()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.step(10); e1.record(); torch.cuda.synchronize()
    print(N, "strips, push", push, ":", round(e0.elapsed_time(e1) / 10, 3), "ms/step, tiles (marched, copied, skipped)", g.tile_stats(), flush=True)
    g.destroy()
