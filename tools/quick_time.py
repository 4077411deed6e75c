"""Ad-hoc timing of both paths on C3/C5 (development aid, not the bench)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2103_15196_b200 import csph

for name, n, steps in [("C3", 4096, 20), ("C5", 8192, 10)]:
    c = synth.config(name, n)
    h, hu, hv, b, psi = synth.fill(c)
    for path in (0, 1):
        g = csph.csph_create(c.nx, c.ny, 1.0, csph.params_from(c.params, path=path))
        g.set_state(h, hu, hv, b, psi)
        g.step(3)
        torch.cuda.synchronize()
        t = time.time(); g.step(steps); dt = time.time() - t
        print(f"{name} {n}^2 path={'fused' if path == 0 else 'staged'}: {dt/steps*1e3:.3f} ms/step, "
              f"{c.cells*steps/dt/1e9:.2f} Gcell/s", flush=True)
        g.destroy()
