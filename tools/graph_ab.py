"""CUDA-graph replay vs plain launches (dev aid, GPU): step time per config, measured with
CUDA events around csph_step (params.graphs = 1 / 0)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, synth
from paper_2103_15196_b200 import csph
cases = [("C2", 512, 400), ("C2", 1024, 400), ("C3", 2048, 200), ("C3", 4096, 100), ("C5", 16384, 20)]
for name, n, steps in cases:
    c = synth.config(name, n)
    f = synth.fill(c)
    out = []
    for graphs in (1, 0):
        g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, graphs=graphs))
        g.set_state(*f)
        g.step(10); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for rep in range(3):
            e0.record(); g.step(steps); e1.record(); torch.cuda.synchronize()
            best = min(best, e0.elapsed_time(e1) / steps)
        out.append(f"graphs={graphs}: {best * 1e3:8.1f} us/step {c.cells / best / 1e6:7.2f} Gcell/s")
        g.destroy()
    print(f"{name} {n:5d} | " + " | ".join(out), flush=True)
