"""Per-cell cost of the fused kernel on all-wet, all-dry and C5 (dev aid)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2103_15196_b200 import csph

n = int(os.environ.get("N", "8192"))
phys = dict(n_manning=0.03, A_J=0.001, C_J=2.0, C_Sh=4.0, d50=1e-3)
x = np.linspace(0, 20 * np.pi, n)
X, Y = np.meshgrid(x, x)
wet = (1.0 + 0.2 * np.sin(X) * np.cos(Y), 0.8 * np.ones((n, n)), 0.3 * np.ones((n, n)),
       0.05 * np.cos(X + Y), np.full((n, n), 0.4))
dry = (np.zeros((n, n)), np.zeros((n, n)), np.zeros((n, n)), 0.05 * np.cos(X + Y), np.full((n, n), 0.4))
dry[0][n // 2, n // 2] = 1.0
c5 = synth.fill(synth.config("C5", n))
only = os.environ.get("ONLY")
for name, f in [("all-wet", wet), ("all-dry", dry), ("C5", c5)]:
    if only and name != only:
        continue
    for ty in [int(v) for v in os.environ.get("TYS", "64,128").split(",")]:
        g = csph.csph_create(n, n, 1.0, csph.params_from(phys, tile_rows=ty))
        g.set_state(*f)
        g.step(2); torch.cuda.synchronize()
        g.profile(True)
        g.step(int(os.environ.get("STEPS", "10"))); torch.cuda.synchronize()
        ms, k = g.get_profile()
        print(f"{name:8s} TY={ty}: kernel {ms/k:.3f} ms, {n*n/(ms/k)/1e6:.2f} Gcell/s", flush=True)
        g.destroy()
