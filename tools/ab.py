"""A/B kernel timing of libcsph variants (dev aid, GPU):

    python tools/ab.py variants/libcsph_a.so variants/libcsph_b.so ...

Each library runs in its own process (the child points the binding's SO_PATH at it before
the first call -- a tool-side override, the product binding has no switch) on the bench
workload C5 (N = $N, default 16384) and an all-wet field (N/2), and prints the fused
kernel's CUDA-event time per step (best of 3 x 10 steps) and Gcell/s.  Variants are
interleaved over $ROUNDS rounds (default 2) so that clock drift hits all of them alike."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys
sys.path.insert(0, %r)
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
csph.SO_PATH = sys.argv[1]
n = int(os.environ.get("N", "16384"))
phys = dict(n_manning=0.03, A_J=0.001, C_J=2.0, C_Sh=4.0, d50=1e-3)
m = n // 2
x = np.linspace(0, 20 * np.pi, m)
X, Y = np.meshgrid(x, x)
wet = (1.0 + 0.2 * np.sin(X) * np.cos(Y), 0.8 * np.ones((m, m)), 0.3 * np.ones((m, m)),
       0.05 * np.cos(X + Y), np.full((m, m), 0.4))
c = synth.config("C5", n)
out = []
cases = [("C5", n, lambda: synth.fill(c), c.params), ("wet", m, lambda: wet, phys)]
if os.environ.get("C34"):
    c3, c4 = synth.config("C3"), synth.config("C4")
    cases += [("C3", 4096, lambda: synth.fill(c3), c3.params), ("C4", 8192, lambda: synth.fill(c4), c4.params)]
for name, nn, ff, p in cases:
    f = ff()
    g = csph.csph_create(nn, nn, 1.0, csph.params_from(p, precision=int(os.environ.get("PREC", "64"))))
    g.set_state(*f)
    del f
    g.step(3); torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        g.profile(True); g.step(10); torch.cuda.synchronize()
        ms, k = g.get_profile(); best = min(best, ms / k)
    out.append("%%s %%.3f ms %%.2f Gcell/s" %% (name, best, nn * nn / best / 1e6))
    g.destroy()
print(" | ".join(out))
''' % ROOT
libs = sys.argv[1:]
for rnd in range(int(os.environ.get("ROUNDS", "2"))):
    for lib in libs:
        r = subprocess.run([sys.executable, "-c", code, os.path.abspath(lib)], capture_output=True,
                           text=True)
        print(f"r{rnd} {os.path.basename(lib):28s}", r.stdout.strip(), r.stderr.strip()[-300:],
              flush=True)
