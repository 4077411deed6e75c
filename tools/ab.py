"""A/B kernel timing of libcsph variants (dev aid): python tools/ab.py variants/libcsph_a.so ...

Each library runs in its own process (CSPH_LIB_DEV) on all-wet and C5 (N = $N, default 8192);
prints the fused kernel's CUDA-event time per step and Gcell/s."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import os, sys
sys.path.insert(0, %r)
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
n = int(os.environ.get("N", "8192"))
phys = dict(n_manning=0.03, A_J=0.001, C_J=2.0, C_Sh=4.0, d50=1e-3)
x = np.linspace(0, 20 * np.pi, n)
X, Y = np.meshgrid(x, x)
wet = (1.0 + 0.2 * np.sin(X) * np.cos(Y), 0.8 * np.ones((n, n)), 0.3 * np.ones((n, n)),
       0.05 * np.cos(X + Y), np.full((n, n), 0.4))
c = synth.config("C5", n)
out = []
for name, f, p in [("wet", wet, phys), ("C5", synth.fill(c), c.params)]:
    g = csph.csph_create(n, n, 1.0, csph.params_from(p))
    g.set_state(*f)
    g.step(3); torch.cuda.synchronize()
    best = 1e9
    for rep in range(3):
        g.profile(True); g.step(10); torch.cuda.synchronize()
        ms, k = g.get_profile(); best = min(best, ms / k)
    out.append("%%s %%.3f ms %%.2f Gcell/s" %% (name, best, n * n / best / 1e6))
    g.destroy()
print(" | ".join(out))
''' % ROOT
for lib in sys.argv[1:]:
    env = dict(os.environ, CSPH_LIB_DEV=os.path.abspath(lib))
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print(os.path.basename(lib), r.stdout.strip(), r.stderr.strip()[-400:], flush=True)
