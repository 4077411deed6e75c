"""Time fused-kernel variants (CSPH_FUSED_VARIANT) and tile heights on C3/C5 (dev aid)."""
import os, sys, subprocess, json
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys, time, os
sys.path.insert(0, %r)
import torch, synth
from paper_2103_15196_b200 import csph
res = []
for name, n, steps in [("C3", 4096, 20), ("C5", 8192, 10)]:
    c = synth.config(name, n)
    f = synth.fill(c)
    for ty in [int(x) for x in os.environ.get("TYS", "128").split(",")]:
        g = csph.csph_create(c.nx, c.ny, 1.0, csph.params_from(c.params, tile_rows=ty))
        g.set_state(*f)
        g.step(3); torch.cuda.synchronize()
        t = time.time(); g.step(steps); torch.cuda.synchronize(); dt = time.time() - t
        res.append((name, ty, round(c.cells * steps / dt / 1e9, 2)))
        g.destroy()
print(res)
''' % ROOT
for v in sys.argv[1].split(","):
    env = dict(os.environ, CSPH_FUSED_VARIANT=v)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("variant", v, out.stdout.strip(), out.stderr.strip()[-300:], flush=True)
