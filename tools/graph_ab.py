"""CUDA-graph replay vs plain launches on small grids (dev aid): step time per config."""
import os, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
code = r'''
import sys; sys.path.insert(0, %r)
import torch, synth
from paper_2103_15196_b200 import csph
out = []
for name, n in [("C2", 512), ("C2", 1024), ("C3", 2048)]:
    c = synth.config(name, n)
    g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params))
    g.set_state(*synth.fill(c))
    g.step(10); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.step(400); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 400
    out.append("%%s %%d: %%.1f us/step %%.2f Gcell/s" %% (name, n, ms * 1e3, c.cells / ms / 1e6))
    g.destroy()
print(" | ".join(out))
''' % ROOT
for nog in ("", "1"):
    env = dict(os.environ)
    if nog:
        env["CSPH_NO_GRAPHS"] = "1"
    else:
        env.pop("CSPH_NO_GRAPHS", None)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True)
    print("no-graphs" if nog else "graphs   ", r.stdout.strip(), r.stderr.strip()[-300:], flush=True)
