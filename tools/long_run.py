"""Long run of a workload (dev aid; CFG, default C5 16384^2) for N steps in chunks; reports the
simulated time, tau range, limiter histogram, wet fraction, volume/sediment bookkeeping
and throughput per chunk (the flood spreads, so the cost per step changes)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
c = synth.config(os.environ.get("CFG", "C5"))
f = synth.fill(c)
W = 1.0 / (1.0 - f[4])
vol0, sed0 = float(np.sum(f[0])), float(np.sum(f[3] / W))
g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(c.params, precision=int(os.environ.get("PREC", "64"))))
g.set_state(*f)
del f
steps, chunk = int(os.environ.get("STEPS", "3000")), 500
done = 0
while done < steps:
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); st = g.step(chunk, check=False); e1.record(); torch.cuda.synchronize()
    done += chunk
    t, n, last = g.get_time()
    dt, lim = g.get_dt_log(chunk)
    vol = sed = wet = 0.0; hmin = np.inf
    for j0 in range(0, c.ny, 2048):
        h, hu, hv, b = g.get_state_rows(j0, min(c.ny, j0 + 2048))
        vol += float(np.sum(h)); sed += float(np.sum(b / W[j0:min(c.ny, j0 + 2048)]))
        wet += float(np.count_nonzero(h > 1e-6)); hmin = min(hmin, float(h.min()))
    print(f"steps {n} status {st} t={t:.2f}s tau [{dt.min():.4f},{dt.max():.4f}] "
          f"lim {np.bincount(lim, minlength=4).tolist()} wet {wet / c.cells:.3f} "
          f"dvol {abs(vol - vol0) / vol0:.1e} dsed {abs(sed - sed0) / abs(sed0):.1e} "
          f"hmin {hmin:.1e} {c.cells * chunk / e0.elapsed_time(e1) / 1e6:.1f} Gcell/s", flush=True)
    if st:
        break
g.destroy()
