"""Where does the long C5 run degrade (dev aid)? Max |b - b0|, max |v| and their cells."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
from paper_2103_15196_b200 import csph
c = synth.config("C5")
f = synth.fill(c)
b0 = f[3].copy()
ph = dict(c.params)
for k in ("C_J", "K", "eps_dry", "C_Sh"):
    if os.environ.get(k):
        ph[k] = float(os.environ[k])
print("params", ph, flush=True)
g = csph.csph_create(c.nx, c.ny, c.dx, csph.params_from(ph))
g.set_state(*f)
del f
done = 0
for target in [int(x) for x in os.environ.get("TARGETS", "500,600,650,700,800,1000").split(",")]:
    g.step(target - done); done = target
    h, hu, hv, b = g.get_state()
    db = np.abs(b - b0)
    wet = h > 1e-6
    sp = np.zeros_like(h); sp[wet] = np.hypot(hu[wet], hv[wet]) / h[wet]
    jb = np.unravel_index(np.argmax(db), db.shape); jv = np.unravel_index(np.argmax(sp), sp.shape)
    dt, lim = g.get_dt_log(1)
    print(f"step {done} tau {dt[-1]:.2e} lim {lim[-1]} | max|db| {db[jb]:.3e} at {jb} h={h[jb]:.3e} "
          f"| max|v| {sp[jv]:.3e} at {jv} h={h[jv]:.3e} hu={hu[jv]:.3e} | "
          f"cells |db|>1m: {int((db > 1).sum())}, |v|>20: {int((sp > 20).sum())}", flush=True)
    if os.environ.get("WIN") and done == 1000:
        j, i = jv
        print("h window\n", np.array2string(h[j-2:j+3, i-2:i+3], precision=3))
        print("b window\n", np.array2string(b[j-2:j+3, i-2:i+3], precision=3))
g.destroy()
