"""Where the per-strip overhead of the multi-GPU partition goes (dev aid).

For the whole C5 grid and each strip of the N-GPU balanced partition (each run alone as a
walled domain on one B200, as tools/scaling_sim.py does): step time, fused-kernel time,
HGS tiles marched / copied / skipped per step, the tile height, and the kernel time per
marched tile-row-iteration x resident CTA slots (us) -- equal across strips when a strip's
kernel is as efficient as the whole grid's."""
import os, sys
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2103_15196_b200 import csph

c = synth.config("C5")
n = c.nx
N = int(os.environ.get("N", "8"))
TY = int(os.environ.get("TY", "0"))
steps = 10
slots = torch.cuda.get_device_properties(0).multi_processor_count * 3
wet_rows = np.zeros(c.ny)
for j0 in range(0, c.ny, 2048):
    wet_rows[j0:j0 + 2048] = (synth.fill(c, j0, j0 + 2048)[0] > 1e-6).sum(axis=1)
w = wet_rows + 0.03 * n


def anatomy(j0, j1):
    f = synth.fill(c, j0, j1)
    g = csph.csph_create(n, j1 - j0, c.dx, csph.params_from(c.params, tile_rows=TY))
    g.set_state(*f)
    del f
    g.step(4)  # even: the timed steps start at parity 0, whose pair graph is captured here
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); g.step(steps); e1.record(); torch.cuda.synchronize()
    step_ms = e0.elapsed_time(e1) / steps
    g.reset_tile_stats(); g.profile(True); g.step(steps); torch.cuda.synchronize()
    kms, k = g.get_profile(); kms /= k
    m, ci, sk = (x / steps for x in g.tile_stats())
    g.profile(False); g.destroy()
    ntx = (n + 119) // 120
    ty = (j1 - j0) * ntx / (m + ci + sk)  # tiles per step = ntx * ceil(rows / ty)
    ty = min([16, 32, 64, 128], key=lambda t: abs(ntx * -(-(j1 - j0) // t) - (m + ci + sk)))
    it = m * (ty + 6)
    print(f"rows [{j0:5d},{j1:5d}) {j1 - j0:5d}  step {step_ms:.3f} ms  kernel {kms:.3f} ms  "
          f"TY {ty:3d}  tiles marched {m:7.0f} copied {ci:5.0f} skipped {sk:6.0f}  "
          f"waves {m / slots:5.2f}  us/(tile-iter/slot) {kms * 1e3 / (it / slots):.2f}", flush=True)
    return step_ms, kms


t1, k1 = anatomy(0, c.ny)
b = csph.csph_balance_rows(c.ny, N, w)
ts = [anatomy(b[r], b[r + 1]) for r in range(N)]
print(f"sum of strip steps {sum(t for t, _ in ts):.3f} ms (whole {t1:.3f}), kernels "
      f"{sum(k for _, k in ts):.3f} ms (whole {k1:.3f})")
