"""Predicted strong scaling of C5 16384^2 on one GPU (dev aid): each rank's strip
of rows [j0, j1) is run alone as a walled domain and its step time measured; the N-GPU step
time is the slowest strip plus the communication the step cannot hide, modelled as:

  * HALO=push (default; csph_ipc_link, the bench's --halo push): the ghost rows are written by
    the edge tiles' K8 epilogue over NVLink (3 rows x 4 fields x the padded row per side,
    ~1.6 MB, ~2 us at NVLink 5 rates) inside the step kernel -- nothing exposed, and the strip
    is launched whole exactly as timed here;
    HALO=nccl: 3 rows x 4 fields x the padded row (2 sides) over NVLink 5 at HALO_GBS
    (default 300 GB/s effective for ~1.6 MB NCCL send/recv) + HALO_US latency (default 15 us)
    on the comm stream while the interior tile rows compute (only the excess over the
    interior launch is exposed); the strips are timed through a 1-rank DIST handle with
    halo_push = 0, i.e. with the edge / interior split launches;
  * the combine of the Eq.7 maxima, fully exposed (the ctrl kernel needs tau before the next
    step): with HALO=push the ctrl kernels' peer combine -- 8 x 40 B of NVLink stores and a
    flag poll, COMBINE_US (default 5 us); with HALO=nccl the 32 B max-allreduce, ALLRED_US
    (default 20 us, NCCL on 8 GPUs of one NVSwitch node).

Compares the paper's even Ny_dev split with the wet-count-balanced one."""
import os, sys
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")  # see bench.py
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth
from paper_2103_15196_b200 import csph

c = synth.config("C5")
n = c.nx
steps = int(os.environ.get("STEPS", "10"))
REPS = int(os.environ.get("REPS", "3"))
REBAL = int(os.environ.get("REBAL", "2"))  # measured-time re-balancing rounds
TY = int(os.environ.get("TY", "0"))  # tile rows (0 = the library's auto rule)
NS = [int(x) for x in os.environ.get("NS", "2,4,8").split(",")]
KINDS = os.environ.get("KINDS", "even,balanced").split(",")
wet_rows = np.zeros(c.ny)
for j0 in range(0, c.ny, 2048):
    wet_rows[j0:j0 + 2048] = (synth.fill(c, j0, j0 + 2048)[0] > 1e-6).sum(axis=1)
w = wet_rows + 0.03 * n


def strip_ms(j0, j1):
    f = synth.fill(c, j0, j1)
    if HALO == "push":  # a pushing rank launches its strip whole, as a single grid does
        g = csph.csph_create(n, j1 - j0, c.dx, csph.params_from(c.params, tile_rows=TY))
    else:  # the send/recv rank's split launches (edge tile rows, interior), NCCL at 1 rank
        g = csph.csph_create_dist_rows(n, j1 - j0, c.dx,
                                       csph.params_from(c.params, tile_rows=TY, halo_push=0),
                                       0, 1, [0, j1 - j0], 0, csph.csph_make_nccl_id())
    g.set_state(*f)
    g.step(4)  # even: the timed steps start at parity 0, whose pair graph is captured here
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for rep in range(REPS):  # the steady state: the fastest of REPS timed regions (a rare
        e0.record(); g.step(steps); e1.record(); torch.cuda.synchronize()  # slow one is noted)
        ts.append(e0.elapsed_time(e1) / steps)
    g.destroy()
    if max(ts) > 1.2 * min(ts):
        print(f"  note: rows [{j0}, {j1}) timed {[round(t, 3) for t in ts]} ms/step", flush=True)
    return min(ts)


HALO_GBS = float(os.environ.get("HALO_GBS", "300"))
HALO_US = float(os.environ.get("HALO_US", "15"))
ALLRED_US = float(os.environ.get("ALLRED_US", "20"))
COMBINE_US = float(os.environ.get("COMBINE_US", "5"))
pitch = ((n + 4 + 3 + 4) + 31) // 32 * 32


HALO = os.environ.get("HALO", "push")


def comm_ms(rows, t_strip):
    """Exposed communication per step of a strip of `rows` rows (see the module doc)."""
    if HALO == "push":
        return COMBINE_US * 1e-3
    halo = 2 * 3 * 4 * pitch * 8 / (HALO_GBS * 1e9) * 1e3 + HALO_US * 1e-3
    interior = t_strip * max(0.0, 1.0 - 2 * 128 / rows)  # the interior launch's share
    return max(0.0, halo - interior) + ALLRED_US * 1e-3  # (the split launches are timed)


def report(N, kind, b, ts):
    tc = [t + comm_ms(b[r + 1] - b[r], t) for r, t in enumerate(ts)]
    tN, tNc = max(ts), max(tc)
    print(f"N={N} {kind:8s}: strips {[b[r + 1] - b[r] for r in range(N)]} ms "
          f"{[round(x, 3) for x in ts]} -> {c.cells / tN / 1e6:.1f} Gcell/s, "
          f"efficiency {t1 / (N * tN):.2f} (compute only); with modelled comm "
          f"{tNc:.3f} ms -> {c.cells / tNc / 1e6:.1f} Gcell/s, efficiency "
          f"{t1 / (N * tNc):.2f}", flush=True)


t1 = strip_ms(0, c.ny)
print(f"N=1: {t1:.3f} ms/step, {c.cells / t1 / 1e6:.1f} Gcell/s", flush=True)
for N in NS:
    for kind in KINDS:
        b = ([csph.csph_strip_rows(c.ny, N, r)[0] for r in range(N)] + [c.ny]) if kind == "even" \
            else csph.csph_balance_rows(c.ny, N, w)
        ts = [strip_ms(b[r], b[r + 1]) for r in range(N)]
        report(N, kind, b, ts)
        if kind != "balanced":
            continue
        # measured-time re-balancing: scale each strip's row weights by its
        # measured step time over the mean, balance again, measure again
        wm = w.copy()
        for it in range(REBAL):
            mean = sum(ts) / N
            for r in range(N):
                wm[b[r]:b[r + 1]] *= ts[r] / mean
            b = csph.csph_balance_rows(c.ny, N, wm)
            ts = [strip_ms(b[r], b[r + 1]) for r in range(N)]
            report(N, f"measured{it + 1}", b, ts)
