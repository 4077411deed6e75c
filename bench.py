#!/usr/bin/env python3
"""Benchmark of the CSPH-TVD step (BASELINE.json metric: Gcell-updates/s of the fp64
step at 1/2/4/8 B200, and % of HBM peak).

  python bench.py [--gpus N --steps K --warmup W]            # our CUDA path
  python bench.py --impl reference [--steps K --warmup W]    # the CPU oracle (reference arm)
  torchrun --nproc-per-node N bench.py --gpus N ...          # N > 1: row strips over NCCL

Workload: C5, the synthetic river-floodplain flood with sediment
transport on a 16384 x 16384 grid (268 M cells, ~30 % wet, heterogeneous psi), the
largest configuration of BASELINE.json that fits one GPU.  N > 1 splits the same grid
into N row strips (strong scaling).  A "step" is one full CSPH-TVD step (K1..K8 + Eq.7 +
halo exchange).  Inputs (19 GB of state) are larger than the 126 MB L2, so no flush is
needed between steps.  Prints one JSON line from rank 0.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
# The input generator (synth/gen.c) is OpenMP: its threads must sleep, not spin, once a fill is
# done -- spinning threads starve the thread that launches the timed steps -- and under
# torchrun the ranks share the host's cores.
os.environ.setdefault("OMP_WAIT_POLICY", "PASSIVE")
if int(os.environ.get("WORLD_SIZE", "1")) > 1:
    os.environ.setdefault("OMP_NUM_THREADS",
                          str(max(1, (os.cpu_count() or 1) // int(os.environ["WORLD_SIZE"]))))

import numpy as np  # noqa: E402

METRIC = "Gcell-updates/s (fp64 CSPH-TVD step) at 1/2/4/8 B200; % of HBM peak"
UNIT = "Gcell-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", default="C5")
    ap.add_argument("--grid-n", "--n", dest="n", type=int, default=None,
                    help="override the grid size (n x n); spell it --grid-n under torchrun "
                         "(its parser swallows the ambiguous prefix --n)")
    ap.add_argument("--path", choices=["fused", "staged"], default="fused")
    ap.add_argument("--tile-rows", type=int, default=0)
    ap.add_argument("--partition", choices=["balanced", "even"], default="balanced",
                    help="N > 1 row strips: balanced by the initial wet cells per row "
                         "(csph_balance_rows, DESIGN.md 9) or the paper's even Ny_dev split")
    ap.add_argument("--halo", choices=["push", "nccl"], default="push",
                    help="N > 1: ghost rows written by the step kernel into the neighbours' "
                         "buffers over NVLink (CUDA IPC; DESIGN.md 9) or NCCL send/recv")
    ap.add_argument("--scaling", choices=["strong", "weak"], default="strong",
                    help="strong: the whole 16384^2 C5 grid split over N GPUs (default); "
                         "weak: rows [0, 2048 N) of the same C5 field, 2048 rows per GPU")
    ap.add_argument("--precision", type=int, choices=[64, 32], default=64,
                    help="32 = the NEXT-2 fp32 mode (not the headline metric)")
    ap.add_argument("--e2e-steps", type=int, default=100,
                    help="steps between host saves in the end-to-end run (P:131: 100-1000)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-intervals", type=int, default=3,
                    help="save intervals of the e2e_run measurement (1 GPU)")
    ap.add_argument("--cpu-crop", type=int, default=2048)
    ap.add_argument("--cpu-steps", type=int, default=15)
    ap.add_argument("--repeats", type=int, default=3,
                    help="timed regions of exactly --steps steps each; value = the median "
                         "(SURVEY 8(d): median of 3 runs)")
    ap.add_argument("--dist", action="store_true",
                    help="take the multi-GPU code path (torch.distributed + NCCL id broadcast + "
                         "csph_create_dist_rows) even with one rank (torchrun --nproc-per-node 1)")
    return ap.parse_args()


def host_info():
    """CPU model and core count of the box the oracle runs on."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    try:
        aff = len(os.sched_getaffinity(0))
    except AttributeError:
        aff = None
    return {"cpu_model": model, "nproc": os.cpu_count(), "affinity_cores": aff}


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md: 6.65 TB/s)"


def ncu_traffic(key: str):
    """Per-launch DRAM bytes of the dominant kernel from the committed ncu summary."""
    p = os.path.join(ROOT, "profiles", "ncu_summary.json")
    try:
        d = json.load(open(p))
        return d.get("kernels", {}).get(key)
    except Exception:
        pass
    return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled every 50 ms during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.proc = None
        self.rows = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)  # let the first sample land before the timed region
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc is None:
            return
        time.sleep(0.1)
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:
            self.proc.kill()
            out, _ = self.proc.communicate()
        for line in out.splitlines():
            r = [x.strip() for x in line.split(",")]
            if len(r) >= 7:
                self.rows.append(r)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        sm = [v for v in (num(r[1]) for r in self.rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in self.rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4)
                          if r[3 + k].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows)}


def cpu_baseline(cfg_name, n, crop, steps):
    """The oracle as it stands, single-threaded, on a centre crop of the workload run as
    its own walled domain."""
    import oracle
    import synth
    c = synth.config(cfg_name, n)
    j0 = (c.ny - crop) // 2
    i0 = (c.nx - crop) // 2
    f = synth.fill(c, j0, j0 + crop)
    f = [a[:, i0:i0 + crop].copy() for a in f]
    o = oracle.Oracle(crop, crop, c.dx, oracle.Params(**c.params))
    assert o.set_state(*f) == 0
    t = time.perf_counter()
    st, dt, _ = o.step(steps)
    el = time.perf_counter() - t
    return {"value": crop * crop * len(dt) / el / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": f"{cfg_name} {c.nx}x{c.ny} centre crop {crop}x{crop} as its own walled "
                      f"domain, {len(dt)} steps, {el:.1f} s, single thread (status {st})",
            "host": host_info()}


def workload_name(a, c, gen):
    """The `config.workload` string both arms print for the same run."""
    return ((f"{a.config} river-floodplain flood + sediment transport"
             if a.config == "C5" else a.config)
            + (f", rows [0, {c.ny}) of the {gen.nx}x{gen.ny} field (weak scaling, "
               f"2048 rows per GPU)" if a.scaling == "weak" else ""))


def run_reference(a, rank, world):
    if rank != 0:
        return
    import oracle
    import synth
    c = synth.config(a.config, a.n)
    crop = a.cpu_crop
    j0 = (c.ny - crop) // 2
    i0 = (c.nx - crop) // 2
    f = [x[:, i0:i0 + crop].copy() for x in synth.fill(c, j0, j0 + crop)]
    o = oracle.Oracle(crop, crop, c.dx, oracle.Params(**c.params))
    assert o.set_state(*f) == 0
    o.step(a.warmup)
    t = time.perf_counter()
    st, dt, _ = o.step(a.steps)
    el = time.perf_counter() - t
    v = crop * crop * len(dt) / el / 1e9
    cw = c  # our arm's domain: weak scaling runs rows [0, 2048 N) of the same field
    if a.scaling == "weak":
        cw = synth.Config(c.name, c.cfg, c.nx, min(c.ny, 2048 * world), c.dx, c.variant,
                          dict(c.params))
    sample = (f"each step = one oracle step on the {crop}x{crop} centre crop of {a.config} "
              f"{c.nx}x{c.ny} (own walled domain), single thread")
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus,
        "steps": a.steps, "warmup": a.warmup, "ms_per_step": el / max(len(dt), 1) * 1e3,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic",
        # the same workload as our arm's line (each timed step a bounded sample of it: one
        # oracle step on a centre crop, see cpu_baseline.sample)
        "config": {"workload": workload_name(a, cw, c), "grid": [cw.nx, cw.ny],
                   "cells": cw.nx * cw.ny, "dx_m": c.dx, "physics": c.params,
                   "sample": f"{crop}x{crop} centre crop, own walled domain"},
        "cpu_baseline": {"value": v, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": sample,
                         "host": host_info()},
        "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def strip_bounds(gen, ny, nx, world, rank, kind, device):
    """Row-strip bounds [0, ..., ny] for `world` ranks (identical on every rank).
    kind "even": the paper's Ny_dev split (csph_strip_rows).  kind "balanced": per-row cost
    of the fused kernel ~ wet cells (full-cost work) + 0.03 nx (dry rows, skipped tiles)
    of the initial state; each rank counts its even strip of the field
    `gen`, the counts are all-gathered and every rank runs csph_balance_rows on them."""
    from paper_2103_15196_b200 import csph
    if world == 1 and kind != "dist1":
        return [0, ny]
    kind = "balanced" if kind == "dist1" else kind
    bounds = [csph.csph_strip_rows(ny, world, r)[0] for r in range(world)] + [ny]
    if kind == "even":
        return bounds
    import torch
    import torch.distributed as dist
    import synth
    e0, e1 = bounds[rank], bounds[rank + 1]
    cnt = (synth.fill(gen, e0, e1)[0] > 1e-6).sum(axis=1).astype(np.float64)
    mx = max(bounds[r + 1] - bounds[r] for r in range(world))
    buf = torch.zeros(mx, dtype=torch.float64, device=device)
    buf[:e1 - e0] = torch.from_numpy(cnt)
    parts = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    w = np.concatenate([parts[r][:bounds[r + 1] - bounds[r]].cpu().numpy()
                        for r in range(world)]) + 0.03 * nx
    return csph.csph_balance_rows(ny, world, w)


def run_ours(a, rank, world, local):
    import torch
    import torch.distributed as dist

    import synth
    from paper_2103_15196_b200 import csph

    torch.cuda.set_device(local)
    distributed = world > 1 or a.dist
    if distributed:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    c = synth.config(a.config, a.n)
    # weak scaling: the domain is rows [0, 2048 N) of the same global field,
    # a walled sub-domain generated with the global coordinates
    gen = c
    if a.scaling == "weak":
        c = synth.Config(c.name, c.cfg, c.nx, min(c.ny, 2048 * world), c.dx, c.variant,
                         dict(c.params))
    path = csph.CSPH_PATH_FUSED if a.path == "fused" else csph.CSPH_PATH_STAGED
    p = csph.params_from(c.params, path=path, device=local, tile_rows=a.tile_rows,
                         precision=a.precision, halo_push=1 if a.halo == "push" else 0)
    bounds = strip_bounds(gen, c.ny, c.nx, world, rank,
                          "dist1" if (a.dist and world == 1 and a.partition == "balanced")
                          else a.partition, "cuda")
    j0, j1 = bounds[rank], bounds[rank + 1]
    wa, wb = max(0, j0 - 3), min(c.ny, j1 + 3)
    fields = synth.fill(gen, wa, wb)
    wet_local = float(np.count_nonzero(fields[0][j0 - wa:j1 - wa] > 1e-6))
    if distributed:
        idt = torch.zeros(csph.csph_nccl_id_bytes(), dtype=torch.uint8, device="cuda")
        if rank == 0:
            idt.copy_(torch.frombuffer(bytearray(csph.csph_make_nccl_id()), dtype=torch.uint8))
        dist.broadcast(idt, 0)
        g = csph.csph_create_dist_rows(c.nx, c.ny, c.dx, p, rank, world, bounds, local,
                                       bytes(idt.cpu().numpy().tobytes()))
        # peer memory: every rank maps the others' buffers through CUDA IPC, so
        # the step kernels write the ghost rows and the ctrl kernels combine the Eq.7 maxima
        # over NVLink (no send/recv, no edge split, no allreduce)
        if a.halo == "push" and world > 1:
            blob = torch.frombuffer(bytearray(g.ipc_export()), dtype=torch.uint8).cuda()
            blobs = [torch.empty_like(blob) for _ in range(world)]
            dist.all_gather(blobs, blob)
            nb = [bytes(x.cpu().numpy().tobytes()) for x in blobs]
            ok = torch.ones(1, device="cuda")
            try:
                g.ipc_link(nb)
            except csph.CsphError as e:
                print(f"rank {rank}: halo push unavailable ({e}); NCCL halos", file=sys.stderr)
                ok.zero_()
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() < 1:  # one transport for all ranks
                g.ipc_link(None)
                a.halo = "nccl"
    else:
        g = csph.csph_create(c.nx, c.ny, c.dx, p)
    stream = torch.cuda.current_stream()
    g.set_stream(stream.cuda_stream)
    g.set_state_rows(wa, wb, *fields)
    psi_field = not np.all(fields[4] == fields[4].flat[0])

    def barrier():
        if distributed:
            dist.barrier()

    def max_over_ranks(x: float) -> float:
        if not distributed:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def sum_over_ranks(x: float) -> float:
        if not distributed:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    # ---- warm-up, then `repeats` timed regions of exactly K steps each (median) ----
    g.step(a.warmup)
    torch.cuda.synchronize()
    barrier()
    g.profile(True)
    g.reset_tile_stats()
    runs = []
    with ClockSampler(local) as clk:
        for _ in range(max(1, a.repeats)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            barrier()
            e0.record(stream)
            g.step(a.steps)
            e1.record(stream)
            torch.cuda.synchronize()
            barrier()
            runs.append(max_over_ranks(e0.elapsed_time(e1)))
    ms = float(np.median(runs))
    launches = g.last_launch_count()
    tiles = g.tile_stats()
    kern_ms, kern_steps = g.get_profile()
    g.profile(False)
    cells = c.nx * c.ny
    value = cells * a.steps / (ms / 1e3) / 1e9
    t_sim, steps_done, _ = g.get_time()
    dtl, liml = g.get_dt_log(min(steps_done, 100000))
    wet = sum_over_ranks(wet_local) / cells

    # ---- roofline of the dominant kernel (the fused step kernel) ----
    peak, peak_src = peaks()
    es = 8 if a.precision == 64 else 4
    bpc = (9 if psi_field else 8) * es  # algorithmic bytes per cell-update
    own_cells = c.nx * (j1 - j0)
    kern_ms_per = kern_ms / max(kern_steps, 1)
    # HGS: marched tiles move bpc B/cell, identity-copied tiles read H, b (+W) and write
    # 4 fields, skipped tiles move nothing
    ntile = sum(tiles)
    # no HGS counters (the staged path): every cell's bytes move
    f_march, f_copy, f_skip = (x / ntile for x in tiles) if ntile else (1.0, 0.0, 0.0)
    bpc_copy = ((3 if psi_field else 2) + 4) * es
    bytes_per_step = own_cells * (bpc * f_march + bpc_copy * f_copy)
    achieved = bytes_per_step / (kern_ms_per / 1e3) / 1e9
    # the committed capture of the same kernel and precision (fp32: its own entry, else none)
    tr = ncu_traffic(("fused_step_kernel" + ("" if a.precision == 64 else "_fp32"))
                     if path == csph.CSPH_PATH_FUSED else "k7_fluxes")
    roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
            "frac": achieved / peak, "traffic": (tr or {}).get("dram_bytes_per_launch"),
            "kernel": "fused_step_kernel" if path == csph.CSPH_PATH_FUSED else "staged K1..K8",
            "algorithmic_bytes_per_cell": bpc,
            "algorithmic_bytes_per_launch": bytes_per_step,
            "hgs_tiles": {"marched": f_march, "identity_copy": f_copy, "skipped": f_skip},
            "kernel_ms_per_launch": kern_ms_per,
            "kernel_share_of_step": kern_ms_per / (ms / a.steps), "peak_source": peak_src,
            # SURVEY 8(d)'s dense count: bpc bytes for EVERY cell-update, HGS-skipped tiles
            # included -- bytes the launch did not have to move (reported beside, not as, the
            # achieved figure above)
            "dense_equivalent": {"achieved": own_cells * bpc / (kern_ms_per / 1e3) / 1e9,
                                 "frac": own_cells * bpc / (kern_ms_per / 1e3) / 1e9 / peak},
            # report the binding roof.  The fp64 step is not HBM-bound: ncu puts
            # DRAM at ~1.0x the algorithmic bytes and the fp64 pipe / issue slots ahead of it
            # (DESIGN.md 8), so the binding roof is roofline_fp64 below, when present.
            "binding_roof": "roofline_fp64" if a.precision == 64 else "issue (ALU)"}
    fp64 = None
    if tr and tr.get("fp64_inst_per_launch"):
        # fp64 pipe roof: 64 fp64 lanes/clk/SM x 148 SMs x the SM clock
        # sampled during the timed region; instruction count per launch from the
        # committed ncu capture of the same workload (scaled to this rank's cells).
        clk_mhz = None
        inst = tr["fp64_inst_per_launch"] * own_cells / cells
        fp64 = {"bound": "alu", "unit": "fp64 thread-inst/s",
                "inst_per_cell": inst / own_cells,
                "achieved": inst / (kern_ms_per / 1e3),
                "pipe_active_pct_ncu": tr.get("fp64_pipe_pct")}

    # ---- end to end through the public API: host (pinned) -> device -> host ----
    e2e = None
    if not a.no_e2e:
        pin = [torch.from_numpy(x).pin_memory() for x in fields]
        outp = [torch.empty((j1 - j0, c.nx), dtype=torch.float64).pin_memory() for _ in range(4)]
        pin_np = [x.numpy() for x in pin]
        E = a.e2e_steps
        torch.cuda.synchronize()
        barrier()
        t0 = time.perf_counter()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        g.set_state_rows(wa, wb, *pin_np)
        g.step(E)
        res = csph.lib().csph_get_state_rows(g.h, j0, j1, *[csph._p(x.numpy()) for x in outp])
        f1.record(stream)
        torch.cuda.synchronize()
        host_s = time.perf_counter() - t0
        barrier()
        assert res == 0
        ems = max_over_ranks(max(f0.elapsed_time(f1), host_s * 1e3))
        h2d = sum_over_ranks(5 * 8 * fields[0].size) / E
        d2h = sum_over_ranks(4 * 8 * c.nx * (j1 - j0)) / E
        e2e = {"value": cells * E / (ems / 1e3) / 1e9, "unit": UNIT,
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
               "how": f"csph_set_state_rows(pinned host) + csph_step({E}) + "
                      f"csph_get_state_rows(pinned host) per save interval (P:131)"}
        # The paper's run: Main uploads the state once, Solver steps, Save records
        # the state every E steps with the copies on their own CUDA stream -- here
        # csph_save_begin after each interval, overlapped with the next one's steps, and one
        # csph_save_wait at the end (single GPU: the Save arrays are global-layout).
        if world == 1 and a.e2e_intervals > 0:
            R = a.e2e_intervals
            torch.cuda.synchronize()
            f0.record(stream)
            t0 = time.perf_counter()
            g.set_state_rows(wa, wb, *pin_np)
            for _ in range(R):
                g.step(E)
                g.save_begin(*[x.numpy() for x in outp])
            g.save_wait()
            f1.record(stream)
            torch.cuda.synchronize()
            rms = max(f0.elapsed_time(f1), (time.perf_counter() - t0) * 1e3)
            e2e["run"] = {
                "value": cells * E * R / (rms / 1e3) / 1e9, "unit": UNIT,
                "h2d_bytes_per_step": 5 * 8 * fields[0].size / (E * R),
                "d2h_bytes_per_step": 4 * 8 * cells / E,
                "how": f"csph_set_state_rows(pinned host) once + {R} x (csph_step({E}) + "
                       f"csph_save_begin(pinned host), the device->host copy overlapping the "
                       f"next interval) + csph_save_wait (P:131 Main/Solver/Save)"}

    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu_baseline:
        cpu = cpu_baseline(a.config, a.n, min(a.cpu_crop, c.nx, c.ny), a.cpu_steps)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": ms / a.steps, "higher_is_better": True,
            "timed_runs_ms": runs,
            "scaling": a.scaling, "vs_baseline": None,
            "dtype": "f64" if a.precision == 64 else "f32", "data": "synthetic",
            "config": {
                "workload": workload_name(a, c, gen),
                "grid": [c.nx, c.ny], "cells": cells, "dx_m": c.dx, "wet_fraction": wet,
                "psi": "field" if psi_field else "uniform", "physics": c.params,
                "path": a.path, "parallelism": f"row strips x{world} ("
                + ("kernel-pushed halos over NVLink" if a.halo == "push" else "NCCL halos")
                + " + NCCL max-allreduce)"
                if distributed else "single GPU",
                "partition": {"kind": a.partition, "bounds": bounds} if distributed else None,
                "l2": "state (>= 19 GB) larger than the 126 MB L2; no flush needed",
                "tau_mean": float(np.mean(dtl)) if len(dtl) else None,
                "limiter_hist": np.bincount(liml, minlength=4).tolist() if len(liml) else None,
            },
            "roofline": roof,
            "gpu_launches": launches,
            "clocks": clk.summary(),
            "e2e": e2e,
            "cpu_baseline": cpu,
        }
        if fp64:
            ck = line["clocks"].get("sm_mhz") or 1965.0
            fp64["peak"] = 64 * 148 * ck * 1e6
            fp64["frac"] = fp64["achieved"] / fp64["peak"]
            fp64["peak_source"] = f"64 DFMA lanes/clk/SM x 148 SMs x {ck:.0f} MHz (sampled)"
            line["roofline_fp64"] = fp64
        print(json.dumps(line), flush=True)
    g.destroy()
    if distributed:
        dist.destroy_process_group()


def main():
    a = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != a.gpus and world > 1:
        a.gpus = world
    if a.impl == "reference":
        run_reference(a, rank, world)
        return
    if a.n is None and a.config == "C5":
        a.n = 16384
    run_ours(a, rank, world, local)


if __name__ == "__main__":
    main()
