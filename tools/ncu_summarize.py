"""Summarise ncu reports / launch lists into small JSON/CSV files for profiles/.

  python tools/ncu_summarize.py full  <report.ncu-rep> <cells> <out.json>
  python tools/ncu_summarize.py launches <launches.csv> <out.csv>
"""
import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

KEYS = {
    "time_ms": "gpu__time_duration.sum",
    "dram_read_bytes": "dram__bytes_read.sum",
    "dram_write_bytes": "dram__bytes_write.sum",
    "inst_executed": "smsp__inst_executed.sum",
    "fp64_pipe_active_pct": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "issue_active_pct": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "warps_active_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "registers": "launch__registers_per_thread",
    "smem_per_block_kb": "launch__shared_mem_per_block",
    "grid": "launch__grid_size",
    "block": "launch__block_size",
    "l2_hit_pct": "lts__t_sector_hit_rate.pct",
    "sm_clock_ghz": "sm__cycles_elapsed.avg.per_second",
    "stall_wait": "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "stall_barrier": "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "stall_short_sb": "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "stall_long_sb": "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "stall_branch": "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "stall_math": "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
}
UNIT_SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0, "ms": 1.0, "us": 1e-3,
              "usecond": 1e-3, "msecond": 1.0, "nsecond": 1e-6, "ns": 1e-6}


def full(rep, cells, out):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    res = {"report": rep.split("/")[-1], "cells": cells, "kernels": {}}
    for vals in rows[2:]:
        d = dict(zip(hdr, vals))
        u = dict(zip(hdr, units))
        name = d.get("Kernel Name", "?")
        k = {}
        for short, key in KEYS.items():
            v = d.get(key)
            if v in (None, ""):
                continue
            try:
                x = float(v.replace(",", ""))
            except ValueError:
                continue
            sc = UNIT_SCALE.get(u.get(key, ""), 1.0)
            if short.endswith("bytes"):
                x *= sc
            if short == "time_ms":
                x *= sc
            k[short] = x
        if "dram_read_bytes" in k:
            k["dram_bytes_per_launch"] = k["dram_read_bytes"] + k["dram_write_bytes"]
            k["dram_bytes_per_cell"] = k["dram_bytes_per_launch"] / cells
        if "inst_executed" in k:
            k["thread_inst_per_cell"] = k["inst_executed"] * 32 / cells
        res["kernels"][name] = k
    # fp64-pipe instruction counts from the SASS page (executed warp instructions x 32)
    sass = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    lines = list(csv.reader(io.StringIO(sass)))
    cur = None
    fp64 = defaultdict(int)
    for r in lines:
        if len(r) >= 2 and r[0] == "Kernel Name":
            cur = r[1]
            continue
        if len(r) < 6 or r[0] == "Address" or cur is None:
            continue
        src = r[1].strip()
        op = src.split()[0] if src else ""
        if op.startswith("@"):
            op = src.split()[1] if len(src.split()) > 1 else ""
        try:
            ex = int(r[5] or 0)
        except ValueError:
            continue
        if op.split(".")[0] in ("DADD", "DMUL", "DFMA", "DSETP", "DMNMX"):
            fp64[cur] += ex
    for name, k in res["kernels"].items():
        for kn, n in fp64.items():
            if kn.split("(")[0].split("::")[-1][:20] in name:
                k["fp64_inst_per_launch"] = n * 32
                k["fp64_inst_per_cell"] = n * 32 / cells
    json.dump(res, open(out, "w"), indent=1)
    print(json.dumps(res, indent=1))


def launches(path, out):
    txt = open(path).read()
    i = txt.find('"ID"')
    rows = list(csv.DictReader(io.StringIO(txt[i:])))
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"].replace(",", ""))
        sc = UNIT_SCALE.get(r.get("Metric Unit", ""), 1.0)
        name = r["Kernel Name"].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += v * sc
    tot = sum(a[1] for a in agg.values())
    # kernels of csph_set_state (input validation, W, initial maxima, ghosts, tiling) run
    # once per upload, outside the timed steps
    setup = ("validate", "w_from_psi", "maxima", "mirror", "init_ctrl", "wet_blocks", "to_f32")
    step_tot = sum(a[1] for k, a in agg.items() if not any(x in k for x in setup))
    with open(out, "w") as f:
        f.write("kernel,launches,total_ms_cold,share,share_of_steps\n")
        for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
            st = "" if any(x in k for x in setup) else f"{t / step_tot:.4f}"
            f.write(f"{k},{n},{t:.4f},{t / tot:.4f},{st}\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "full":
        full(sys.argv[2], float(sys.argv[3]), sys.argv[4])
    else:
        launches(sys.argv[2], sys.argv[3])
