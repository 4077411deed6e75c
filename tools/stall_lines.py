"""Aggregate ncu warp-stall samples and executed instructions per CUDA source line (dev aid).
usage: python tools/stall_lines.py report.ncu-rep [top]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
per = collections.Counter(); ins = collections.Counter(); src = {}; fname = ""
tot_s = tot_i = 0
for r in rows:
    if r and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r
        iS = hdr.index("Warp Stall Sampling (All Samples)")
        iE = hdr.index("Instructions Executed")
        continue
    if hdr is None or len(r) < len(hdr) or not r[0].isdigit():
        continue
    if r[2] != "-":  # sass rows carry addresses; cuda rows have '-'
        continue
    key = (fname, int(r[0]))
    s = int(r[iS] or 0); e = int(r[iE] or 0)
    per[key] += s; ins[key] += e; src[key] = r[1][:90]
    tot_s += s; tot_i += e
print(f"total samples {tot_s}, warp instructions {tot_i}")
for key, s in per.most_common(top):
    print(f"{s / tot_s * 100:5.1f}% stalls {ins[key] / max(tot_i, 1) * 100:5.1f}% inst  {key[0]}:{key[1]:<4d} {src[key]}")
