"""Dynamic SASS opcode mix of one kernel from an ncu source page (dev aid).
usage: python tools/sass_mix.py report.ncu-rep [cells_full_cost]"""
import csv, subprocess, sys, collections
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
cnt = collections.Counter(); thr = collections.Counter(); stall = collections.Counter()
for r in rows:
    if r and r[0] == "Address":
        hdr = r; iE = hdr.index("Instructions Executed"); iT = hdr.index("Thread Instructions Executed")
        iS = hdr.index("Warp Stall Sampling (All Samples)"); iSrc = hdr.index("Source"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    ins = r[iSrc].strip().split()
    if not ins:
        continue
    op = ins[1] if ins[0].startswith("@") else ins[0]
    base = op.split(".")[0]
    try:
        cnt[base] += int(r[iE] or 0); thr[base] += int(r[iT] or 0); stall[base] += int(r[iS] or 0)
    except ValueError:
        pass
tot = sum(cnt.values()); ts = sum(stall.values())
cells = float(sys.argv[2]) if len(sys.argv) > 2 else None
print(f"total warp inst {tot:.4g}")
for op, c in cnt.most_common(45):
    extra = f"  {thr[op] / cells:8.1f} thread-inst/cell" if cells else ""
    print(f"{op:10s} {c / tot * 100:5.1f}% inst  {stall[op] / ts * 100:5.1f}% stalls{extra}")
