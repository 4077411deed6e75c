"""Executed thread-instructions per CUDA source line and per opcode class (dev aid).
usage: python tools/line_inst.py report.ncu-rep file.cu first_line last_line [cells]"""
import csv, subprocess, sys, collections
rep, fname, l0, l1 = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4])
cells = float(sys.argv[5]) if len(sys.argv) > 5 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None; cur = ""; key = None
per = collections.defaultdict(collections.Counter); src = {}
for r in rows:
    if r and r[0] == "File Path":
        cur = r[1].split("/")[-1]
    if r and r[0] == "Line No":
        hdr = r; iE = hdr.index("Thread Instructions Executed"); continue
    if hdr is None or len(r) < len(hdr):
        continue
    if r[0].isdigit():
        key = (cur, int(r[0])); src[key] = r[1][:100]; continue
    ins = r[3].strip().split() if len(r) > 3 else []
    if not ins or key is None or key[0] != fname or not (l0 <= key[1] <= l1):
        continue
    op = (ins[1] if ins[0].startswith("@") else ins[0]).split(".")[0]
    try:
        per[key][op] += int(r[iE] or 0)
    except ValueError:
        pass
tot = collections.Counter()
for k in sorted(per):
    c = per[k]; tot.update(c)
    print(f"{k[1]:4d} {sum(c.values())/cells:7.1f}  " + " ".join(f"{o}:{v/cells:.1f}" for o, v in c.most_common(6)) + f"   | {src[k][:60]}")
print("total", round(sum(tot.values()) / cells, 1), " ".join(f"{o}:{v/cells:.1f}" for o, v in tot.most_common(12)))
