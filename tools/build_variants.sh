#!/bin/bash
# Build libcsph variants for A/B timing: tools/build_variants.sh name "-DFLAG=.." [name "-D.."]...
# Output: gpurun_out/../variants/libcsph_<name>.so (load with CSPH_LIB_DEV=path)
set -e
cd "$(dirname "$0")/.."
mkdir -p variants
while [ $# -gt 0 ]; do
  name=$1; flags=$2; shift 2
  python - "$name" "$flags" <<'PY'
import sys, subprocess
sys.path.insert(0, ".")
from paper_2103_15196_b200 import build
cmd = build.nvcc_cmd("variants/libcsph_%s.so" % sys.argv[1])
cmd[1:1] = sys.argv[2].split()
r = subprocess.run(cmd, capture_output=True, text=True)
if r.returncode:
    print(r.stderr[-2000:]); sys.exit(1)
import re
m = re.findall(r"Compiling entry function '(\S*IdLi128ELb1ELi8ELi3ELi3ELb0E\S*)'.*?Used (\d+) registers", r.stderr, re.S)
print(sys.argv[1], "regs", [x[1] for x in m][:1])
PY
done
