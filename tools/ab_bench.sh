#!/bin/bash
# A/B of libcsph variants on the bench workload (C5 16384^2): bench.py per variant (dev aid).
# usage: tools/ab_bench.sh variants/libcsph_a.so variants/libcsph_b.so ...
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for v in "$@"; do
  CSPH_LIB_DEV=$(realpath $v) timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline --precision ${PREC:-64} 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['value'],2), 'Gcell/s', 'kernel ms', round(d['roofline']['kernel_ms_per_launch'],3), 'tiles', [round(x,3) for x in d['roofline']['hgs_tiles'].values()])"
done
