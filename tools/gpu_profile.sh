#!/bin/bash
# Profiling session for profiles/: bench line, ncu launch list of the bench command,
# one ncu --set full capture of the dominant kernel (the fused step kernel).
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-r01}
python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${TAG}_launches.csv \
    python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_step -s 3 -c 1 \
    -o gpurun_out/${TAG}_fused_full -f \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu --set full --clock-control none -k regex:"k7_fluxes|k2_forces|k8_update" -s 3 -c 3 \
    -o gpurun_out/${TAG}_staged_full -f \
    python bench.py --path staged --steps 1 --warmup 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out | tail -8
