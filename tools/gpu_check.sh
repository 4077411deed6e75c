#!/bin/bash
# One GPU session: parity tests, bench, ncu launch list and a full capture of the top kernel.
set -x
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt
python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 1 --no-e2e --no-cpu-baseline > gpurun_out/bench_ncu_launch.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_step -s 6 -c 1 \
    -o gpurun_out/prof_fused -f python bench.py --steps 2 --warmup 5 --no-e2e --no-cpu-baseline \
    > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
