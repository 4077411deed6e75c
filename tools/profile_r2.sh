#!/bin/bash
# Round-2 profiling session (one gpurun call): the bench line, the ncu launch list of the bench
# command, one --set full capture (with source) of the fp64 fused kernel in a timed step of the
# bench workload, and the fp32 bench line.  Outputs gpurun_out/${TAG}_*; summarise with
# tools/ncu_summarize.py into profiles/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
T=${TAG:-r2p}
timeout 600 python bench.py > gpurun_out/${T}_bench.json 2> gpurun_out/${T}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv \
    --log-file gpurun_out/${T}_launches.csv \
    python bench.py --steps 5 --warmup 3 --repeats 1 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fused_step -s 6 -c 1 \
    -o gpurun_out/${T}_fused_full -f \
    python bench.py --steps 2 --warmup 5 --repeats 1 --no-e2e --no-cpu-baseline > gpurun_out/${T}_ncu_full.log 2>&1
timeout 300 python bench.py --precision 32 --no-cpu-baseline --no-e2e > gpurun_out/${T}_bench32.json 2>&1
ls -la gpurun_out | grep ${T}_
