#!/bin/bash
# ncu --set full captures of the fused kernel on all-wet and C5 (N=8192) for source-level
# stall analysis (dev aid).  TAG names the outputs in gpurun_out/.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${TAG:-p}
for c in all-wet C5; do
  ONLY=$c TYS=128 STEPS=1 ncu --set full --clock-control none --import-source on -k regex:fused_step -s 2 -c 1 \
    -o gpurun_out/${TAG}_${c} -f python tools/costs.py > gpurun_out/${TAG}_${c}.log 2>&1
done
ls -la gpurun_out | grep ${TAG}_
