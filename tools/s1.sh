cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s1_pytest.txt
timeout 300 ./tools/fp64probe > gpurun_out/s1_probe.txt 2>&1
N=8192 timeout 600 python tools/ab.py variants/libcsph_base.so variants/libcsph_sq.so variants/libcsph_squ2.so variants/libcsph_sqg1.so variants/libcsph_base.so variants/libcsph_sq.so > gpurun_out/s1_ab.txt 2>&1
timeout 300 python bench.py --precision 32 --no-cpu-baseline --no-e2e > gpurun_out/s1_bench32.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fused_step -s 6 -c 1 -o gpurun_out/s1_sq -f python bench.py --steps 2 --warmup 5 --no-e2e --no-cpu-baseline > gpurun_out/s1_ncu.log 2>&1
ls gpurun_out
