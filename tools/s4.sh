cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/s4_bench.json 2> gpurun_out/s4_bench.err
PREC=32 bash tools/ab_bench.sh variants/libcsph_f32m3.so variants/libcsph_f32m4.so variants/libcsph_f32m5.so > gpurun_out/s4_ab32.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_fp32.py -q -x 2>&1 | tail -3 > gpurun_out/s4_pytest32.txt
