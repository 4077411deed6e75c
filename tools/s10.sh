cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
bash tools/ab_bench.sh variants/libcsph_u2cur.so variants/libcsph_yd1.so variants/libcsph_yd.so variants/libcsph_u2cur.so variants/libcsph_yd1.so > gpurun_out/s10_ab.txt 2>&1
N=8192 timeout 600 python tools/ab.py variants/libcsph_u2cur.so variants/libcsph_yd1.so variants/libcsph_yd.so >> gpurun_out/s10_ab.txt 2>&1
timeout 600 python bench.py > gpurun_out/s10_bench.json 2> gpurun_out/s10_bench.err
