cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s5_pytest.txt
bash tools/ab_bench.sh variants/libcsph_band.so variants/libcsph_hllD.so variants/libcsph_band.so variants/libcsph_hllD.so > gpurun_out/s5_ab.txt 2>&1
N=8192 timeout 600 python tools/ab.py variants/libcsph_band.so variants/libcsph_hllD.so >> gpurun_out/s5_ab.txt 2>&1
