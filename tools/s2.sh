cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s2_pytest.txt
bash tools/ab_bench.sh variants/libcsph_base.so variants/libcsph_sq.so variants/libcsph_band.so variants/libcsph_bandu2.so variants/libcsph_band.so > gpurun_out/s2_ab.txt 2>&1
N=8192 timeout 600 python tools/ab.py variants/libcsph_sq.so variants/libcsph_band.so variants/libcsph_bandu2.so >> gpurun_out/s2_ab.txt 2>&1
