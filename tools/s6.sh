cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s6_pytest.txt
bash tools/ab_bench.sh variants/libcsph_hllD.so variants/libcsph_mmg.so variants/libcsph_hllD.so variants/libcsph_mmg.so > gpurun_out/s6_ab.txt 2>&1
N=8192 timeout 600 python tools/ab.py variants/libcsph_hllD.so variants/libcsph_mmg.so >> gpurun_out/s6_ab.txt 2>&1
for n in 1024 2048; do for g in 0 1; do CSPH_NO_GRAPHS=$([ $g = 1 ] && echo 1) timeout 300 python bench.py --config C2 --n $n --steps 200 --warmup 5 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C2 $n nograph=$g', round(d['value'],2), d['ms_per_step'])" >> gpurun_out/s6_ab.txt; done; done
