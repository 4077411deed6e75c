cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s8_pytest.txt
timeout 600 python bench.py > gpurun_out/s8_bench.json 2> gpurun_out/s8_bench.err
for ty in 64 96 128 192; do timeout 300 python bench.py --tile-rows $ty --steps 20 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TY $ty', round(d['value'],2), [round(x,3) for x in d['roofline']['hgs_tiles'].values()])" >> gpurun_out/s8_ab.txt; done
bash tools/ab_bench.sh variants/libcsph_cur.so variants/libcsph_cur2u.so variants/libcsph_cur.so variants/libcsph_cur2u.so >> gpurun_out/s8_ab.txt 2>&1
timeout 300 python tools/graph_ab.py >> gpurun_out/s8_ab.txt 2>&1
