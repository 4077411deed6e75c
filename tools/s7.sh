cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
CSPH_LIB_DEV=$(realpath variants/libcsph_mmg.so) timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7_mmg.json 2> gpurun_out/s7_mmg.err
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -5 > gpurun_out/s7_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/s7_bench.json 2> gpurun_out/s7_bench.err
timeout 300 python tools/graph_ab.py > gpurun_out/s7_graph.txt 2>&1
CSPH_LIB_DEV=$(realpath variants/libcsph_mmg.so) timeout 300 python tools/graph_ab.py >> gpurun_out/s7_graph.txt 2>&1
