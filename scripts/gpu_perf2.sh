mkdir -p gpurun_out
timeout 300 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for sg in 1024 4096 8192 32768; do OSM_SIGMA=$sg timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | tee gpurun_out/perf2_timing.log
for g in 0 1; do OSM_NO_GRAPH=$g timeout 300 python tools/cg_bench.py --solves 2; done 2>&1 | tee gpurun_out/perf2_graph.log
