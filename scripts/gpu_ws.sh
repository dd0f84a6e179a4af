mkdir -p gpurun_out
OSM_SPMV=1 timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -2
for v in 0 1; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | tee gpurun_out/ws_timing.log
for v in 0 1; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 2; done 2>&1 | tee gpurun_out/ws_solve.log
