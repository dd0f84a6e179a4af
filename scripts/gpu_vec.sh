timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_batch.py -m gpu -x -q 2>&1 | tail -2
for v in 0 2; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | cut -c1-700
for v in 0 2; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 3; done 2>&1
