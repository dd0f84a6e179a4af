mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for v in 2 3; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | cut -c1-800 | tee gpurun_out/vi_timing.log
for v in 2 3; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 3; done 2>&1 | tee gpurun_out/vi_solve.log
