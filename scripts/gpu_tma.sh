mkdir -p gpurun_out
OSM_SPMV=1 timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
OSM_SPMV=0 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
for v in 0 1; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | tee gpurun_out/tma_timing.log
for v in 0 1; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 2; done 2>&1 | tee gpurun_out/tma_solve.log
timeout 900 python tools/alpha_scan.py C3 1e-3:1e-4:2000:2000 5e-4:1e-4:2000:2000 2e-3:1e-4:2000:2000 1e-3:5e-5:2000:2000 1e-3:2e-4:2000:2000 1e-3:1e-4:3000:1000 1e-3:1e-4:1500:1500 1e-3:1e-4:3000:3000 3e-3:3e-4:4000:1000 --max-outer 100 2>&1 | tee gpurun_out/oo2_scan2_C3.log
