timeout 300 python -m pytest tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -1
for v in 3 4; do OSM_SPMV=$v timeout 300 python tools/cg_bench.py --timing --solves 1; done 2>&1 | cut -c1-560
OSM_UPD=1 timeout 300 python tools/cg_bench.py --timing --solves 1 2>&1 | cut -c1-560
for e in "OSM_SPMV=3" "OSM_SPMV=4" "OSM_UPD=1"; do env $e timeout 300 python tools/cg_bench.py --solves 3; done 2>&1
