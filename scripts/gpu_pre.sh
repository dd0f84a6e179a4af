timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_matrix_free.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for L in "" expt/b/libosm.so "" expt/b/libosm.so; do
  OSM_LIB=$L OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv','cg_update','cg_dir')})"
  OSM_LIB=$L timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', [round(x,4) for x in d['seconds']])"
  OSM_LIB=$L OSM_SORT=4 OSM_SPMV=5 timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L MF', [round(x,4) for x in d['seconds']])"
done
