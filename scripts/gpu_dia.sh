timeout 900 python -m pytest tests/test_gpu_matrix_free.py -m gpu -x -q 2>&1 | tail -3
for v in 9 5; do
  OSM_SORT=4 OSM_SPMV=$v OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv','cg_update','cg_dir')})"
  OSM_SORT=4 OSM_SPMV=$v timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', [round(x,4) for x in d['seconds']], d.get('active'))"
done
timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('6/order3', [round(x,4) for x in d['seconds']])"
