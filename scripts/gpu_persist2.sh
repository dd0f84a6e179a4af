OSM_PERSIST=1 timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -1
for E in "OSM_PERSIST=0" "OSM_PERSIST=1"; do
  env $E OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'])"
  env $E OSM_SORT=4 OSM_SPMV=5 OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E MF', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)})"
done
