for E in "OSM_PERSIST=0" "OSM_PERSIST=2" "OSM_PERSIST=0" "OSM_PERSIST=2"; do
  env $E OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'])"
  env $E timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E', [round(x,4) for x in d['seconds']], d['h'])"
  env $E OSM_SORT=4 OSM_SPMV=5 OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$E MF', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)})"
done
