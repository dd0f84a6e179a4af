timeout 300 python tools/mf_window_check.py
for env in "OSM_SORT=4 OSM_SPMV=5" "OSM_SORT=4 OSM_SPMV=8"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']])"
  env $env OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['us_per_launch'],2) for k,v in d['kernels'].items()})"
done
