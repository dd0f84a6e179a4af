for env in "OSM_UPD=0" "OSM_UPD=1"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']])"
  env $env timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['us_per_launch'],2) for k,v in d['kernels'].items()})"
done
