for env in "OSM_SORT=3" "OSM_SORT=5"; do
  env $env OSM_GROUPS=1 python tools/spmv_probe.py
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']], d['outer'], d['inner_total'], d['h'])"
done
OSM_SORT=5 OSM_SPMV=2 timeout 300 python tools/cg_bench.py --solves 1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], d['h'], d['inner_total'])"
