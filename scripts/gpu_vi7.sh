for env in "OSM_SORT=3 OSM_SPMV=6" "OSM_SORT=3 OSM_SPMV=4"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']], d['outer'], d['inner_total'])"
  env $env timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['us_per_launch'],2) for k,v in d['kernels'].items()})"
done
timeout 600 python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -2
