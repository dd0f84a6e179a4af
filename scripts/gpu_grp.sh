timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py tests/test_gpu_nccl_path.py tests/test_gpu_matrix_free.py -x -q 2>&1 | tail -2
for env in "OSM_GROUPS=4" "OSM_GROUPS=8" "OSM_GROUPS=4" "OSM_GROUPS=8"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']], d['outer'], d['inner_total'], d['h'])"
done
