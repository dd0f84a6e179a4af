timeout 900 python -m pytest tests/test_gpu_matrix_free.py tests/test_gpu_variants.py -x -q 2>&1 | tail -3
for env in "OSM_SORT=3 OSM_SPMV=6" "OSM_SORT=4 OSM_SPMV=6" "OSM_SORT=4 OSM_SPMV=5"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']], d['outer'], d['inner_total'])"
  env $env timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['us_per_launch'],2) for k,v in d['kernels'].items()}, round(d['spmv_gbs'],1))"
done
timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 --spmv 6 > gpurun_out/r01h_c5_viwide_S8.log 2>&1; echo rc $?; tail -c 700 gpurun_out/r01h_c5_viwide_S8.log
