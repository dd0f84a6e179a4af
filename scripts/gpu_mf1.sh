mkdir -p gpurun_out
for env in "OSM_SORT=3 OSM_SPMV=4" "OSM_SORT=4 OSM_SPMV=5" "OSM_SORT=4 OSM_SPMV=2"; do
  env $env timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']], d['outer'], d['inner_total'])"
  env $env timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print({k:round(v['us_per_launch'],2) for k,v in d['kernels'].items()})"
done
OSM_SORT=4 OSM_SPMV=5 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_cg -s 300 -c 60 --csv --log-file gpurun_out/mf_launches.csv python tools/cg_bench.py --solves 1 > /dev/null 2>&1; echo ncu rc $?
OSM_SORT=4 OSM_SPMV=5 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cg_spmv -s 100 -c 1 -o gpurun_out/mf_spmv_full python tools/cg_bench.py --solves 1 > /dev/null 2>&1; echo ncu2 rc $?
