OSM_TWO=1 timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -1
for C in "OSM_TWO=0" "OSM_TWO=1" "OSM_TWO=1 OSM_LIB=expt/m16/libosm.so" "OSM_TWO=1 OSM_LIB=expt/m10/libosm.so"; do
  env $C OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'])"
  env $C timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$C', [round(x,4) for x in d['seconds']], d['h'])"
done
