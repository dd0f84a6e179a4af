OSM_LIB=expt/s4/libosm.so timeout 900 python -m pytest tests/test_gpu_variants.py -m gpu -x -q 2>&1 | tail -1
for L in "" expt/b/libosm.so expt/s2/libosm.so expt/s4/libosm.so; do
  OSM_LIB=$L OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'])"
  OSM_LIB=$L timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', [round(x,4) for x in d['seconds']])"
done
