for L in "" expt/u2/libosm.so expt/u4/libosm.so; do
  OSM_LIB=$L OSM_GROUPS=1 timeout 300 python tools/cg_bench.py --solves 2 --timing | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', {k:round(v['us_per_launch'],2) for k,v in d['kernels'].items() if k in ('cg_spmv',)}, d['h'])"
  OSM_LIB=$L timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', [round(x,4) for x in d['seconds']])"
done
