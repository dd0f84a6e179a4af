for k in 2 3; do OSM_SORT=$k timeout 300 python tools/cg_bench.py --timing --solves 1 2>&1 | python -c "
import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); k=d['kernels']
print('sort', '$k', 'spmv us', round(k['cg_spmv']['us_per_launch'],2), 'pad', round(d['pad_frac'],4), 'h', d['h'])"; done
for k in 2 3; do OSM_SORT=$k timeout 300 python tools/cg_bench.py --solves 3 2>&1 | tail -1 | cut -c1-200; done
