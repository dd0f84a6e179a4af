mkdir -p gpurun_out
for v in 2 4 3 2 4 3; do OSM_VT=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_vt$v.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_vt$v.json'));r=d['roofline'];kl=r['kernel_launches'];km=r['kernel_ms']
print('vt=$v', round(d['ms_per_step'],2), [round(km[x]/kl[x]*1e3,2) for x in ('cg_spmv','cg_update','cg_dir')], d['inner_total'])"; done
