mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py -x -q 2>&1 | tail -2
python -c "
import os; os.environ['OSM_SPMV']='10'
import synth, paper_2112_03851_b200 as P
cfg=dict(synth.CONFIGS['C3']); o=P.setup(cfg, synth.density(cfg)); print('variant at C3:', o.spmv_variant() if hasattr(o,'spmv_variant') else '?')
" 2>&1 | tail -1
for k in 10 6 10 6; do
  OSM_SPMV=$k timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_v$k.json 2>gpurun_out/bench_v$k.err; python -c "
import json;d=json.load(open('gpurun_out/bench_v$k.json'));r=d['roofline'];kl=r['kernel_launches'];km=r['kernel_ms']
print('$k', r['kernel'], round(d['ms_per_step'],2), [round(km[x]/kl[x]*1e3,2) for x in ('cg_spmv','cg_update','cg_dir')], d['outer_iters'], d['inner_total'], round(r['frac'],3), round(d['roofline_cg_step']['frac'],3))"
done
