mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
BASE=$PWD/paper_2112_03851_b200/_exp/libosm_base.so
for k in vt8 vt4 vt8 vt4; do
  if [ $k = vt4 ]; then export OSM_LIB=$BASE; else unset OSM_LIB; fi
  timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$k.json 2>gpurun_out/bench_$k.err; python -c "
import json;d=json.load(open('gpurun_out/bench_$k.json'));r=d['roofline'];kl=r['kernel_launches'];km=r['kernel_ms']
print('$k', round(d['ms_per_step'],2), [round(km[x]/kl[x]*1e3,2) for x in ('cg_spmv','cg_update','cg_dir')], d['outer_iters'], d['inner_total'], d['matrix_free']['time_to_tol_s'])"
done
