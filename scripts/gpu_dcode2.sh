mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_variants.py tests/test_gpu_matrix_free.py -x -q 2>&1 | tail -3
for v in 1 0 1 0; do OSM_DCODE=$v timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_dcode$v.json 2>gpurun_out/bench_dcode$v.err; python -c "
import json;d=json.load(open('gpurun_out/bench_dcode$v.json'));r=d['roofline']
print('dcode=$v', round(d['ms_per_step'],2), r['kernel_ms']['cg_update']/r['kernel_launches']['cg_update']*1e3, r['kernel_ms']['cg_dir']/r['kernel_launches']['cg_dir']*1e3, d['outer_iters'], d['inner_total'], d['roofline_cg_step']['frac'], d['matrix_free']['time_to_tol_s'], d['matrix_free']['cg_kernels_us'])"; done
