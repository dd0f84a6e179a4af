mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
for g in 4 8 4 8; do OSM_GROUPS=$g timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_g$g.json 2>/dev/null; python -c "
import json;d=json.load(open('gpurun_out/bench_g$g.json'));print('groups=$g', round(d['ms_per_step'],2))"; done
