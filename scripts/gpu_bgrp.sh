timeout 600 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -1
for G in 1 2; do
OSM_GROUPS=$G timeout 600 python tools/c4_alpha_batch.py --B 64 --seq 1 > gpurun_out/c4_g$G.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/c4_g$G.json')); print($G, {k:round(v,3) for k,v in d.items() if k in ('B','batch_cost_seconds','batch_to_tol_seconds','inner_total')})"
OSM_GROUPS=$G timeout 600 python tools/c4_alpha_batch.py --B 32 --seq 1 > gpurun_out/c4_g${G}_32.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/c4_g${G}_32.json')); print($G, {k:round(v,3) for k,v in d.items() if k in ('B','batch_cost_seconds','batch_to_tol_seconds','inner_total')})"
done
