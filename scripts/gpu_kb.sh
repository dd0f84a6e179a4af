mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -3
for B in 64 32 16; do
timeout 600 python tools/c4_alpha_batch.py --B $B > gpurun_out/c4_kb_$B.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/c4_kb_$B.json')); print({k:v for k,v in d.items() if k not in ('alphas','cost','iters')})"
done
