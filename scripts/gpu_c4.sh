mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python tools/c4_cmaes.py --mode oo0_unsym --gens 12 2>&1 | tee gpurun_out/c4_cmaes_r01.log | tail -3
timeout 600 python tools/c4_alpha_batch.py > gpurun_out/c4_r01b.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/c4_r01b.json')); print({k:v for k,v in d.items() if k not in ('alphas','cost','iters')})"
