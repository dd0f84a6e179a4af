mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 600 python tools/c4_alpha_batch.py --B 64 --seq 4 > gpurun_out/r01f_c4_alpha_batch.json 2>&1; tail -c 600 gpurun_out/r01f_c4_alpha_batch.json
timeout 900 python tools/c4_cmaes.py --mode oo0_unsym --gens 12 2>&1 | tee gpurun_out/r01f_c4_cmaes.log | tail -3
