timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 > gpurun_out/r01k_c5_vi_S8.log 2>&1; echo rc $?; tail -c 400 gpurun_out/r01k_c5_vi_S8.log
timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 --row-order 4 --spmv 5 > gpurun_out/r01k_c5_mf_S8.log 2>&1; echo rc $?; tail -c 400 gpurun_out/r01k_c5_mf_S8.log
timeout 300 python tools/cg_bench.py --solves 3 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['env'], [round(x,4) for x in d['seconds']])"
