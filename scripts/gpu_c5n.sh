mkdir -p gpurun_out
timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 --row-order 4 --spmv 5 > gpurun_out/r01n_c5_mf_S8.log 2>&1; echo rc $?; tail -c 1200 gpurun_out/r01n_c5_mf_S8.log
timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 > gpurun_out/r01n_c5_vi_S8.log 2>&1; echo rc $?; tail -c 1200 gpurun_out/r01n_c5_vi_S8.log
