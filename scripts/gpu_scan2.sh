mkdir -p gpurun_out
timeout 1200 python tools/alpha_scan.py C3 5e-3 7e-3 1e-2 1.2e-2 1.6e-2:4e-3 3.2e-2:2e-3 6.4e-2:1e-3 4e-3:1.6e-2 2e-3:3.2e-2 1e-1:1e-3 --max-outer 120 2>&1 | tee gpurun_out/alpha_scan2_C3.log
