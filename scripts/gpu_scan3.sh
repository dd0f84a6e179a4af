mkdir -p gpurun_out
timeout 1200 python tools/alpha_scan.py C3 1e-1:1e-3 2e-1:1e-3 4e-1:1e-3 1e-1:5e-4 2e-1:5e-4 4e-1:5e-4 1e-1:2e-3 2e-1:2e-3 1:1e-3 2e-1:2.5e-4 --max-outer 300 2>&1 | tee gpurun_out/alpha_scan3_C3.log
