mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout 1500 python tools/alpha_scan.py C3 0.1:5e-4 1e-3:1e-3:2000:2000 1e-2:1e-3:2000:2000 1e-2:1e-3:500:500 1e-2:1e-3:8000:8000 1e-3:1e-4:2000:2000 3e-3:3e-4:4000:1000 1e-2:1e-4:8000:2000 3e-2:3e-4:2000:500 1e-3:1e-3:8000:8000 1e-4:1e-4:4000:4000 --max-outer 150 2>&1 | tee gpurun_out/oo2_scan_C3.log
