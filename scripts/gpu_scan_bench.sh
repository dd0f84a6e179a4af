set -x
mkdir -p gpurun_out
timeout 900 python tools/alpha_scan.py C3 1e-3 2e-3 4e-3 8e-3 1.6e-2 3.2e-2 6.4e-2 --max-outer 400 2>&1 | tee gpurun_out/alpha_scan_C3.log
A=$(grep '^best' gpurun_out/alpha_scan_C3.log | python -c "import sys,json; print(json.loads(sys.stdin.read().split(' ',1)[1])['alpha'])")
timeout 900 python bench.py --alpha $A --steps 3 --warmup 3 > gpurun_out/bench1.json 2> gpurun_out/bench1.err; echo rc=$?
tail -5 gpurun_out/bench1.err; cat gpurun_out/bench1.json
