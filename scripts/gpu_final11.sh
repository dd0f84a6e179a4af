mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_r01p.json 2> gpurun_out/bench_r01p.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01p.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"; echo "smoke rc=$?"
