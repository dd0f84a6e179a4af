mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r01s.json 2> gpurun_out/bench_r01s.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01s.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref_r01s.json 2> gpurun_out/bench_ref_r01s.err; echo "ref rc=$?"; cat gpurun_out/bench_ref_r01s.json | head -c 600
