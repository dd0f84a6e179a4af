mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r01t.json 2> gpurun_out/bench_r01t.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01t.err
timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --timing-steps 1 > gpurun_out/bench_small.json 2>&1 && \
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 6000 --csv --log-file gpurun_out/launches_bench_r01t.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --timing-steps 1 > gpurun_out/ncu_launch_bench.log 2>&1; echo "ncu1 rc=$?"
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
OSM_GROUPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv|k_cg_update|k_cg_dir" -s 300 -c 3 -o gpurun_out/prof_cg_r01t python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
