mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/bench_r01c.json 2> gpurun_out/bench_r01c.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01c.err
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01c.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv|k_cg_update|k_cg_dir" -s 300 -c 3 -o gpurun_out/prof_cg_r01c python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
