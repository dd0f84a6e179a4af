mkdir -p gpurun_out
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv
timeout 900 python bench.py > gpurun_out/bench_r01.json 2> gpurun_out/bench_r01.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_r01.err; cat gpurun_out/bench_r01.json
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && cat gpurun_out/prof_plain.log && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r01.csv python tools/profile_step.py > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_cg_spmv -s 200 -c 2 -o gpurun_out/prof_spmv_r01 python tools/profile_step.py > gpurun_out/ncu_full.log 2>&1; echo "ncu2 rc=$?"
tail -3 gpurun_out/ncu_full.log
