mkdir -p gpurun_out
OSM_GROUPS=1 timeout 600 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --timing-steps 1 > gpurun_out/bench_small_g1.json 2>&1 && \
OSM_GROUPS=1 timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -s 3000 -c 6000 --csv --log-file gpurun_out/launches_bench_r01o_g1.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 1 --timing-steps 1 > gpurun_out/ncu_launch_bench_g1.log 2>&1; echo "ncu rc=$?"
