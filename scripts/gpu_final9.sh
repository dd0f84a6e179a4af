mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 900 python bench.py > gpurun_out/bench_r01n.json 2> gpurun_out/bench_r01n.err; echo "bench rc=$?"; tail -2 gpurun_out/bench_r01n.err
OSM_SORT=4 OSM_SPMV=5 timeout 300 python tools/profile_step.py > gpurun_out/prof_plain_mf.log 2>&1 && \
OSM_SORT=4 OSM_SPMV=5 OSM_GROUPS=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv|k_cg_update|k_cg_dir" -s 300 -c 3 -o gpurun_out/prof_cg_r01n_mf python tools/profile_step.py > gpurun_out/ncu_full_mf.log 2>&1; echo "ncu rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
