mkdir -p gpurun_out
timeout 300 python tools/profile_step.py > gpurun_out/prof_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv" -s 100 -c 2 -o gpurun_out/prof_vi python tools/profile_step.py > gpurun_out/ncu_vi.log 2>&1; echo "ncu rc=$?"
