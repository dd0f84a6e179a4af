mkdir -p gpurun_out
timeout 300 python tools/batch_profile.py --B 32 --outer 1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:kb_spmm -s 5 -c 1 -o gpurun_out/kb_spmm_full10 python tools/batch_profile.py --B 32 --outer 1 > /dev/null 2>&1; echo ncu2 rc $?
