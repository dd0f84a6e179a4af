mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_batch.py -x -q 2>&1 | tail -2
for RB in 512 256 128; do for B in 64 32; do
OSM_BATCH_RB=$RB timeout 600 python tools/c4_alpha_batch.py --B $B --seq 1 > gpurun_out/c4_kb3_${RB}_$B.json 2>&1; python -c "import json; d=json.load(open('gpurun_out/c4_kb3_${RB}_$B.json')); print($RB, {k:round(v,3) for k,v in d.items() if k in ('B','batch_cost_seconds','batch_to_tol_seconds','sequential_seconds_per_candidate','batch_speedup_vs_sequential')})"
done; done
timeout 300 python tools/batch_profile.py --B 32 --outer 1 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:kb_ -c 300 --csv --log-file gpurun_out/batch_launches3.csv python tools/batch_profile.py --B 32 --outer 1 > /dev/null 2>&1; echo ncu rc $?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:kb_spmm -s 5 -c 1 -o gpurun_out/kb_spmm_full python tools/batch_profile.py --B 32 --outer 1 > /dev/null 2>&1; echo ncu2 rc $?
