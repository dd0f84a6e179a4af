#!/bin/bash
# One GPU session of the round's measurements (run under gpurun from the repo root):
#   GPU test suite, bench.py (the driver's default invocation), the bench's ncu launch list, and ncu
#   --set full captures of the CG kernels of the default path (brick SpMV k_cg_spmv_kuhn, update,
#   direction; single stream) and of the 3-byte value-indexed SELL SpMV (variant 10, row order 3).
# Outputs land in gpurun_out/<tag>_*; summaries are copied to profiles/ by hand.
tag=${1:-r02}
mkdir -p gpurun_out
python -m pytest tests -q -m gpu > gpurun_out/${tag}_gputests.log 2>&1; echo "rc=$?" >> gpurun_out/${tag}_gputests.log
python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc=$?" >> gpurun_out/${tag}_bench.err
# launch list of a short bench run (cold, serialised: shares, not absolutes)
python bench.py --steps 2 --warmup 1 --no-c5 --no-cpu-baseline --no-alt-spmv > gpurun_out/${tag}_plain.log 2>&1 &&
  ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/${tag}_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-c5 --no-cpu-baseline --no-alt-spmv > gpurun_out/${tag}_ncu_launch.log 2>&1
# full captures: one launch each of the SpMV / k_cg_update / k_cg_dir over all 8 C3 subdomains
python tools/cg_bench.py --solves 1 --timing --no-warm > gpurun_out/${tag}_cg_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"k_cg_(spmv_kuhn|spmv_kuhn_fused|update|dir)($|<)" -s 30 -c 3 \
    -o gpurun_out/${tag}_cg python tools/cg_bench.py --solves 1 --timing --no-warm > gpurun_out/${tag}_ncu_cg.log 2>&1
python tools/cg_bench.py --solves 1 --timing --no-warm --row-order 3 --spmv 10 > gpurun_out/${tag}_sell_plain.log 2>&1 &&
  ncu --set full --clock-control none --import-source on -k regex:"k_cg_spmv" -s 20 -c 1 \
    -o gpurun_out/${tag}_sell python tools/cg_bench.py --solves 1 --timing --no-warm --row-order 3 --spmv 10 \
    > gpurun_out/${tag}_ncu_sell.log 2>&1
echo done
