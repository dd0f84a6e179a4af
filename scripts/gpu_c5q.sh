mkdir -p gpurun_out
for v in 1 0; do
OSM_DCODE=$v timeout 900 python tools/c5_probe.py 2e-4:5e-5:700:300 --nsub 8 > gpurun_out/r01q_c5_vi_S8_dcode$v.log 2>&1; echo rc $?; tail -c 420 gpurun_out/r01q_c5_vi_S8_dcode$v.log
done
