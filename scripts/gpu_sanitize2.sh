mkdir -p gpurun_out
timeout 300 python tools/sanitize_case.py > gpurun_out/sanitize_plain.log 2>&1; echo "plain rc=$?"; tail -3 gpurun_out/sanitize_plain.log
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --print-limit 20 python tools/sanitize_case.py > gpurun_out/r01n_memcheck.log 2>&1; echo "memcheck rc=$?"; tail -5 gpurun_out/r01n_memcheck.log
