mkdir -p gpurun_out
timeout 300 python scripts/sanitize_cases.py > gpurun_out/r02_san_plain.log 2>&1 && timeout 1500 compute-sanitizer --tool memcheck --print-limit 50 python scripts/sanitize_cases.py > gpurun_out/r02_sanitizer_memcheck.log 2>&1; echo "memcheck exit $?"; tail -15 gpurun_out/r02_sanitizer_memcheck.log
