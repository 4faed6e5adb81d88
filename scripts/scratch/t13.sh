mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "opt_in" > gpurun_out/t13_tests.log 2>&1; echo "dec test $?"; tail -5 gpurun_out/t13_tests.log
VNM_DEC=1 timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "toy or token_tails or decode or slab or shapes" > gpurun_out/t13_tests2.log 2>&1; echo "dec suite $?"; tail -5 gpurun_out/t13_tests2.log
VNM_DEC=1 timeout 120 python /tmp/td.py 2>&1 | sed 's/^/dec: /'
VNM_DEC=1 timeout 200 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t13_dec.json 2> gpurun_out/t13_dec.err || tail -3 gpurun_out/t13_dec.err
python scripts/bench_summary.py gpurun_out/t13_dec.json
