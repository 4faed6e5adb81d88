mkdir -p gpurun_out
timeout 900 python -m pytest -q -x tests/test_gpu_graph_replay.py tests/test_gpu_spmm.py tests/test_gpu_bounds.py 2>&1 | tail -3
VNM_SPMM_TRACE=2 timeout 120 python scripts/trace_spmm.py 11008 4096 5 16 > gpurun_out/r02c_trace_up_mb2b.txt 2>&1; echo "trace exit $?"
for s in "4096 4096 5 16" "11008 4096 5 16" "4096 11008 5 16" "11008 4096 8 16" "4096 11008 8 16" "11008 4096 5 1" "11008 4096 5 32"; do
timeout 120 python scripts/time_spmm.py $s 2>&1 | tail -1
done
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b_dec.json 2>gpurun_out/b_dec.err; python scripts/bench_summary.py gpurun_out/b_dec.json
