timeout 900 python -m pytest -q -x tests/test_gpu_spmm_batched.py tests/test_gpu_graph_replay.py 2>&1 | tail -3
for w in llama_decode llama_block_decode; do
for f in "" "--no-weights-ready"; do
timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines $f > gpurun_out/b_$w.json 2>gpurun_out/b_$w.err; echo "$w $f $?"; python scripts/bench_summary.py gpurun_out/b_$w.json 2>/dev/null | head -1
done; done
