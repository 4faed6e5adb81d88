# tc2 with the specialised MMA loop: Llama prefill layers (T = 2048) and parity
for m in 5 8; do for sh in "11008 4096" "4096 11008" "4096 4096"; do timeout 120 python scripts/time_spmm.py $sh $m 2048 tc | sed "s/^/m=$m /"; done; done
VNM_TS_V=128 timeout 120 python scripts/time_spmm.py 11008 4096 13 2048 tc
timeout 900 python -m pytest -q -x tests/test_gpu_spmm.py tests/test_gpu_window16.py tests/test_gpu_timed_path.py -k "llama or window or pair or natural or m16 or timed or prefill" 2>&1 | tail -2
for w in llama_prefill llama_mlp_m8 llama_prefill_v128_m13 deit_b; do timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null > gpurun_out/r02h_bench_$w.json; python scripts/bench_summary.py gpurun_out/r02h_bench_$w.json | head -1; done
