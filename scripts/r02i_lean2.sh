# prune2 LEAN = 2 (no score / mask compiled out, tensor-core form kept) vs the general kernel, batched prune pass
for rep in 1 2; do for l in 1 0; do for w in llama_prefill deit_s llama_prefill_v128_m13 llama_mlp_m16; do
  VNM_PRUNE_LEAN2=$l timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('lean2=$l', '$w', d['detail']['prune_compress_batched_us'], d['ms_per_step'])"
done; done; done
timeout 900 python -m pytest -q -x tests/test_gpu_prune.py tests/test_gpu_window16.py tests/test_gpu_bounds.py 2>&1 | tail -1
