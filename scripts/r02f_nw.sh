# prune2 at V = 128: one 16-warp CTA per SM vs one 8-warp CTA (shared memory allows one either way)
for nw in 8 16; do for w in llama_prefill_v128_m13 llama_prefill_v128_m5 llama_decode_v128_m13 llama_decode_v128_m8; do
  VNM_PRUNE_NW=$nw timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('nw=$nw', '$w', d['detail']['prune_compress_batched_us'], d['ms_per_step'])"
done; done
timeout 900 python -m pytest -q -x tests/test_gpu_prune.py -k "128 or m9_to_16 or llama or window" 2>&1 | tail -2
