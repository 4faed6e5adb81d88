# DeiT prune pass: 16-warp CTAs (one tile each) up to k x 148 tiles (VNM_PRUNE_SMALL=k) vs 8-warp CTAs
for k in 1 2 3; do for w in deit_s deit_b; do
  VNM_PRUNE_SMALL=$k timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('k=$k', '$w', d['detail']['prune_compress_batched_us'], d['ms_per_step'])"
done; done
