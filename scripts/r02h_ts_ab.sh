# TS form (A in TMEM, NT = 256, one accumulator) vs the SS form (NT = 224, two accumulators), fast MMA loop, same box
for rep in 1 2 3; do for ts in 0 1; do
  VNM_TC3_TS=$ts timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ts=$ts step', d['ms_per_step'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
