# TS form with A stored into TMEM by the epilogue warps (deeper X^T ring) vs the SS default: parity, then the DeiT-S step
timeout 600 python -m pytest -q -x tests/test_gpu_tc3_ts.py 2>&1 | tail -2
VNM_TC3_TS=1 VNM_SPMM_TRACE=1 timeout 120 python scripts/trace_spmm.py 1152 384 5 50432 64 tc 2>&1 | grep "^tc3" | tail -1
for rep in 1 2 3; do for ts in 0 1; do
  VNM_TC3_TS=$ts timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('ts=$ts step', d['ms_per_step'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
