# 1-CTA kernel with compile-time-zero ablation tests: DeiT-S fc2 / proj and the step (vs r02h: fc2 65.1-67.0, proj 27.9-28.1)
for sh in "384 1536" "384 384"; do timeout 120 python scripts/time_spmm.py $sh 5 50432 tc; done
for rep in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('step', d['ms_per_step'], d['roofline']['frac'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"; done
timeout 900 python -m pytest -q -x tests/test_gpu_spmm.py -k "deit or window or toy or shapes" 2>&1 | tail -1
