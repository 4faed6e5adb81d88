# tc3 epilogue: shared-memory reads hoisted before the global stores (new) vs the previous HEAD build, DeiT-S step
for rep in 1 2 3; do for lib in prev new; do
  if [ $lib = prev ]; then export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_prev.so; else unset VNM_LIB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib step', d['ms_per_step'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
unset VNM_LIB
timeout 900 python -m pytest -q -x tests/test_gpu_spmm.py tests/test_gpu_timed_path.py tests/test_gpu_bounds.py -k "deit or pair_resident or window or bench_step or writes_only" 2>&1 | tail -1
