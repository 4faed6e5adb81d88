# tc3 epilogue releasing the accumulator before its stores (two accumulators): libvnm_early.so vs HEAD, DeiT-S step
for rep in 1 2 3; do for lib in head early; do
  if [ $lib = early ]; then export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_early.so; else unset VNM_LIB; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib step', d['ms_per_step'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_early.so
timeout 600 python -m pytest -q -x tests/test_gpu_spmm.py tests/test_gpu_timed_path.py -k "deit or pair_resident or window or bench_step" 2>&1 | tail -1
