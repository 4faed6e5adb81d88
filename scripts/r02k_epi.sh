# tc3 with 8 (HEAD) / 12 / 16 epilogue warps now that the MMA loop is fast, DeiT-S step
for rep in 1 2; do for lib in head epi12 epi16; do
  if [ $lib = head ]; then unset VNM_LIB; else export VNM_LIB=$PWD/paper_2410_16135_b200/libvnm_$lib.so; fi
  timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$lib step', d['ms_per_step'], [l['spmm_us'] for l in d['detail']['layers']], d['clocks']['sm_mhz'])"
done; done
