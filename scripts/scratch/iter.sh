# quick iteration: spmm parity, then perf on the main workloads, then optional extra command
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -x -q --timeout 200 > gpurun_out/it_spmm.log 2>&1; rc=$?; echo "spmm tests exit $rc"; tail -25 gpurun_out/it_spmm.log
if [ $rc -eq 0 ]; then
for w in deit_s llama_prefill llama_decode deit_b; do
  timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it_bench_$w.json 2> gpurun_out/it_bench_$w.err; echo "$w exit $?"
  python -c "
import json; d=json.load(open('gpurun_out/it_bench_$w.json'))
print('$w', d['value'], d['unit'], 'ms', d['ms_per_step'], 'roof', d['roofline']['achieved'], d['roofline']['unit'], d['roofline']['frac'])
for l in d['detail']['layers']: print('   ', l['name'], 'spmm_us', l['spmm_us'], 'TF', l['spmm_useful_tflops'], 'GBs', l['spmm_gbs'], 'prune_us', l['prune_compress_us'])
" 2>&1 | tail -6
done
fi
if [ -n "$EXTRA" ]; then eval "$EXTRA"; fi
