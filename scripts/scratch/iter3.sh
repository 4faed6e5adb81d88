mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prune.py tests/test_gpu_spmm.py -m gpu -q --timeout 200 -x > gpurun_out/it_all.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/it_all.log
for cfg in "256,1" "192,1" "192,2"; do
  for w in llama_prefill deit_s; do
    VNM_TC_CFG=$cfg timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err || { echo "$cfg $w FAIL"; tail -3 gpurun_out/sw_$w.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/sw_$w.json'))
print('$cfg', '$w', d['value'], ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_useful_tflops']}TF\" for l in d['detail']['layers']), 'pc', [l['prune_compress_us'] for l in d['detail']['layers']])"
  done
done
timeout 200 python bench.py --workload llama_decode --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_dec.json 2>&1; python -c "
import json; d=json.load(open('gpurun_out/sw_dec.json'))
print('decode', d['value'], ' '.join(f\"{l['name']}={l['spmm_us']}us\" for l in d['detail']['layers']), 'pc', [l['prune_compress_us'] for l in d['detail']['layers']])"
