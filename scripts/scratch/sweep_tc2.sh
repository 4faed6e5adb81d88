mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_prune.py -m gpu -q --timeout 200 -k "window or llama_prefill or deit" > gpurun_out/it_tc.log 2>&1; echo "tc tests exit $?"; tail -5 gpurun_out/it_tc.log
for cfg in "192,2" "128,2" "192,1" "256,1"; do
  VNM_TC_CFG=$cfg timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 -k "window_plan" > gpurun_out/it_tc_$cfg.log 2>&1; echo "cfg $cfg window tests exit $?"
  for w in llama_prefill deit_s deit_b; do
    VNM_TC_CFG=$cfg timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err || { echo "$cfg $w FAIL"; tail -3 gpurun_out/sw_$w.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/sw_$w.json'))
print('$cfg', '$w', ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_useful_tflops']}TF/{l['spmm_gbs']}GBs\" for l in d['detail']['layers']), 'pc', [l['prune_compress_us'] for l in d['detail']['layers']])"
  done
done
