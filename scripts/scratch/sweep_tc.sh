mkdir -p gpurun_out
for cfg in "2,192" "1,192" "4,192" "2,128" "4,128" "2,256" "1,256" "4,256"; do
  for w in llama_prefill deit_s; do
    VNM_TC_CFG=$cfg timeout 200 python bench.py --workload $w --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err || { echo "$cfg $w FAIL"; tail -3 gpurun_out/sw_$w.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/sw_$w.json'))
print('$cfg', '$w', ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_useful_tflops']}TF/{l['spmm_gbs']}GBs\" for l in d['detail']['layers']))"
  done
done
