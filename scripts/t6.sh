timeout 600 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x -k "window or prefill or deit or tails or shapes or bf16 or identity or integer" --timeout 200 2>&1 | tail -2
for w in deit_s llama_prefill deit_b; do
    timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/sw_$w.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/sw_$w.json'))
print('$w', d['value'], d['roofline']['achieved'], d['roofline']['unit'], d['roofline']['frac'], ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_useful_tflops']}TF/{l['spmm_gbs']}GBs\" for l in d['detail']['layers']))"
done
