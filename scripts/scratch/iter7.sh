mkdir -p gpurun_out
bash scripts/trace3.sh 2>&1 | head -32
timeout 900 python -m pytest tests/test_gpu_spmm.py tests/test_gpu_prune.py -k "slab or decode or toy or tails or shapes"  -m gpu -q --timeout 200 -x > gpurun_out/it_all.log 2>&1; echo "gpu tests exit $?"; tail -3 gpurun_out/it_all.log
for w in llama_decode; do
    timeout 200 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_$w.json 2> gpurun_out/sw_$w.err || { echo "$w FAIL"; tail -3 gpurun_out/sw_$w.err; continue; }
    python -c "
import json; d=json.load(open('gpurun_out/sw_$w.json'))
print('$w', d['value'], d['roofline']['achieved'], d['roofline']['unit'], d['roofline']['frac'], ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_useful_tflops']}TF/{l['spmm_gbs']}GBs\" for l in d['detail']['layers']))"
done
