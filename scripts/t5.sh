timeout 200 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/sw_dec.json 2> gpurun_out/sw_dec.err || tail -5 gpurun_out/sw_dec.err
python -c "
import json; d=json.load(open('gpurun_out/sw_dec.json'))
print(d['value'], d['roofline'], ' '.join(f\"{l['name']}={l['spmm_us']}us/{l['spmm_gbs']}GBs\" for l in d['detail']['layers']))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/dec_launches.csv python bench.py --workload llama_decode --steps 2 --warmup 3 --no-cpu-baseline --no-baselines > /dev/null 2>&1; echo "ncu $?"
python scripts/summarize_ncu.py launches gpurun_out/dec_launches.csv 2>&1 | head -30
