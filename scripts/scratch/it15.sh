timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it15_deit_s.json 2>gpurun_out/it15_deit_s.err; echo "bench exit $?"; tail -3 gpurun_out/it15_deit_s.err
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it15_dec.json 2>/dev/null
python scripts/bench_summary.py gpurun_out/it15_*.json
python -c "
import json
for f in ['gpurun_out/it15_deit_s.json','gpurun_out/it15_dec.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(f, d['e2e'])"
