timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/it25_deit_s.json 2>gpurun_out/it25.err; echo "bench $?"; tail -2 gpurun_out/it25.err
timeout 300 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/it25_dec.json 2>/dev/null; echo "dec $?"
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 1 --steps 4 --warmup 3 --mode out --no-cpu-baseline --no-baselines > gpurun_out/it25_out.json 2>/dev/null; echo "out $?"
python scripts/bench_summary.py gpurun_out/it25_*.json
python -c "
import json; d=json.loads(open('gpurun_out/it25_deit_s.json').read().strip().splitlines()[-1]); print(json.dumps(d['roofline'])); print(d['e2e'], d['gpu_launches'], d['clocks'], d['cpu_baseline'])"
