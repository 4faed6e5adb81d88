mkdir -p gpurun_out
timeout 300 python bench.py --workload llama_prefill --mode out --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t18_out.json 2> gpurun_out/t18_out.err; echo "out mode $?"; tail -2 gpurun_out/t18_out.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t18_trun.json 2> gpurun_out/t18_trun.err; echo "torchrun token $?"; tail -2 gpurun_out/t18_trun.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 1 --workload llama_decode --mode out --steps 5 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/t18_trun_out.json 2> gpurun_out/t18_trun_out.err; echo "torchrun out $?"; tail -2 gpurun_out/t18_trun_out.err
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29535 bench.py --impl reference --gpus 1 --steps 2 --warmup 1 > gpurun_out/t18_ref.json 2> gpurun_out/t18_ref.err; echo "torchrun ref $?"
python scripts/bench_summary.py gpurun_out/t18_*.json
python -c "
import json
for f in ['gpurun_out/t18_out.json','gpurun_out/t18_trun_out.json']:
    d=json.loads(open(f).read().strip().splitlines()[-1]); print(d['scaling'], d['config']['parallelism'], d['value'])"
