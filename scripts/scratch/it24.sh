for w in deit_s llama_decode; do VNM_BENCH_NOEV=1 timeout 300 python bench.py --workload $w --steps 10 --warmup 3 --no-cpu-baseline --no-baselines 2>&1 >/dev/null | grep "without"; done
