mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/probe_smi.txt 2>&1
for cfg in "128 0 0" "64 0 0" "64 1 0" "64 0 1" "64 0 2" "128 1 0"; do
  timeout 120 python tests/probe_layouts.py sparse $cfg > gpurun_out/probe_sparse_$(echo $cfg | tr ' ' _).log 2>&1
  echo "cfg $cfg exit $?"
done
timeout 120 python tests/probe_layouts.py dense > gpurun_out/probe_dense.log 2>&1; echo dense $?
timeout 300 python tests/probe_layouts.py bench > gpurun_out/probe_bench.log 2>&1; echo bench $?
