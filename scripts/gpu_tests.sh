mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,driver_version --format=csv > gpurun_out/smi.txt 2>&1
timeout 180 python __graft_entry__.py > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
tail -3 gpurun_out/smoke.log
timeout 900 python -m pytest tests/test_gpu_prune.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_prune.log 2>&1; echo "prune exit $?"
tail -15 gpurun_out/pytest_prune.log
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_spmm.log 2>&1; echo "spmm exit $?"
tail -30 gpurun_out/pytest_spmm.log
