mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_ria.py -m gpu -q -x --timeout 300 > gpurun_out/t11_ria.log 2>&1; echo "ria tests $?"; tail -15 gpurun_out/t11_ria.log
timeout 300 python tests/probe_dram.py > gpurun_out/probe_dram.log 2>&1; echo "probe $?"; cat gpurun_out/probe_dram.log
