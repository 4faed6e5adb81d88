mkdir -p gpurun_out
VNM_SPMM_TRACE=2 timeout 120 python scripts/trace_smallt.py 11008 4096 5 16 > gpurun_out/r02d_trace_up.txt 2>&1; echo "trace $?"
timeout 300 python tests/probes/probe4.py > gpurun_out/r02d_probe4.txt 2>&1; echo "probe4 $?"; cat gpurun_out/r02d_probe4.txt
