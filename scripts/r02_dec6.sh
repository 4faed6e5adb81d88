mkdir -p gpurun_out
timeout 300 python tests/probes/probe_stream.py > gpurun_out/r02g_probe_stream.txt 2>&1; echo "probe $?"; cat gpurun_out/r02g_probe_stream.txt
