mkdir -p gpurun_out
for i in 1 2 3; do timeout 60 python tests/probe2.py interleave $i > gpurun_out/probe3_interleave_$i.log 2>&1; echo "interleave $i exit $?"; head -2 gpurun_out/probe3_interleave_$i.log | cut -c1-300; done
timeout 120 python tests/probe2.py mma_multi > gpurun_out/probe3_mma_multi.log 2>&1; echo "mma_multi exit $?"; cat gpurun_out/probe3_mma_multi.log | grep "{"
timeout 300 python tests/probe2.py tma_bw > gpurun_out/probe3_tma_bw.log 2>&1; echo "tma exit $?"; grep "{" gpurun_out/probe3_tma_bw.log
