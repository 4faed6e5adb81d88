mkdir -p gpurun_out
for i in 0 1 2 3 4 5 6 7 8; do timeout 60 python tests/probe2.py window $i > gpurun_out/probe5_window_$i.log 2>&1; echo "window $i exit $?"; grep "{" gpurun_out/probe5_window_$i.log | cut -c1-400; done
