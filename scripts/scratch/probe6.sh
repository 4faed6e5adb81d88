mkdir -p gpurun_out
for i in 9 10 11 12 13 14; do timeout 60 python tests/probe2.py window $i > gpurun_out/probe6_window_$i.log 2>&1; echo "window $i exit $?"; grep "{" gpurun_out/probe6_window_$i.log | cut -c1-200; done
