mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -x > gpurun_out/r02_gputests.log 2>&1; echo "gpu tests exit $?"; tail -15 gpurun_out/r02_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke exit $?"; tail -2 gpurun_out/r02_smoke.log
