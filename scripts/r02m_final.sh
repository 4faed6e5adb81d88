# last HEAD check of the round: the full GPU suite and smoke
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 > gpurun_out/r02m_gputests.log 2>&1; echo "gpu tests exit $?"; tail -2 gpurun_out/r02m_gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
