# final HEAD sanity: smoke, the window-form / timed-path / window-16 / prune tests, the default bench line
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1500 python -m pytest -q tests/test_gpu_spmm.py tests/test_gpu_timed_path.py tests/test_gpu_window16.py tests/test_gpu_tc3_ts.py tests/test_gpu_bounds.py 2>&1 | tail -1
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02l_bench_deit_s.json 2>/dev/null; python scripts/bench_summary.py gpurun_out/r02l_bench_deit_s.json | head -1
