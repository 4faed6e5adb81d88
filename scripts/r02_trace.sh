timeout 900 python -m pytest -q -x tests/test_gpu_spmm_batched.py tests/test_gpu_graph_replay.py tests/test_gpu_spmm.py tests/test_gpu_bounds.py tests/test_gpu_timed_path.py 2>&1 | tail -3
