mkdir -p gpurun_out
for v in 0 1 2 3; do
VNM_DEC_META=$v timeout 300 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 100 -k "toy or token_tails" > gpurun_out/t9_meta$v.log 2>&1; echo "meta variant $v: $?"; tail -2 gpurun_out/t9_meta$v.log | head -1
done
