# 1-CTA kernel with all three 128-row tiles of a 384-row layer per CTA (NT = 128, RT = 3): X^T read once per token tile
for cfg in "0 0" "128 3" "128 1" "192 2"; do set -- $cfg
  for sh in "384 1536" "384 384"; do
    VNM_TC_PLAN=1 VNM_TC_CFG_NT=$1 VNM_TC_CFG_RT=$2 timeout 120 python scripts/time_spmm.py $sh 5 50432 tc 2>&1 | sed "s/^/nt=$1 rt=$2 /"
  done
done
VNM_TC_PLAN=1 VNM_TC_CFG_NT=128 VNM_TC_CFG_RT=3 timeout 600 python -c "
import torch, numpy as np, oracle
from tests.test_gpu_spmm import sampled_check, make, gpu_y, assert_within
sampled_check(384, 1536, 5, 50432, seed=3, out_dtype=torch.bfloat16, tc=True)
W, XT, Wm = make(384, 1000, 64, 5, 1000, seed=4); Yref, Aref = oracle.gemm_ref(XT, Wm); assert_within(gpu_y(W, XT, 64, 5, 1000, tc=True), Yref, Aref)
W, XT, Wm = make(300, 333, 64, 7, 520, seed=5); Yref, Aref = oracle.gemm_ref(XT, Wm); assert_within(gpu_y(W, XT, 64, 7, 520, tc=True, out_dtype=torch.bfloat16), Yref, Aref, bf16=True)
print('rt3 parity ok')"
