cat > /tmp/tr.py <<'PY'
import torch, sys, os
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
rows, cols, T, M = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
W = synth.weights(rows, cols, seed=1); X = synth.activations_t(cols, T, seed=2)
Wd = to_dev_bf16(W); Xd = to_dev_bf16(X)
P = vnm.prune_compress(Wd, 64, M, tc=True)
for i in range(3): vnm.spmm(Xd, P, T=T, out_dtype=torch.bfloat16)
torch.cuda.synchronize()
os.environ["VNM_SPMM_TRACE"] = "1"
vnm.spmm(Xd, P, T=T, out_dtype=torch.bfloat16); torch.cuda.synchronize()
PY
for cfg in "11008 4096 2048 5" "1152 384 50432 5" "384 1536 50432 5"; do echo "== $cfg"; timeout 60 python /tmp/tr.py $cfg 2>&1 | tail -12; done
