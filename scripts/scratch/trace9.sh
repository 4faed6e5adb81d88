cat > /tmp/tr2.py <<'PY'
import torch, sys, os
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
rows, cols, T = int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3])
W = synth.weights(rows, cols, seed=1); X = synth.activations_t(cols, T, seed=2)
P = vnm.prune_compress(to_dev_bf16(W), 64, 5); Xd = to_dev_bf16(X)
for i in range(3): vnm.spmm(Xd, P, T=T)
torch.cuda.synchronize()
os.environ["VNM_SPMM_TRACE"] = "1"
vnm.spmm(Xd, P, T=T); torch.cuda.synchronize()
PY
timeout 60 python /tmp/tr2.py 4096 4096 16 2>&1 | tail -25
timeout 60 python /tmp/tr2.py 11008 4096 16 2>&1 | tail -25
