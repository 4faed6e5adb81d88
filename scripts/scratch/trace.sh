mkdir -p gpurun_out
cat > /tmp/tr.py <<'PY'
import torch, numpy as np, sys
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
T = int(sys.argv[1])
W = synth.weights(11008, 4096, seed=1)
X = synth.activations_t(4096, T, seed=2)
P = vnm.prune_compress(to_dev_bf16(W), 64, 5)
Xd = to_dev_bf16(X)
for i in range(3): vnm.spmm(Xd, P, T=T)
torch.cuda.synchronize()
import os; os.environ["VNM_SPMM_TRACE"] = "1"
vnm.spmm(Xd, P, T=T); torch.cuda.synchronize()
PY
python /tmp/tr.py 16 > gpurun_out/trace16.log 2>&1; tail -66 gpurun_out/trace16.log | head -30
