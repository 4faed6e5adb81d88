cat > /tmp/trd.py <<'PY'
import torch, sys, os
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
for rows, cols, T in [(4096, 4096, 8), (11008, 4096, 16)]:
    W = to_dev_bf16(synth.weights(rows, cols, seed=1)); P = vnm.prune_compress(W, 64, 5)
    X = to_dev_bf16(synth.activations_t(cols, T, seed=2))
    for i in range(3): vnm.spmm(X, P, T=T)
    torch.cuda.synchronize()
    os.environ["VNM_SPMM_TRACE"] = "1"
    vnm.spmm(X, P, T=T); torch.cuda.synchronize()
    del os.environ["VNM_SPMM_TRACE"]
PY
VNM_DEC=1 timeout 60 python /tmp/trd.py 2>&1 | tail -40
