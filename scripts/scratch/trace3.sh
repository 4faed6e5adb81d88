mkdir -p gpurun_out
cat > /tmp/tr.py <<'PY'
import torch, numpy as np, sys, os
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
os.environ["VNM_SPMM_TRACE"] = sys.argv[2]
fl = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
if len(sys.argv) > 3: fl.zero_()
vnm.spmm(Xd, P, T=T); torch.cuda.synchronize()
PY
timeout 60 python /tmp/tr.py 16 1 flush > gpurun_out/trace_cold.log 2>&1; echo "== cold"; grep "trace q" gpurun_out/trace_cold.log | sed -n "1,30p"
