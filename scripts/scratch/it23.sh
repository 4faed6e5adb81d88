python - <<'PY'
import os, torch
os.environ["VNM_PRUNE_TRACE"] = "1"
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
for rows, cols, tc in [(11008, 4096, False), (11008, 4096, True), (1152, 384, True)]:
    W = to_dev_bf16(synth.weights(rows, cols, seed=1))
    for _ in range(2):
        P = vnm.prune_compress(W, 64, 5, tc=tc)
    torch.cuda.synchronize()
PY
