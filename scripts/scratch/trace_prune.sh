cat > /tmp/tp.py <<'PY'
import torch, sys, os
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
for rows, cols, M, tc in [(1152, 384, 5, True), (11008, 4096, 5, False), (11008, 4096, 5, True)]:
    W = to_dev_bf16(synth.weights(rows, cols, seed=1))
    for i in range(3): vnm.prune_compress(W, 64, M, tc=tc)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(20): vnm.prune_compress(W, 64, M, tc=tc)
    e1.record(); torch.cuda.synchronize()
    print(rows, cols, M, tc, "avg us (eager, incl. alloc)", e0.elapsed_time(e1) / 20 * 1e3)
    os.environ["VNM_PRUNE_TRACE"] = "1"
    vnm.prune_compress(W, 64, M, tc=tc); torch.cuda.synchronize()
    del os.environ["VNM_PRUNE_TRACE"]
PY
timeout 120 python /tmp/tp.py 2>&1 | tail -12
