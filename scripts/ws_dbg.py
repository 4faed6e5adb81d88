import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import oracle
from paper_2410_16135_b200 import vnm
from tests.gpu_util import to_dev_bf16
from tests.test_gpu_spmm import make, _spmm_raw, ctypes_ptr
shapes = [(11008, 4096, 5, 32), (4096, 11008, 5, 16), (4096, 4096, 5, 8), (11008, 4096, 5, 1), (512, 3000, 11, 24)]
order = [int(c) for c in sys.argv[1]] if len(sys.argv) > 1 else [0,1,2,3,4,4,3,2,1,0]
cases = []
for i, (rows, cols, M, T) in enumerate(shapes):
    W, XT, Wm = make(rows, cols, 64, M, T, seed=100 + i)
    Yref, Aref = oracle.gemm_ref(XT, Wm)
    cases.append((vnm.prune_compress(to_dev_bf16(W), 64, M), to_dev_bf16(XT), T, Yref, Aref))
nws = max(vnm.spmm_workspace_bytes(P.g, T) for P, _, T, _, _ in cases)
ws = torch.empty(nws // 4 + 4, dtype=torch.float32, device="cuda")
assert vnm.lib().vnm_spmm_workspace_init(ctypes_ptr(ws), ws.numel() * 4, None) == 0
for k in order:
    P, Xd, T, Yref, Aref = cases[k]
    Y = torch.empty((P.g.rows, (T + 7) // 8 * 8), dtype=torch.float32, device="cuda")[:, :T]
    _spmm_raw(Xd, P, T, Y, ws, ws.numel() * 4)
    torch.cuda.synchronize()
    tick = ws[:4096].view(torch.int32).cpu().numpy()
    tol = oracle.tolerance(Yref, Aref)
    bad = np.abs(Y.cpu().numpy().astype(np.float64) - Yref) > tol
    print("case", k, shapes[k], "bad", int(bad.sum()), "of", bad.size, "nonzero tickets", int((tick != 0).sum()), tick[np.nonzero(tick)][:8], flush=True)
