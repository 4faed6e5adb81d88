timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 300 -k "deit or window or natural" > gpurun_out/it36.log 2>&1; echo "tests $?"; tail -1 gpurun_out/it36.log
python - <<'PY'
import numpy as np, torch, oracle
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
# full-Y check of the split path (odd row tiles, large T) against the oracle on a 1152 x 384 weight, 8448 tokens
rows, cols, M, T = 1152, 384, 5, 8448
W = synth.weights(rows, cols, seed=5); XT = synth.activations_t(cols, T, seed=6)
mask = oracle.prune(W, 64, M); Wm = oracle.apply_mask(W, mask, 64, M)
P = vnm.prune_compress(to_dev_bf16(W), 64, M, tc=True)
Y = vnm.spmm(to_dev_bf16(XT), P, T=T).cpu().numpy().astype(np.float64)
Yref, Aref = oracle.gemm_ref(XT, Wm)
print("split path full check:", bool(np.all(np.abs(Y - Yref) <= oracle.tolerance(Yref, Aref))))
PY
S="python scripts/time_spmm.py"
for i in 1 2; do timeout 60 $S 1152 384 5 50432 tc 2>&1 | tail -1; done
for i in 1 2; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-baselines > gpurun_out/it36_deit_s_$i.json 2>/dev/null; done
python scripts/bench_summary.py gpurun_out/it36_*.json
