mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_permute.py tests/test_gpu_ria.py -m gpu -q -x --timeout 600 > gpurun_out/t16_tests.log 2>&1; echo "tests $?"; tail -15 gpurun_out/t16_tests.log
cat > /tmp/tp2.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
for rows, cols, V, M in [(1152, 384, 64, 5), (3072, 768, 64, 8), (4096, 4096, 64, 5)]:
    W = to_dev_bf16(synth.weights(rows, cols, seed=1))
    act = vnm.act_norms(to_dev_bf16(synth.activations_t(cols, 512, seed=2)))
    s = vnm.ria_score(W, act, 0.5)
    for i in range(2): c = vnm.permute_gain(s, V, M)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); c = vnm.permute_gain(s, V, M); e1.record(); torch.cuda.synchronize()
    e2, e3 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e2.record(); s2 = vnm.ria_score(W, act, 0.5); e3.record(); torch.cuda.synchronize()
    print(f"{rows}x{cols} {V}:2:{M}: permute_gain {e0.elapsed_time(e1):.3f} ms ({c.shape[0]}^2 entries), ria_score {e2.elapsed_time(e3)*1e3:.1f} us")
PY
timeout 300 python /tmp/tp2.py
