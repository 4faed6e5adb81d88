mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_spmm.py -m gpu -q -x --timeout 200 > gpurun_out/t10_tests.log 2>&1; echo "spmm tests $?"; tail -3 gpurun_out/t10_tests.log
timeout 200 python bench.py --workload llama_decode --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/t10_dec.json 2> gpurun_out/t10_dec.err || tail -3 gpurun_out/t10_dec.err
python scripts/bench_summary.py gpurun_out/t10_dec.json
cat > /tmp/td.py <<'PY'
import torch, sys
sys.path.insert(0, '.')
from paper_2410_16135_b200 import synth, vnm
from tests.gpu_util import to_dev_bf16
for rows, cols in [(4096, 4096), (11008, 4096), (4096, 11008)]:
    W = to_dev_bf16(synth.weights(rows, cols, seed=1)); P = vnm.prune_compress(W, 64, 5)
    for T in (1, 2, 4, 8, 16):
        X = to_dev_bf16(synth.activations_t(cols, T, seed=2))
        out = torch.empty(rows, 8 * ((T + 7) // 8), dtype=torch.bfloat16, device='cuda')
        ws = torch.empty(max(vnm.spmm_workspace_bytes(P.g, T), 16) // 4, dtype=torch.float32, device='cuda')
        fl = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device='cuda')
        ts = []
        for i in range(12):
            fl.zero_(); fl.sum()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(); vnm.spmm(X, P, T=T, out=out, workspace=ws); e1.record(); torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3)
        us = sorted(ts[2:])[len(ts[2:]) // 2]
        byt = rows * P.g.ld_val * 2 + rows * P.g.ld_meta * 4 + rows // 64 * P.g.nb_pad * 4
        print(f"{rows}x{cols} T={T}: {us:.2f} us  {byt / us / 1e3:.0f} GB/s")
PY
timeout 120 python /tmp/td.py
VNM_NO_DEC=1 timeout 120 python /tmp/td.py 2>&1 | sed 's/^/pair: /'
