"""HBM rate for write-heavy streams (DeiT SpMM traffic is ~80% Y^T writes): fill / copy / 1:4 read:write."""
import torch
ev = lambda: torch.cuda.Event(enable_timing=True)
def t(f, n=20):
    for _ in range(3): f()
    a, b = ev(), ev(); ts = []
    for _ in range(n):
        a.record(); f(); b.record(); torch.cuda.synchronize(); ts.append(a.elapsed_time(b) * 1e3)
    ts.sort(); return ts[len(ts) // 2]
for mb in (39, 155, 310, 1024):
    y = torch.empty(mb << 20, dtype=torch.uint8, device="cuda")
    x = torch.empty(mb << 18, dtype=torch.uint8, device="cuda").fill_(1)
    us = t(lambda: y.fill_(0)); print(f"fill {mb} MB: {us:.1f} us {mb*1.048576/us*1e3:.0f} GB/s")
    yv = y.view(4, -1)
    us = t(lambda: yv.copy_(x.view(1, -1).expand(4, -1))); print(f"read {mb/4} MB -> write {mb} MB: {us:.1f} us {(mb*1.25)*1.048576/us*1e3:.0f} GB/s")
    z = torch.empty_like(y)
    us = t(lambda: z.copy_(y)); print(f"copy {mb} MB: {us:.1f} us {2*mb*1.048576/us*1e3:.0f} GB/s")
