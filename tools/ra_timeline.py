"""Warm per-kernel device times of the standalone R(A) product (single and 16-vector block)
at n=1024 from the torch profiler (CUPTI)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
from paper_2410_00233_b200.lowrank import _EngineOp
n = 1024
op = _EngineOp(kb.RearrangedBlur(datagen.mixture_psf(n), n))
x = torch.randn(n * n, device="cuda"); y = torch.empty_like(x)
X = torch.randn(16, n * n, device="cuda")
for _ in range(5):
    op.apply(x, 0, y); op.apply_block(X, 0)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(10):
        op.apply(x, 0, y); op.apply(x, 1, y)
    for _ in range(10):
        op.apply_block(X, 0)
    torch.cuda.synchronize()
tot = {}
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        key = (e.name[:40], )
        tot.setdefault(key, []).append(e.time_range.end - e.time_range.start)
for k, v in tot.items(): print(f"{k[0]:42s} n={len(v):3d} mean={sum(v)/len(v):8.2f} us  min={min(v):7.2f}")
