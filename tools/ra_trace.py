"""Phase times of k_ra_block for one vector and a 16-vector block at n=1024 (KB_PK_TRACE=1)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D
from paper_2410_00233_b200.lowrank import _EngineOp
n = 1024
op = _EngineOp(kb.RearrangedBlur(datagen.mixture_psf(n), n))
x = torch.randn(n * n, device="cuda")
y = torch.empty_like(x)
X = torch.randn(16, n * n, device="cuda")
for _ in range(3):
    op.apply(x, 0, y); op.apply_block(X, 0)
torch.cuda.synchronize()
print("single:", flush=True); op.apply(x, 0, y); torch.cuda.synchronize()
print("block16:", flush=True); op.apply_block(X, 0); torch.cuda.synchronize()
