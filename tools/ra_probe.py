import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
op = kb.RearrangedBlur(datagen.mixture_psf(n), n)
q = torch.randn(n * n, device="cuda")
for _ in range(3): op.matvec(q)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record(); y = op.matvec(q); e1.record(); torch.cuda.synchronize()
print("one product (incl. launch) us", e0.elapsed_time(e1) * 1e3)
