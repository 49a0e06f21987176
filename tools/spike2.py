"""Which part of the 2nd timed bench step is slow? (device phases vs host gaps)"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D
prob = datagen.make_problem("n1024")
n = prob.n
cfg = kb.EgkbConfig(**bench.egkb_cfg_kwargs())
scheme = kb.BlockScheme.square_image(n)
blur = kb.RearrangedBlur(prob.psf, n)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device=D.device())
def step():
    svd, tr = kb.egkb(blur, cfg)
    return kb.assemble(svd, scheme)
for _ in range(3): step()
torch.cuda.synchronize()
mode = sys.argv[1] if len(sys.argv) > 1 else "flush"
for i in range(6):
    if mode == "flush": flush.zero_()
    elif mode == "sleep": time.sleep(0.005)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(); step(); b.record(); torch.cuda.synchronize()
    print(mode, i, "device %.3f wall %.3f" % (a.elapsed_time(b), (time.perf_counter() - t0) * 1e3), flush=True)
