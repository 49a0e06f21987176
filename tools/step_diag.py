"""Per-step device times of the bench step under flush / clock-sampling variants."""
import os, sys
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
for mode in ("plain", "flush", "flush+clocks", "plain"):
    clk = bench.Clocks(0) if "clocks" in mode else None
    ts = []
    for i in range(10):
        if "flush" in mode:
            flush.zero_()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if clk: clk.stop()
    print(mode, " ".join(f"{t:.2f}" for t in ts))
