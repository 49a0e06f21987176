"""Per-step device times of the bench step with the nvidia-smi sampler running (spike hunt)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
prob = datagen.make_problem("n1024")
n = prob.n
cfg = kb.EgkbConfig(**bench.egkb_cfg_kwargs())
scheme = kb.BlockScheme.square_image(n)
blur = kb.RearrangedBlur(prob.psf, n)
def step():
    svd, tr = kb.egkb(blur, cfg)
    return kb.assemble(svd, scheme)
for _ in range(3): step()
for label, interval in (("no-sampler", None), ("smi-200ms", 200)):
    clk = bench.Clocks(0) if interval else None
    for _ in range(3): step()
    torch.cuda.synchronize()
    ts = []
    for i in range(150):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); step(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    if clk: print(clk.stop())
    ts = np.array(ts)
    print(label, "median %.3f max %.3f mean %.3f  >3ms: %d" % (np.median(ts), ts.max(), ts.mean(), (ts > 3).sum()),
          np.round(ts[ts > 3], 1))
