"""Device time of one eGKB (persistent kernel) at side n with the config's PSF family."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D
name = sys.argv[1] if len(sys.argv) > 1 else "n2048"
prob = datagen.make_problem(name)
n = prob.n
blur = kb.RearrangedBlur(prob.psf, n)
cfg = kb.EgkbConfig(**prob.egkb)
y0 = D.to_device(np.random.default_rng(0).standard_normal(n * n).astype(np.float32))
for _ in range(2):
    svd, tr = kb.egkb(blur, cfg, y0=y0)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t = time.perf_counter(); e0.record()
svd, tr = kb.egkb(blur, cfg, y0=y0)
e1.record(); torch.cuda.synchronize()
print(name, "k_p", tr.k_p, "chosen", tr.chosen_k, "egkb call ms", e0.elapsed_time(e1), "wall", (time.perf_counter() - t) * 1e3)
for _ in range(2):
    kb.egkb(blur, cfg)
torch.cuda.synchronize()
t = time.perf_counter(); e0.record()
svd, tr = kb.egkb(blur, cfg)
e1.record(); torch.cuda.synchronize()
print(name, "device-RNG egkb call ms", e0.elapsed_time(e1), "wall", (time.perf_counter() - t) * 1e3)
scheme = kb.BlockScheme.square_image(n)
kb.assemble(svd, scheme); torch.cuda.synchronize()
t = time.perf_counter(); e0.record()
op = kb.assemble(svd, scheme)
e1.record(); torch.cuda.synchronize()
print(name, "assemble ms", e0.elapsed_time(e1), "wall", (time.perf_counter() - t) * 1e3)
