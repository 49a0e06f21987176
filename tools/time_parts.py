"""Split one n=1024 KP approximation into device graph time and host work."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, ctypes as C
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D, _lib, lowrank
n = 1024
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
y0 = D.to_device(np.random.default_rng(0).standard_normal(n * n).astype(np.float32))
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for _ in range(3):
    svd, tr = kb.egkb(blur, cfg, y0=y0)
torch.cuda.synchronize()
orig = lowrank._lib.load().kb_egkb_run
lib = _lib.load()
times = {"graph": [], "total": []}
class Wrap:
    def __getattr__(self, k): return getattr(lib, k)
    def kb_egkb_run(self, *a):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); r = lib.kb_egkb_run(*a); e1.record(); torch.cuda.synchronize()
        times["graph"].append(e0.elapsed_time(e1)); return r
lowrank._lib.load = lambda: Wrap()
for fl in (False, True):
    times = {"graph": [], "total": []}
    for _ in range(5):
        if fl: flush.zero_()
        torch.cuda.synchronize()
        t = time.perf_counter()
        svd, tr = kb.egkb(blur, cfg, y0=y0)
        op = kb.assemble(svd, kb.BlockScheme.square_image(n))
        torch.cuda.synchronize()
        times["total"].append((time.perf_counter() - t) * 1e3)
    print("flush" if fl else "warm ", "graph ms", np.round(times["graph"], 3), "total ms", np.round(times["total"], 3))
