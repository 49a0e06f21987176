"""Host-side cost of one bench step (egkb with device RNG + assemble), n=1024."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
n = 1024
prob = datagen.make_problem("n1024", n=n)
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
sch = kb.BlockScheme.square_image(n)
keep = [None]
def step():
    svd, tr = kb.egkb(blur, cfg); keep[0] = kb.assemble(svd, sch); torch.cuda.synchronize()
for _ in range(5): step()
ts = []
for _ in range(20):
    t = time.perf_counter(); step(); ts.append((time.perf_counter() - t) * 1e3)
print("step wall ms median", np.median(ts))
pr = cProfile.Profile(); pr.enable()
for _ in range(10): step()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(25)
