"""Host-side profile of one eGKB + assemble call at n=1024 (where the non-kernel time goes)."""
import cProfile, os, pstats, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**bench.egkb_cfg_kwargs())
blur = kb.RearrangedBlur(prob.psf, prob.n)
scheme = kb.BlockScheme.square_image(prob.n)
def step():
    svd, tr = kb.egkb(blur, cfg)
    return kb.assemble(svd, scheme)
for _ in range(5): step()
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(20): step()
torch.cuda.synchronize()
print("wall per step ms", (time.perf_counter() - t) / 20 * 1e3)
pr = cProfile.Profile(); pr.enable()
for _ in range(20): step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
