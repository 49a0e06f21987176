import cProfile, pstats, time, torch, numpy as np, sys
sys.path.insert(0, '/root/repo')
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
prob = datagen.make_problem("n1024")
blur = kb.RearrangedBlur(prob.psf, prob.n)
cfg = kb.EgkbConfig(**prob.egkb)
scheme = kb.BlockScheme.square_image(prob.n)
def step():
    svd, tr = kb.egkb(blur, cfg)
    op = kb.assemble(svd, scheme)
    return op
for _ in range(5): step()
torch.cuda.synchronize()
t0=time.perf_counter()
for _ in range(50): step()
torch.cuda.synchronize()
print("ms/step", (time.perf_counter()-t0)/50*1e3)
pr=cProfile.Profile(); pr.enable()
for _ in range(50): step()
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
