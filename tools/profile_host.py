"""Host-side profile of one KP approximation at n=1024 (resident and e2e)."""
import cProfile, pstats, sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
prob = datagen.make_problem("n1024", n=n)
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
y0 = D.to_device(np.random.default_rng(0).standard_normal(n * n).astype(np.float32))
sch = kb.BlockScheme.square_image(n)
def resident():
    svd, tr = kb.egkb(blur, cfg, y0=y0); op = kb.assemble(svd, sch); torch.cuda.synchronize(); return tr
def e2e():
    b = kb.RearrangedBlur(prob.psf, n); svd, tr = kb.egkb(b, cfg); op = kb.assemble(svd, sch); s = np.asarray(svd.sigma); torch.cuda.synchronize()
for f in (resident, e2e):
    for _ in range(3): f()
    t = time.perf_counter(); 
    for _ in range(5): f()
    print(f.__name__, (time.perf_counter() - t) / 5 * 1e3, "ms")
    pr = cProfile.Profile(); pr.enable(); f(); pr.disable()
    pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
