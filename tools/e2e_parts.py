"""Wall-time breakdown of the bench e2e step (public API from host arrays)."""
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
psf_host = prob.psf
def step(parts):
    t0 = time.perf_counter()
    blur = kb.RearrangedBlur(psf_host, n); t1 = time.perf_counter()
    blur._device_kernels(); torch.cuda.synchronize(); t2 = time.perf_counter()
    svd, tr = kb.egkb(blur, cfg); t3 = time.perf_counter()
    op = kb.assemble(svd, scheme); sig = np.asarray(svd.sigma); torch.cuda.synchronize(); t4 = time.perf_counter()
    for k, v in zip(("psf", "upload", "egkb", "assemble"), (t1 - t0, t2 - t1, t3 - t2, t4 - t3)):
        parts.setdefault(k, []).append(v * 1e3)
for _ in range(3): step({})
parts = {}
for _ in range(10): step(parts)
print({k: round(float(np.median(v)), 3) for k, v in parts.items()})
import cProfile, pstats
pr = cProfile.Profile(); pr.enable()
for _ in range(5): step({})
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
