"""Host cost of kronop.assemble's pieces at n=1024 (after an eGKB)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D, _lib
n = 1024
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
scheme = kb.BlockScheme.square_image(n)
keep = []
acc = {}
def tick(name, t0):
    t = time.perf_counter(); acc[name] = acc.get(name, 0) + t - t0; return t
for it in range(25):
    svd, tr = kb.egkb(blur, cfg)
    torch.cuda.synchronize()
    t = time.perf_counter()
    k = svd.k; m_u, m_v = svd.shape; t = tick("shape/k", t)
    f = D.empty((k, m_u), np.float64); t = tick("empty f", t)
    g = D.empty((k, m_v), np.float64); t = tick("empty g", t)
    sig = np.ascontiguousarray(svd.sigma.astype(np.float64)); t = tick("sig", t)
    svd._lazy.assemble(sig, f, g); t = tick("lazy.assemble", t)
    op = kb.KroneckerSum.from_device(f, g, scheme); t = tick("from_device", t)
    torch.cuda.synchronize(); t = tick("sync(lift)", t)
    keep = [op]
    if it == 4: acc.clear()
for k_, v in acc.items(): print(f"{k_:16s} {v / 20 * 1e6:8.1f} us")
