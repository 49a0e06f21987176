import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from types import SimpleNamespace
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
from oracle import lowrank as olr, structured as ost
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
name = {512: "n512", 1024: "n1024"}[n]
psf = datagen.mixture_psf(n); k32 = psf.astype(np.float32)
cfg = kb.EgkbConfig(**datagen.CONFIGS[name]["egkb"])
for passes in (1, 2):
    svd, tr = kb.egkb(kb.RearrangedBlur(psf, n), cfg, reorth_passes=passes)
    print("gpu passes", passes, tr.chosen_k, tr.k_p, tr.stop_reason, tr.breakdown)
    print("  alphas", np.array(tr.alphas))
    print("  ts    ", np.array(tr.ts))
def cgs1_64(vec, basis):
    S = np.stack(basis).astype(np.float64); v = vec.astype(np.float64)
    return (v - S.T @ (S @ v)).astype(np.float32)
olr.project_out = cgs1_64
ocfg = SimpleNamespace(k_max=cfg.k_max, p=cfg.p, tau=cfg.tau, k_min=cfg.k_min, reorth=None, seed=0, break_tol=None, keep_basis=False)
(u, s, v), tr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q), lambda x: ost.ra_rmatvec(k32, n, x), (n*n, n*n), np.float32, ocfg)
print("cpu cgs1_64", tr.chosen_k, tr.k_p)
print("  alphas", np.array(tr.alphas))
print("  ts    ", np.array(tr.ts))
# single-step comparison of the first products
blur = kb.RearrangedBlur(psf, n)
y0 = np.random.default_rng(0).standard_normal(n*n).astype(np.float32)
s1 = y0 / np.float32(np.linalg.norm(y0))
g = blur.rmatvec(s1); c = ost.ra_rmatvec(k32, n, s1)
print("rmatvec rel", np.linalg.norm(g - c) / np.linalg.norm(c), "norms", np.linalg.norm(g.astype(np.float64)), np.linalg.norm(c.astype(np.float64)))
