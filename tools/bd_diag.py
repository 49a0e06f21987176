"""Breakdown diagnostics at n=1024 rank 30+2: GPU alphas/ts vs the oracle's."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
from oracle import lowrank as olr
from oracle import structured as ost
from types import SimpleNamespace
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
name = {256: "n256", 512: "n512", 1024: "n1024", 2048: "n2048"}[n]
psf = datagen.mixture_psf(n)
cfg = kb.EgkbConfig(**datagen.CONFIGS[name]["egkb"])
svd, tr = kb.egkb(kb.RearrangedBlur(psf, n), cfg)
print("gpu k", tr.chosen_k, tr.k_p, tr.stop_reason, tr.breakdown)
print("gpu alphas", np.array(tr.alphas))
print("gpu ts", np.array(tr.ts))
k32 = psf.astype(np.float32)
oc = SimpleNamespace(k_max=cfg.k_max, p=cfg.p, tau=cfg.tau, k_min=cfg.k_min, reorth=None, seed=0, break_tol=None, keep_basis=False)
(_, os_, _), otr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q), lambda s: ost.ra_rmatvec(k32, n, s), (n * n, n * n), np.float32, oc)
print("cpu k", otr.chosen_k, otr.k_p, otr.stop_reason)
print("cpu alphas", np.array(otr.alphas))
print("cpu ts", np.array(otr.ts))
print("sigma gpu", svd.sigma)
print("sigma cpu", os_)
