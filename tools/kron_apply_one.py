"""Two Kronecker applies (forward, transpose) at n=1024 on eGKB factors, for an
ncu capture of the banded G-stage and the dense F-stage DGEMMs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen

prob = datagen.make_problem("n1024")
n = prob.n
svd, _ = kb.egkb(kb.RearrangedBlur(prob.psf.astype(np.float32), n), kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"]))
op = kb.assemble(svd, kb.BlockScheme.square_image(n))
x = np.random.default_rng(0).standard_normal(n * n)
for _ in range(2):
    y = op.apply(x)
    xt = op.apply_t(y)
print("k", op.k, "band", op._band.cpu().numpy().tolist(), "norm", float(np.linalg.norm(xt)))
