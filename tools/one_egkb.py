"""One eGKB run at n (default 1024) after one warm-up: a short target for ncu."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, device as D
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1024
prob = datagen.make_problem("n1024", n=n)
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
y0 = D.to_device(np.random.default_rng(0).standard_normal(n * n).astype(np.float32))
for _ in range(2):
    svd, tr = kb.egkb(blur, cfg, y0=y0)
    op = kb.assemble(svd, kb.BlockScheme.square_image(n))
torch.cuda.synchronize()
print("ok", tr.chosen_k, tr.k_p)
