"""KroneckerSum.toeplitz_split over several PSFs (five mixture seeds + the rotated Gaussian), sides
128 / 256 / 512 and automatic / fixed rank: what the split drops, the dense-term share and the
apply gap against the unsplit operator (all at the fp32 rounding level, 5e-8 .. 8e-8, on B200)."""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
rng = np.random.default_rng(5)
for n in (128, 256, 512):
    for seed in range(1, 7):
        psf = datagen.mixture_psf(n, seed=seed) if seed < 6 else datagen.rotated_gaussian_psf(n)
        for cfg in (kb.EgkbConfig(k_max=20, k_min=2, p=2, tau=1e-4), kb.EgkbConfig(k_max=12, k_min=12, p=2, tau=1e300)):
            svd, tr = kb.egkb(kb.RearrangedBlur(psf, n), cfg)
            op = kb.assemble(svd, kb.BlockScheme.square_image(n))
            try:
                sp, dropped = op.toeplitz_split()
            except kb.ValidationError as e:
                print("REFUSED", n, seed, tr.chosen_k, str(e)[:80]); continue
            x = rng.standard_normal(n * n)
            a, b = sp.apply(x), op.apply(x)
            at, bt = sp.apply_t(x), op.apply_t(x)
            g1 = np.linalg.norm(a - b) / np.linalg.norm(b); g2 = np.linalg.norm(at - bt) / np.linalg.norm(bt)
            flag = "" if max(g1, g2) < 1e-6 else "  <-- large"
            print(n, seed, "k", op.k, "->", sp.k, "dropped %.1e share %.1e apply gap %.1e %.1e" % (dropped, sp.split_dense_share, g1, g2), flag)
