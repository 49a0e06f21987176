import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import io as kio
psf = kb.Psf(kio.read_mtx('/root/repo/tests/golden/cli/psf.mtx'))
n = 16
blur = kb.RearrangedBlur(psf, n, dtype=np.float64)
cfg = kb.EgkbConfig(k_max=8, k_min=8, tau=1e300)
svd, tr = kb.egkb(blur, cfg)
print(svd, tr.chosen_k, tr.k_p)
op = kb.assemble(svd, kb.BlockScheme.square_image(n))
u = svd.u; v = svd.v
print("u norms", np.linalg.norm(u, axis=0)[:5])
f = op.f_dev.cpu().numpy()
print("F vs sigma*u", np.abs(f - (u * svd.sigma).T).max())
svd2, _ = kb.egkb(blur, cfg)
u2 = svd2.u
print("u vs fresh u", np.abs(u - u2).max())
