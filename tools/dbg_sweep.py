import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2410_00233_b200 as kb
from conftest import load_golden
g = load_golden("sb_kat")
op = kb.KroneckerSum(list(g["n64_ax"]), list(g["n64_ay"]), kb.BlockScheme.square_image(32))
b, xt = g["n64_b"], g["n64_xtrue"]
lams = np.logspace(np.log10(0.03), np.log10(0.5), 7)
for variant in ("anisotropic",):
    cfgs = [kb.SbConfig.from_gamma(float(l), 2.0, variant=variant, tau=2e-3, l_max=12,
                                   cgls=kb.CglsConfig(i_max=60, tau=1e-4)) for l in lams]
    batch = kb.sb_run_batch(op, b, cfgs, x_true=xt)
    for c, rb in zip(cfgs, batch):
        rs = kb.sb_run(op, b, c, x_true=xt)
        r1 = kb.sb_run_batch(op, b, [c], x_true=xt)[0]
        print(round(c.lam, 4), rb.outer_iters, rs.outer_iters, rb.cgls_iters, rs.cgls_iters, r1.cgls_iters == rs.cgls_iters,
              np.linalg.norm(rb.x - rs.x) / np.linalg.norm(rs.x))
