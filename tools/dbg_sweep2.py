import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np
import paper_2410_00233_b200 as kb
from conftest import load_golden
g = load_golden("sb_kat")
op = kb.KroneckerSum(list(g["n64_ax"]), list(g["n64_ay"]), kb.BlockScheme.square_image(32))
b, xt = g["n64_b"], g["n64_xtrue"]
for l in np.logspace(np.log10(0.03), np.log10(0.5), 7):
    r = kb.sb_run(op, b, kb.SbConfig.from_gamma(float(l), 2.0, tau=0.0, l_max=12, cgls=kb.CglsConfig(i_max=60, tau=1e-4)))
    print(round(l, 4), ["%.1e" % v for v in r.rc_history])
