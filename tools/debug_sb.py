import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
from oracle import sb as osb
g = dict(np.load(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests/golden/sb_kat.npz")))
side = 32
ax, ay = list(g["n64_ax"]), list(g["n64_ay"])
op = kb.KroneckerSum(ax, ay, kb.BlockScheme.square_image(side))
oop = osb.KronOracle(ax, ay, side, side, side, side)
rng = np.random.default_rng(0)
x = rng.standard_normal(side*side)
print("apply rel", np.linalg.norm(op.apply(x)-oop.apply(x))/np.linalg.norm(oop.apply(x)))
print("apply_t rel", np.linalg.norm(op.apply_t(x)-oop.apply_t(x))/np.linalg.norm(oop.apply_t(x)))
aug = kb.AugmentedOp(op, side, datagen.LAM, datagen.LAM)
oaug = osb.AugOracle(oop, side, datagen.LAM, datagen.LAM)
y = rng.standard_normal(aug.shape[0])
print("aug apply", np.linalg.norm(aug.apply(x)-oaug.apply(x))/np.linalg.norm(oaug.apply(x)))
print("aug apply_t", np.linalg.norm(aug.apply_t(y)-oaug.apply_t(y))/np.linalg.norm(oaug.apply_t(y)))
b = g["n64_b"]
rhs = np.concatenate([b, np.zeros(2*side*(side-1))])
for it in (1, 2, 5, 10, 20):
    r = kb.cgls_solve(aug, rhs, kb.CglsConfig(i_max=it, tau=0.0))
    o = osb.cgls(oaug, rhs, it, 0.0)
    print("cgls", it, np.linalg.norm(r.x-o.x)/np.linalg.norm(o.x))
for L in (1, 2, 5):
    cfg = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, tau=0.0, l_max=L, cgls=kb.CglsConfig(i_max=20, tau=0.0))
    r = kb.sb_run(op, b, cfg)
    o = osb.sb_run(oop, b, datagen.LAM, datagen.BETA, tau=0.0, l_max=L, i_max=20, tau_cgls=0.0)
    print("sb", L, np.linalg.norm(r.x-o.x)/np.linalg.norm(o.x))
# second oracle run with reassociated kron (CPU-vs-CPU drift)
class K2(osb.KronOracle):
    def apply(self, x):
        xm = osb._unvec(x, self.n2, self.n1); acc = np.zeros((self.m2, self.m1))
        for a, bb in reversed(list(zip(self.ax, self.ay))): acc += bb @ (xm @ a.T)
        return osb._vec(acc)
o2 = osb.sb_run(K2(ax, ay, side, side, side, side), b, datagen.LAM, datagen.BETA, tau=0.0, l_max=5, i_max=20, tau_cgls=0.0)
o = osb.sb_run(oop, b, datagen.LAM, datagen.BETA, tau=0.0, l_max=5, i_max=20, tau_cgls=0.0)
print("cpu-cpu drift 5x20", np.linalg.norm(o2.x-o.x)/np.linalg.norm(o.x))
