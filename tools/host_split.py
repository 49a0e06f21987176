"""Wall-clock split of one bench step's host path (n=1024) by wrapping the pieces."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, lowrank, _lib, kronop, linalg
n = 1024
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
scheme = kb.BlockScheme.square_image(n)
acc = {}
def wrap(mod, name, label):
    f = getattr(mod, name)
    def g(*a, **k):
        t = time.perf_counter(); r = f(*a, **k); acc[label] = acc.get(label, 0) + time.perf_counter() - t; return r
    setattr(mod, name, g)
lib = _lib.load()
class L:
    def __getattr__(self, k):
        f = getattr(lib, k)
        if not k.startswith("kb_"): return f
        def g(*a):
            t = time.perf_counter(); r = f(*a); acc["lib." + k] = acc.get("lib." + k, 0) + time.perf_counter() - t; return r
        return g
_lib.load = lambda path=None: L()
wrap(lowrank, "svd_small", "svd_small")
wrap(lowrank._LazyLift, "__init__", "lazylift_init")
wrap(lowrank.rng, "standard_normal", "rng")
wrap(lowrank, "_bases", "bases")
keep = [None]
def step():
    svd, tr = kb.egkb(blur, cfg); keep[0] = kb.assemble(svd, scheme); torch.cuda.synchronize()
for _ in range(5): step()
acc.clear()
K = 20
t = time.perf_counter()
for _ in range(K): step()
tot = (time.perf_counter() - t) / K * 1e6
print("step us", round(tot, 1))
for k, v in sorted(acc.items(), key=lambda kv: -kv[1]): print(f"{k:40s} {v / K * 1e6:9.1f} us")
