"""Per-line host timing of lowrank.egkb / kronop.assemble at n=1024 (line profiler via sys.settrace-free
checkpoints: wraps the module functions and samples perf_counter between source lines with a tracer)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen, lowrank, kronop
n = 1024
prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**datagen.CONFIGS["n1024"]["egkb"])
blur = kb.RearrangedBlur(prob.psf, n)
scheme = kb.BlockScheme.square_image(n)
keep = [None]
def step():
    svd, tr = kb.egkb(blur, cfg); keep[0] = kb.assemble(svd, scheme); torch.cuda.synchronize()
for _ in range(5): step()
targets = {lowrank.egkb.__code__: "egkb", kronop.assemble.__code__: "assemble"}
acc = {}
last = {}
def tracer(frame, event, arg):
    if frame.f_code not in targets: return None
    def local(frame, event, arg):
        t = time.perf_counter()
        key = (targets[frame.f_code], frame.f_lineno)
        if frame in last:
            pk, pt = last[frame]
            acc[pk] = acc.get(pk, 0) + t - pt
        last[frame] = (key, time.perf_counter())
        return local
    return local
K = 20
sys.settrace(tracer)
for _ in range(K): step()
sys.settrace(None)
for (f, ln), v in sorted(acc.items(), key=lambda kv: -kv[1])[:25]:
    print(f"{f}:{ln:4d} {v / K * 1e6:9.1f} us")
