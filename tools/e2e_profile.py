"""Where the e2e step's host time goes: RearrangedBlur(psf_host) (validation scan, private
copy, normalise + cast into pinned memory, upload, device transposes) and egkb + assemble +
sigma read-back, 40 repetitions each with the L2 flushed in between."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_00233_b200 as kb  # noqa: E402
from paper_2410_00233_b200 import datagen  # noqa: E402

prob = datagen.make_problem("n1024")
cfg = kb.EgkbConfig(**prob.egkb)
scheme = kb.BlockScheme.square_image(prob.n)
flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")


def stats(a):
    a = np.asarray(a)
    return f"min {a.min():.3f}  median {np.median(a):.3f}  p90 {np.percentile(a, 90):.3f}  max {a.max():.3f} ms"


tb, te, tp = [], [], []
for i in range(45):
    flush.zero_()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    psf_obj = kb.Psf(prob.psf)              # validation scan + private copy
    t1 = time.perf_counter()
    blur = kb.RearrangedBlur(psf_obj, prob.n)
    blur.op_struct()                       # normalise + cast + upload + transposes
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    svd, tr = kb.egkb(blur, cfg)
    op = kb.assemble(svd, scheme)
    sig = np.asarray(svd.sigma)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    if i >= 5:
        tp.append((t1 - t0) * 1e3)
        tb.append((t2 - t1) * 1e3)
        te.append((t3 - t2) * 1e3)
print("Psf(psf_host) validation scan + private copy:", stats(tp))
print("RearrangedBlur + upload + transposes (synced):", stats(tb))
print("egkb + assemble + sigma                      :", stats(te))
print("sum                                          :", stats(np.array(tp) + np.array(tb) + np.array(te)))
