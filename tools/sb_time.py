"""Time a short split-Bregman solve (5 outer iterations, CglsConfig(100, 1e-4)) at n=1024 on
the eGKB factors, with and without KroneckerSum.toeplitz_split."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2410_00233_b200 as kb  # noqa: E402
from paper_2410_00233_b200 import datagen, device as D  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "n1024"
outer = int(sys.argv[2]) if len(sys.argv) > 2 else 5
prob = datagen.make_problem(name)
svd, tr = kb.egkb(kb.RearrangedBlur(prob.psf, prob.n), kb.EgkbConfig(**prob.egkb))
op = kb.assemble(svd, kb.BlockScheme.square_image(prob.n))
sp, resid = op.toeplitz_split()
torch.cuda.synchronize()
t0 = time.perf_counter()
sp, resid = op.toeplitz_split()
torch.cuda.synchronize()
print(f"{name}: k={op.k} split in {(time.perf_counter() - t0) * 1e3:.1f} ms, dropped {resid:.2e}, "
      f"dense-term share |a|/|F_1| = {sp.split_dense_share:.2e}", flush=True)
cfg = kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=outer, cgls=kb.CglsConfig(i_max=100, tau=1e-4))
b = D.to_device(prob.b)
for label, o in (("dense F", op), ("split", sp)):
    kb.sb_run(o, b, kb.SbConfig(lam=0.1150, beta=0.0066, variant="isotropic", tau=0.0, l_max=1,
                                cgls=kb.CglsConfig(i_max=5, tau=0.0)))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    res = kb.sb_run(o, b, cfg)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    it = int(sum(res.cgls_iters))
    if label == "dense F":
        x0 = res.x if isinstance(res.x, np.ndarray) else D.to_host(res.x)
    x = res.x if isinstance(res.x, np.ndarray) else D.to_host(res.x)
    print(f"  {label:8s}: {ms:9.1f} ms  {it} CGLS it  {it / ms * 1e3:7.1f} it/s  band={getattr(o, '_band', None)} "
          f"fband={getattr(o, '_fband', None)}  |x - x_dense|/|x| = {np.linalg.norm(x - x0) / np.linalg.norm(x0):.2e}",
          flush=True)
