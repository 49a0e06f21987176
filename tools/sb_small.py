"""configs[0] (n=64) full pipeline on the GPU: eGKB 10+2 -> assemble -> 100 ANI SB sweeps."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
prob = datagen.make_problem("n64")
n = 64
blur = kb.RearrangedBlur(prob.psf, n)
cfg = kb.EgkbConfig(**prob.egkb)
sbc = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant="anisotropic", tau=0.0, l_max=100,
                  cgls=kb.CglsConfig(100, 1e-4))
for rep in range(3):
    torch.cuda.synchronize(); t = time.perf_counter()
    svd, tr = kb.egkb(blur, cfg)
    op = kb.assemble(svd, kb.BlockScheme.square_image(n))
    t1 = time.perf_counter()
    res = kb.sb_run(op, prob.b, sbc, x_true=prob.x_true)
    torch.cuda.synchronize(); t2 = time.perf_counter()
    print(f"egkb+assemble {1e3*(t1-t):.2f} ms, sb {1e3*(t2-t1):.1f} ms, cgls total {res.iota_total}, "
          f"{res.iota_total/(t2-t1):.0f} CGLS it/s, {res.outer_iters/(t2-t1):.1f} outer it/s, RE {res.re_history[-1]:.4f}")
