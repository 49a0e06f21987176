"""Batched lambda sweep vs one sb_run per lambda (device time, CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen

def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t = time.perf_counter(); a.record(); out = fn(); b.record(); torch.cuda.synchronize()
    return out, a.elapsed_time(b), (time.perf_counter() - t) * 1e3

for name, count, l_max in (("n64", 100, 5), ("n256", 100, 3), ("n512", 20, 2), ("n1024", 8, 1)):
    prob = datagen.make_problem(name)
    n = prob.n
    svd, tr = kb.egkb(kb.RearrangedBlur(prob.psf, n), kb.EgkbConfig(**prob.egkb))
    op = kb.assemble(svd, kb.BlockScheme.square_image(n))
    kw = dict(gamma=datagen.LAM ** 2 / datagen.BETA, lam_lo=0.01, lam_hi=1.0, count=count, x_true=prob.x_true,
              l_max=l_max, tau=0.0, cgls=kb.CglsConfig(100, 1e-4))
    kb.sweep(op, prob.b, **dict(kw, count=2))
    recs, ms_b, wall_b = timed(lambda: kb.sweep(op, prob.b, **kw))
    grid = kb.lambda_grid(0.01, 1.0, count)
    cfgs = [kb.SbConfig.from_gamma(float(l), kw["gamma"], l_max=l_max, tau=0.0, cgls=kw["cgls"]) for l in grid]
    kb.sb_run(op, prob.b, cfgs[0], x_true=prob.x_true)
    seq, ms_s, wall_s = timed(lambda: [kb.sb_run(op, prob.b, c, x_true=prob.x_true) for c in cfgs])
    it_b = sum(r["iota_total"] for r in recs)
    it_s = sum(r.iota_total for r in seq)
    print(f"{name}: k={op.k} {count} lambdas x {l_max} outer: batched {ms_b:.1f} ms ({it_b} CGLS its, "
          f"{it_b / ms_b * 1e3:.0f} it/s), sequential {ms_s:.1f} ms ({it_s} its, {it_s / ms_s * 1e3:.0f} it/s), "
          f"speed-up {ms_s / ms_b:.2f}x")
