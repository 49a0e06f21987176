"""Run every BASELINE.json config's approximation engines on one GPU and print a table."""
import sys, os, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen

def timed(fn):
    torch.cuda.synchronize(); t = time.perf_counter(); r = fn(); torch.cuda.synchronize()
    return r, time.perf_counter() - t

out = {}
for name in sys.argv[1:] or ["n64", "n256", "n512", "n1024", "n2048"]:
    prob = datagen.make_problem(name)
    n = prob.n
    blur = kb.RearrangedBlur(prob.psf, n)
    cfg = kb.EgkbConfig(**prob.egkb)
    kb.egkb(blur, cfg)   # warm-up (graph / plan)
    (svd, tr), t = timed(lambda: kb.egkb(blur, cfg))
    rec = {"n": n, "egkb_ms": t * 1e3, "chosen_k": tr.chosen_k, "k_p": tr.k_p, "stop": tr.stop_reason,
           "breakdown": tr.breakdown, "sigma_head": [float(x) for x in svd.sigma[:4]]}
    if name == "n512":
        tsv, t2 = timed(lambda: kb.tsvd(blur, 20))
        rec["tsvd20_ms"] = t2 * 1e3
        try:
            rs, t3 = timed(lambda: kb.rsvd(blur, kb.RsvdConfig(k=20, p=10, q=2)))
            rec["rsvd_ms"] = t3 * 1e3
        except kb.RankDeficiencyError as e:
            rec["rsvd"] = f"RankDeficiencyError(column={e.column})"
        try:
            rs, t3 = timed(lambda: kb.rsvd(blur, kb.RsvdConfig(k=8, p=2, q=2)))
            rec["rsvd_k8p2_ms"] = t3 * 1e3
        except kb.RankDeficiencyError as e:
            rec["rsvd_k8p2"] = f"RankDeficiencyError(column={e.column})"
    op = kb.assemble(svd, kb.BlockScheme.square_image(n))
    variant = prob.sb["variant"] if prob.sb["variant"] != "both" else "isotropic"
    sbc = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=variant, tau=0.0, l_max=2,
                      cgls=kb.CglsConfig(100, 1e-4))
    kb.sb_run(op, prob.b, kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, l_max=1, cgls=kb.CglsConfig(2, 0.0)))
    res, t4 = timed(lambda: kb.sb_run(op, prob.b, sbc, x_true=prob.x_true))
    rec.update(sb_variant=variant, sb_2outer_ms=t4 * 1e3, sb_cgls_iters=res.cgls_iters,
               cgls_it_per_s=res.iota_total / t4, outer_it_per_s=res.outer_iters / t4)
    out[name] = rec
    print(json.dumps({name: rec}), flush=True)
