"""Reflexive-BC R(A) on the GPU (blurmodel.py:80-84, 122-126).

Every kernel family that applies R(A) -- the cooperative single/block
product (k_ra_block), the persistent eGKB (k_egkb_persistent), the eager
operator path and the structured TSVD lift -- against the reference's dense
reflexive R (golden fixtures) and the oracle restatement at larger sides.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import ROOT, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-300))


def sigma_ok(got, ref, floor=1e-6):
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return bool(np.all(np.abs(got - ref) <= 1e-4 * ref + floor * ref[0]))


def test_products_match_reference_dense(kb):
    g = load_golden("ra_reflexive")
    for i in range(int(g["ncases"])):
        k, n = g[f"c{i}_psf"], int(g[f"c{i}_n"])
        op = kb.RearrangedBlur(k, n, bc="reflexive", dtype=np.float64)
        np.testing.assert_allclose(op.matvec(g[f"c{i}_q"]), g[f"c{i}_Rq"], rtol=0, atol=1e-14)
        np.testing.assert_allclose(op.rmatvec(g[f"c{i}_s"]), g[f"c{i}_RTs"], rtol=0, atol=1e-14)
        op32 = kb.RearrangedBlur(k, n, bc="reflexive")
        assert _rel(op32.matvec(g[f"c{i}_q"].astype(np.float32)), g[f"c{i}_Rq"]) < 1e-6
        assert _rel(op32.rmatvec(g[f"c{i}_s"].astype(np.float32)), g[f"c{i}_RTs"]) < 1e-6


def test_block_products(kb):
    """RSVD block products (lowrank.py:363-367): one cooperative launch per 16 vectors."""
    import torch

    from paper_2410_00233_b200 import device as D
    from paper_2410_00233_b200.lowrank import _EngineOp

    g = load_golden("ra_reflexive")
    k, n = g["c2_psf"], int(g["c2_n"])
    R = g["c2_R"]
    rng = np.random.default_rng(7)
    X = rng.standard_normal((21, n * n))
    op = _EngineOp(kb.RearrangedBlur(k, n, bc="reflexive", dtype=np.float64))
    Y = D.to_host(op.apply_block(D.to_device(X), 0))
    np.testing.assert_allclose(Y, X @ R.T, atol=1e-13)
    Z = D.to_host(op.apply_block(D.to_device(X), 1))
    np.testing.assert_allclose(Z, X @ R, atol=1e-13)
    torch.cuda.synchronize()


@pytest.mark.parametrize("n", [64, 256, 1024])
def test_large_sides_against_oracle(kb, n):
    from oracle import structured as ost
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(n)
    rng = np.random.default_rng(n)
    q = rng.standard_normal(n * n).astype(np.float32)
    k32 = kb.Psf(psf).kernel.astype(np.float32)
    op = kb.RearrangedBlur(psf, n, bc="reflexive")
    assert _rel(op.matvec(q), ost.ra_matvec(k32, n, q, "reflexive")) < 2e-7
    assert _rel(op.rmatvec(q), ost.ra_rmatvec(k32, n, q, "reflexive")) < 2e-7
    op64 = kb.RearrangedBlur(psf, n, bc="reflexive", dtype=np.float64)
    k64 = kb.Psf(psf).kernel
    q64 = q.astype(np.float64)
    assert _rel(op64.matvec(q64), ost.ra_matvec(k64, n, q64, "reflexive")) < 1e-13
    x, y = rng.standard_normal(n * n), rng.standard_normal(n * n)
    assert op64.matvec(x) @ y == pytest.approx(x @ op64.rmatvec(y), rel=1e-12)


@pytest.mark.parametrize("name", ["n64", "n256"])
def test_egkb_blur_configs_vs_reference(kb, name):
    """Persistent eGKB on the structured reflexive R vs the reference's dense fp32 run."""
    import json

    g = load_golden("ra_reflexive")
    pre = f"blur_{name}_"
    n = int(g[pre + "n"])
    cfg = kb.EgkbConfig(**json.loads(str(g[pre + "cfg"])))
    svd, tr = kb.egkb(kb.RearrangedBlur(g[pre + "psf"], n, bc="reflexive"), cfg)
    assert (tr.chosen_k, tr.k_p, tr.stop_reason) == (int(g[pre + "tr_chosen_k"]), int(g[pre + "tr_k_p"]),
                                                     str(g[pre + "tr_stop_reason"]))
    assert sigma_ok(svd.sigma, g[pre + "sigma"], floor=5e-6)
    np.testing.assert_allclose(tr.alphas[:4], g[pre + "tr_alphas"][:4], rtol=1e-4)


@pytest.mark.parametrize("n,name", [(256, "n256"), (512, "n512")])
def test_egkb_large_vs_oracle(kb, n, name):
    from oracle import lowrank as olr
    from oracle import structured as ost
    from paper_2410_00233_b200 import datagen
    from test_gpu_engines import _ocfg

    psf = datagen.mixture_psf(n)
    cfg = kb.EgkbConfig(**datagen.CONFIGS[name]["egkb"])
    svd, tr = kb.egkb(kb.RearrangedBlur(psf, n, bc="reflexive"), cfg)
    k32 = kb.Psf(psf).kernel.astype(np.float32)
    mv = lambda q: ost.ra_matvec(k32, n, q, "reflexive")
    rmv = lambda x: ost.ra_rmatvec(k32, n, x, "reflexive")
    (_, os_, _), otr = olr.egkb(mv, rmv, (n * n, n * n), np.float32, _ocfg(cfg))
    assert tr.stop_reason == otr.stop_reason
    if not otr.breakdown:
        assert (tr.chosen_k, tr.k_p) == (otr.chosen_k, otr.k_p)
    _, s_exact, _ = ost.structured_tsvd(kb.Psf(psf).kernel, n, k=svd.k, bc="reflexive")
    lead = s_exact >= 1e-3 * s_exact[0]
    assert np.all(np.abs(svd.sigma[lead] - s_exact[lead]) <= 1e-4 * s_exact[lead])


def test_tsvd_structured(kb):
    from oracle import structured as ost

    g = load_golden("ra_reflexive")
    for i in (0, 2, 4, 5):
        k, n = g[f"c{i}_psf"], int(g[f"c{i}_n"])
        kk = min(5, min(k.shape))
        svd = kb.tsvd(kb.RearrangedBlur(k, n, bc="reflexive", dtype=np.float64), kk)
        np.testing.assert_allclose(svd.sigma, g[f"c{i}_sigma"][:kk], rtol=1e-12)
        u, s, v = ost.structured_tsvd(k, n, k=kk, bc="reflexive")
        np.testing.assert_allclose((svd.u * svd.sigma) @ svd.v.T, (u * s) @ v.T, atol=1e-12)
        full = kb.tsvd(kb.RearrangedBlur(k, n, bc="reflexive", dtype=np.float64), min(k.shape))
        np.testing.assert_allclose((full.u * full.sigma) @ full.v.T, g[f"c{i}_R"], atol=1e-12)


def test_rsvd_structured(kb):
    from oracle import structured as ost
    from paper_2410_00233_b200 import datagen

    n = 128
    psf = datagen.mixture_psf(n)
    svd = kb.rsvd(kb.RearrangedBlur(psf, n, bc="reflexive", dtype=np.float64), kb.RsvdConfig(k=6, p=4, q=2))
    _, s_exact, _ = ost.structured_tsvd(kb.Psf(psf).kernel, n, k=6, bc="reflexive")
    np.testing.assert_allclose(svd.sigma, s_exact, rtol=1e-8)


def test_eager_paths_match(kb):
    """The non-persistent engine (separate kernels, KB_EGKB_NO_PERSISTENT) gives the
    same reflexive eGKB trace as the persistent kernel."""
    code = r'''
import json, sys, numpy as np
sys.path.insert(0, %r)
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import datagen
psf = datagen.mixture_psf(96)
svd, tr = kb.egkb(kb.RearrangedBlur(psf, 96, bc="reflexive"), kb.EgkbConfig(k_max=12, k_min=12, p=2, tau=1e300))
print(json.dumps([tr.chosen_k, tr.k_p, tr.stop_reason, [float(x) for x in svd.sigma]]))
''' % ROOT
    outs = []
    for env_extra in ({}, {"KB_EGKB_NO_PERSISTENT": "1"}):
        env = dict(os.environ, **env_extra)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(r.stdout.strip().splitlines()[-1])
    import json

    a, b = (json.loads(o) for o in outs)
    assert a[:3] == b[:3]
    assert sigma_ok(b[3], a[3], floor=5e-6)   # the two engines sum in different orders
