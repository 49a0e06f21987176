"""R(A) of an unstructured sparse A on the GPU: CSR products
and the eGKB / RSVD engines on them, against the reference's dense runs."""

import json

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _cfg(kb, js):
    return kb.EgkbConfig(**json.loads(str(js)))


def sigma_ok(got, ref, floor=2e-6):
    got, ref = np.asarray(got, dtype=np.float64), np.asarray(ref, dtype=np.float64)
    return bool(np.all(np.abs(got - ref) <= 1e-4 * ref + floor * ref[0]))


def _scheme(kb, g):
    return kb.BlockScheme(*(int(v) for v in g["s1_scheme"]))


def test_products_match_dense(kb):
    g = load_golden("ra_sparse")
    rng = np.random.default_rng(0)
    for key, scheme in (("s1", _scheme(kb, g)), ("s2", kb.BlockScheme.square_image(int(g["s2_n"])))):
        R = g[f"{key}_R"]
        op = kb.RearrangedSparse(g[f"{key}_a"], scheme, dtype=np.float64)
        x = rng.standard_normal(R.shape[1])
        y = rng.standard_normal(R.shape[0])
        np.testing.assert_allclose(op.matvec(x), R @ x, rtol=0, atol=1e-13)
        np.testing.assert_allclose(op.rmatvec(y), R.T @ y, rtol=0, atol=1e-13)
        op32 = kb.RearrangedSparse(g[f"{key}_a"], scheme)
        got = op32.matvec(x.astype(np.float32))
        assert got.dtype == np.float32
        assert np.linalg.norm(got - R @ x) <= 1e-6 * np.linalg.norm(R @ x)


@pytest.mark.parametrize("tag,dtype", [("s1d_", np.float64), ("s1s_", np.float32)])
def test_egkb_kats(kb, tag, dtype):
    g = load_golden("ra_sparse")
    op = kb.RearrangedSparse(g["s1_a"], _scheme(kb, g), dtype=dtype)
    svd, tr = kb.egkb(op, _cfg(kb, g[tag + "cfg"]))
    assert (tr.chosen_k, tr.k_p, tr.stop_reason) == (int(g[tag + "tr_chosen_k"]), int(g[tag + "tr_k_p"]),
                                                     str(g[tag + "tr_stop_reason"]))
    if dtype == np.float64:
        np.testing.assert_allclose(svd.sigma, g[tag + "sigma"], rtol=1e-10)
        np.testing.assert_allclose(np.abs(svd.u.T @ g[tag + "u"]).diagonal(), 1.0, atol=1e-8)
    else:
        assert sigma_ok(svd.sigma, g[tag + "sigma"])


@pytest.mark.parametrize("tag", ["s2s_", "s2d_"])
def test_egkb_spatially_variant_blur(kb, tag):
    g = load_golden("ra_sparse")
    n = int(g["s2_n"])
    dtype = np.float32 if tag == "s2s_" else np.float64
    op = kb.RearrangedSparse(g["s2_a"], kb.BlockScheme.square_image(n), dtype=dtype)
    svd, tr = kb.egkb(op, _cfg(kb, g[tag + "cfg"]))
    assert (tr.chosen_k, tr.k_p, tr.stop_reason) == (int(g[tag + "tr_chosen_k"]), int(g[tag + "tr_k_p"]),
                                                     str(g[tag + "tr_stop_reason"]))
    assert sigma_ok(svd.sigma, g[tag + "sigma"], floor=1e-10 if dtype == np.float64 else 2e-6)


def test_rsvd_wide_sparse(kb):
    """R is 24 x 35 (wide): rsvd runs on R^T (lowrank.py:352-354) by swapping the CSR copies."""
    g = load_golden("ra_sparse")
    op = kb.RearrangedSparse(g["s1_a"], _scheme(kb, g), dtype=np.float64)
    svd = kb.rsvd(op, kb.RsvdConfig(k=4, p=3, q=2, seed=6))
    np.testing.assert_allclose(svd.sigma, g["s1_rsvd_sigma"], rtol=1e-10)
    assert svd.u.shape == (24, 4) and svd.v.shape == (35, 4)


def test_large_sparse_vs_oracle(kb):
    """n=128 spatially variant blur (PSF + sparse couplings), fp32 eGKB vs the oracle
    restatement over a numpy CSR product."""
    from oracle import lowrank as olr
    from test_gpu_engines import _ocfg

    n = 128
    N = n * n
    rng = np.random.default_rng(5)
    # 7x7 box-ish PSF band + 2 random long-range couplings per row
    r_idx, c_idx, vals = [], [], []
    img = np.arange(N).reshape(n, n, order="F")
    for du in range(-3, 4):
        for dv in range(-3, 4):
            rr, cc = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
            ri, ci = rr - du, cc - dv
            ok = (ri >= 0) & (ri < n) & (ci >= 0) & (ci < n)
            r_idx.append(img[rr[ok], cc[ok]])
            c_idx.append(img[ri[ok], ci[ok]])
            vals.append(np.full(ok.sum(), np.exp(-(du * du + dv * dv) / 6.0)))
    r_idx.append(np.repeat(np.arange(N), 2))
    c_idx.append(rng.integers(0, N, 2 * N))
    vals.append(rng.random(2 * N) * 0.02)
    rows, cols, v = np.concatenate(r_idx), np.concatenate(c_idx), np.concatenate(vals)
    scheme = kb.BlockScheme.square_image(n)
    op = kb.RearrangedSparse((rows, cols, v, (N, N)), scheme)
    cfg = kb.EgkbConfig(k_max=16, tau=1e-4)
    svd, tr = kb.egkb(op, cfg)
    from paper_2410_00233_b200.sparse import _csr

    m1 = m2 = n1 = n2 = n
    i, p = np.divmod(rows, m2)
    j, q = np.divmod(cols, n2)
    rp, ci, va = _csr(j * m1 + i, q * m2 + p, v, N)
    va32 = va.astype(np.float32)
    rid = np.repeat(np.arange(N), np.diff(rp))

    def mv(x):
        return np.bincount(rid, weights=va32.astype(np.float64) * x[ci], minlength=N).astype(np.float32)

    def rmv(y):
        return np.bincount(ci, weights=va32.astype(np.float64) * y[rid], minlength=N).astype(np.float32)

    (_, os_, _), otr = olr.egkb(mv, rmv, (N, N), np.float32, _ocfg(cfg))
    assert (tr.chosen_k, tr.stop_reason) == (otr.chosen_k, otr.stop_reason)
    m = min(svd.k, os_.size)
    assert sigma_ok(svd.sigma[:m], os_[:m], floor=5e-6)
