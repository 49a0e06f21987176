"""Pin the CPU oracle against fixtures produced by the reference itself.

The fixtures in tests/golden/ were written by tests/golden/make_golden.py,
which runs the unmodified reference package.  On dense inputs the oracle
must be BIT-IDENTICAL to the reference (same float ops, same order); the
closed-form structured R(A) must match the dense rearrange(build_blur_matrix)
to rounding.
"""

import json
from types import SimpleNamespace

import numpy as np
import pytest

from conftest import load_golden
from oracle import lowrank as olr
from oracle import sb as osb
from oracle import structured as ost


def _cfg(js):
    d = dict(k_max=1, p=2, tau=1e-4, k_min=2, reorth=None, seed=0, break_tol=None, keep_basis=False)
    d.update(json.loads(str(js)))
    return SimpleNamespace(**d)


class TestStructuredRA:
    def test_closed_form_matches_reference_dense(self):
        g = load_golden("ra_structured")
        for i in range(5):
            k, n = g[f"c{i}_psf"], int(g[f"c{i}_n"])
            np.testing.assert_allclose(ost.ra_matvec(k, n, g[f"c{i}_q"]), g[f"c{i}_Rq"], rtol=0, atol=1e-14)
            np.testing.assert_allclose(ost.ra_rmatvec(k, n, g[f"c{i}_s"]), g[f"c{i}_RTs"], rtol=0, atol=1e-14)
            _, sig, _ = ost.structured_tsvd(k, n)
            ref = g[f"c{i}_sigma"][: sig.size]
            np.testing.assert_allclose(sig, ref, rtol=0, atol=1e-13 * ref[0])

    def test_padded_even_psf(self):
        g = load_golden("ra_structured")
        k, n = g["pad_psf"], int(g["pad_n"])
        assert k.shape == (n + 1, n + 1)
        np.testing.assert_allclose(ost.ra_matvec(k, n, g["pad_q"]), g["pad_Rq"], atol=1e-15)
        np.testing.assert_allclose(ost.ra_rmatvec(k, n, g["pad_s"]), g["pad_RTs"], atol=1e-15)
        np.testing.assert_array_equal(ost.ra_dense(k, n) @ g["pad_q"] != 0, g["pad_Rq"] != 0)

    def test_datagen_blur_equals_reference_blur_matrix(self):
        from paper_2410_00233_b200 import datagen

        g = load_golden("ra_structured")
        n = int(g["pad_n"])
        x = g["pad_x"].reshape(n, n, order="F")
        got = datagen.blur(x, g["pad_psf"]).reshape(-1, order="F")
        np.testing.assert_allclose(got, g["pad_Ax"], rtol=0, atol=1e-15)


class TestReflexiveRA:
    """Reflexive BC (blurmodel.py:80-84, 122-126) vs the reference's dense R."""

    def test_dense_products_and_sigma(self):
        g = load_golden("ra_reflexive")
        for i in range(int(g["ncases"])):
            k, n = g[f"c{i}_psf"], int(g[f"c{i}_n"])
            np.testing.assert_allclose(ost.ra_dense(k, n, "reflexive"), g[f"c{i}_R"], rtol=0, atol=1e-15)
            np.testing.assert_allclose(ost.ra_matvec(k, n, g[f"c{i}_q"], "reflexive"), g[f"c{i}_Rq"],
                                       rtol=0, atol=1e-14)
            np.testing.assert_allclose(ost.ra_rmatvec(k, n, g[f"c{i}_s"], "reflexive"), g[f"c{i}_RTs"],
                                       rtol=0, atol=1e-14)
            u, sig, v = ost.structured_tsvd(k, n, bc="reflexive")
            ref = g[f"c{i}_sigma"][: sig.size]
            np.testing.assert_allclose(sig, ref, rtol=0, atol=1e-13 * ref[0])
            np.testing.assert_allclose((u * sig) @ v.T, g[f"c{i}_R"], atol=1e-13)

    def test_gram_is_incidence_gram(self):
        for n, c, length in [(7, 6, 13), (8, 1, 3), (6, 2, 5)]:
            p = ost.incidence(n, c, length, "reflexive")
            np.testing.assert_array_equal(ost.gram(n, c, length, "reflexive"), p.T @ p)
            assert p.max() == 1.0   # a cell hits an index at most once

    def test_egkb_blur_configs(self):
        """The oracle eGKB on the structured reflexive operator reproduces the
        reference's dense fp32 run (rank decisions exactly, sigma to 1e-4)."""
        from oracle import lowrank as olr

        g = load_golden("ra_reflexive")
        for name in ("n64", "n256"):
            pre = f"blur_{name}_"
            from paper_2410_00233_b200 import blurmodel

            n = int(g[pre + "n"])
            k32 = blurmodel.Psf(g[pre + "psf"]).kernel.astype(np.float32)   # Psf: unit sum (blurmodel.py:25-65)
            mv = lambda q: ost.ra_matvec(k32, n, q, "reflexive")
            rmv = lambda x: ost.ra_rmatvec(k32, n, x, "reflexive")
            (_, s, _), tr = olr.egkb(mv, rmv, (n * n, n * n), np.float32, _cfg(g[pre + "cfg"]))
            assert (tr.chosen_k, tr.k_p, tr.stop_reason) == (int(g[pre + "tr_chosen_k"]), int(g[pre + "tr_k_p"]),
                                                             str(g[pre + "tr_stop_reason"]))
            ref = g[pre + "sigma"].astype(np.float64)
            big = ref >= 1e-3 * ref[0]
            np.testing.assert_allclose(s[big], ref[big], rtol=1e-4)


def _dense(b):
    return (lambda q: b @ q), (lambda s: b.T @ s)


@pytest.mark.parametrize("tag,bkey,dtype", [
    ("diag_", None, np.float64),
    ("rank5_", "rank5_b", np.float64),
    ("fact64_", "fact_b", np.float64),
    ("fact32_", "fact_b", np.float32),
    ("decay_", "decay_b", np.float64),
    ("decay32_", "decay_b", np.float32),
    ("accept3_", "accept3_b", np.float64),
    ("accept3s_", "accept3_b", np.float32),
    ("y0_", "y0_b", np.float64),
])
def test_egkb_bit_identical_on_dense(tag, bkey, dtype):
    g = load_golden("egkb_kat")
    b = np.diag([5.0, 3.0, 1.0]) if bkey is None else g[bkey]
    b = b.astype(dtype)
    mv, rmv = _dense(b)
    y0 = g["y0_y0"] if tag == "y0_" else None
    (u, s, v), tr = olr.egkb(mv, rmv, b.shape, b.dtype, _cfg(g[tag + "cfg"]), y0=y0)
    np.testing.assert_array_equal(s, g[tag + "sigma"])
    np.testing.assert_array_equal(u, g[tag + "u"])
    np.testing.assert_array_equal(v, g[tag + "v"])
    assert tr.chosen_k == int(g[tag + "tr_chosen_k"])
    assert tr.k_p == int(g[tag + "tr_k_p"])
    assert tr.stop_reason == str(g[tag + "tr_stop_reason"])
    assert tr.breakdown == bool(g[tag + "tr_breakdown"])
    np.testing.assert_array_equal(tr.alphas, g[tag + "tr_alphas"])
    np.testing.assert_array_equal(tr.nus, g[tag + "tr_nus"])


@pytest.mark.parametrize("name", ["n64", "n256"])
def test_egkb_structured_blur_matches_reference(name):
    """Structured matvec (fp64 accumulation) vs the reference's dense fp32 R."""
    g = load_golden("egkb_kat")
    pre = f"blur_{name}_"
    k, n = g[pre + "psf"], int(g[pre + "n"])
    mv = lambda q: ost.ra_matvec(k.astype(np.float32), n, q)
    rmv = lambda s: ost.ra_rmatvec(k.astype(np.float32), n, s)
    (u, s, v), tr = olr.egkb(mv, rmv, (n * n, n * n), np.float32, _cfg(g[pre + "cfg"]))
    assert tr.chosen_k == int(g[pre + "tr_chosen_k"])
    assert tr.k_p == int(g[pre + "tr_k_p"])
    assert tr.stop_reason == str(g[pre + "tr_stop_reason"])
    ref = g[pre + "sigma"].astype(np.float64)
    # SURVEY §8c sigma bar: 1e-4 relative + an fp32 floor relative to sigma_1
    assert np.all(np.abs(s - ref) <= 1e-4 * ref + 2e-6 * ref[0])


def test_rsvd_and_orthonormalize_bit_identical():
    g = load_golden("rsvd_kat")
    for tag, dt in (("d", np.float64), ("s", np.float32)):
        b = g["sig_b"].astype(dt)
        u, s, v = olr.rsvd(lambda f: b @ f, lambda y: b.T @ y, b.shape, b.dtype, 5, 8, 2, 2,
                           hmat=lambda y: y.T @ b)
        np.testing.assert_array_equal(s, g[f"sig{tag}_sigma"])
        np.testing.assert_array_equal(u, g[f"sig{tag}_u"])
        np.testing.assert_array_equal(v, g[f"sig{tag}_v"])
    b = g["wide_b"]
    u, s, v = olr.rsvd(lambda f: b @ f, lambda y: b.T @ y, b.shape, b.dtype, 4, 6, 2, 3)
    np.testing.assert_allclose(s, g["wide_sigma"], rtol=1e-12)
    with pytest.raises(olr.OracleRankDeficiency) as err:
        b = g["rankdef_b"]
        olr.rsvd(lambda f: b @ f, lambda y: b.T @ y, b.shape, b.dtype, 4, 2, 1, 5)
    assert err.value.column == int(g["rankdef_col"])
    np.testing.assert_array_equal(olr.orthonormalize(g["orth_in"]), g["orth_out"])
    np.testing.assert_array_equal(olr.orthonormalize(g["orth_in"].astype(np.float32)), g["orth32_out"])


def test_auto_rank_known_answers():
    assert olr.auto_rank((9, 4, 1, 0.5, 0.7), 1e-3) == (4, "nu_rose")
    assert olr.auto_rank((9, 4, 2e-4, 1e-4, 5e-5), 1e-3) == (3, "nu_below_tol")
    assert olr.auto_rank((9, 8, 7, 6, 5), 1e-6) == (5, "hit_kmax")
    assert olr.auto_rank((1, 5, 4, 3), 1e-9, k_min=2) == (2, "nu_rose")
    assert olr.auto_rank((9, 1e-5, 2e-5, 1e-6), 1e-3, k_min=1) == (2, "nu_below_tol")


def test_cgls_bit_identical():
    g = load_golden("cgls_kat")
    for i in range(4):
        res = osb.cgls(osb.DenseOracle(g[f"c{i}_a"]), g[f"c{i}_b"], 40, 1e-6 if i % 2 else 0.0)
        np.testing.assert_array_equal(res.x, g[f"c{i}_x"])
        assert res.iters == int(g[f"c{i}_iters"]) and res.stop == str(g[f"c{i}_stop"])
        np.testing.assert_array_equal(res.rc_history, g[f"c{i}_rc"])


def test_sb_bit_identical():
    from paper_2410_00233_b200 import datagen

    g = load_golden("sb_kat")
    n = 8
    a = g["inter_a"]
    x = osb.sb_run(osb.DenseOracle(a), g["inter_b"], 0.1, 0.005, tau=0.0, l_max=5, i_max=12, tau_cgls=0.0).x
    np.testing.assert_array_equal(x, g["inter_dense_x"])
    op = osb.KronOracle(list(g["inter_ax"]), list(g["inter_ay"]), n, n, n, n)
    x = osb.sb_run(op, g["inter_b"], 0.1, 0.005, tau=0.0, l_max=5, i_max=12, tau_cgls=0.0).x
    np.testing.assert_array_equal(x, g["inter_kron_x"])
    side = 32
    op = osb.KronOracle(list(g["n64_ax"]), list(g["n64_ay"]), side, side, side, side)
    for variant in ("anisotropic", "isotropic"):
        res = osb.sb_run(op, g["n64_b"], datagen.LAM, datagen.BETA, variant=variant, tau=0.0, l_max=5,
                         i_max=20, tau_cgls=0.0, x_true=g["n64_xtrue"])
        np.testing.assert_array_equal(res.x, g[f"n64_{variant}_short_x"])
        res = osb.sb_run(op, g["n64_b"], datagen.LAM, datagen.BETA, variant=variant, tau=0.0, l_max=10,
                         i_max=100, tau_cgls=1e-4, x_true=g["n64_xtrue"])
        np.testing.assert_array_equal(res.x, g[f"n64_{variant}_cfg_x"])
        assert res.cgls_iters == list(g[f"n64_{variant}_cfg_iters"])


class TestSparseRearrangement:
    """the host permutation of sparse entries equals rearrange.py:67-75."""

    def test_permutation_matches_reference(self):
        from paper_2410_00233_b200 import BlockScheme, RearrangedSparse

        g = load_golden("ra_sparse")
        m1, m2, n1, n2 = (int(v) for v in g["s1_scheme"])
        op = RearrangedSparse(g["s1_a"], BlockScheme(m1, m2, n1, n2), dtype=np.float64)
        assert op.shape == g["s1_R"].shape
        np.testing.assert_array_equal(op.to_dense(), g["s1_R"])
        n = int(g["s2_n"])
        op2 = RearrangedSparse(g["s2_a"], BlockScheme.square_image(n))
        np.testing.assert_array_equal(op2.to_dense(), g["s2_R"])
        np.testing.assert_array_equal(op.T.to_dense(), g["s1_R"].T)

    def test_csr_builder_sums_duplicates(self):
        from paper_2410_00233_b200.sparse import _csr

        rows = np.array([2, 0, 2, 1, 2])
        cols = np.array([1, 3, 1, 0, 0])
        vals = np.array([1.0, 2.0, 3.0, 4.0, 5.0])
        rp, ci, va = _csr(rows, cols, vals, 4)
        assert rp.tolist() == [0, 1, 2, 4, 4]
        assert ci.tolist() == [3, 0, 0, 1]
        assert va.tolist() == [2.0, 4.0, 5.0, 4.0]

    def test_validation(self):
        from paper_2410_00233_b200 import BlockScheme, RearrangedSparse, ValidationError

        with pytest.raises(ValidationError):
            RearrangedSparse(np.ones((6, 6)), BlockScheme(2, 2, 2, 2))
        with pytest.raises(ValidationError):
            RearrangedSparse(([0], [9], [1.0], (4, 4)), BlockScheme(2, 2, 2, 2))


def test_kernel_product_is_sequential_in_index_order():
    """oracle.structured._kernel_product: each z entry a sequential fp64 sum of rounded
    products in index order (the order the device's reference-order product repeats)."""
    from oracle import structured as ost

    rng = np.random.default_rng(3)
    for kh, kw in [(1, 1), (7, 9), (129, 65), (1025, 1025)]:
        k = rng.standard_normal((kh, kw)).astype(np.float32)
        for transpose, m in ((False, kh), (True, kw)):
            w = rng.standard_normal(m) * 10.0 ** rng.uniform(-6, 6, m)
            want = np.zeros(kw if not transpose else kh)
            for i in range(m):
                want += (k[i].astype(np.float64) if not transpose else k[:, i].astype(np.float64)) * w[i]
            assert np.array_equal(ost._kernel_product(k, w, transpose), want)
