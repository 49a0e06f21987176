"""Batched lambda sweep (splitbregman.py:195-235 `sweep`).

kb_sb_run_batch runs several SB problems in lock step (stacked GEMMs, one
launch per vector pass).  Each problem must reproduce sb_run of its own
config; the sweep records must match the reference's sequential sweep.
"""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


@pytest.fixture(scope="module")
def case(kb):
    g = load_golden("sb_kat")
    side = 32
    op = kb.KroneckerSum(list(g["n64_ax"]), list(g["n64_ay"]), kb.BlockScheme.square_image(side))
    return op, g["n64_b"], g["n64_xtrue"]


def _close(a, b, rel):
    return np.linalg.norm(np.asarray(a) - b) <= rel * max(np.linalg.norm(b), 1e-300)


@pytest.mark.parametrize("variant", ["anisotropic", "isotropic"])
@pytest.mark.parametrize("tau,tau_cgls,warm", [(0.0, 0.0, False), (2e-3, 1e-4, False), (0.0, 1e-4, True)])
def test_batch_of_one_is_bitwise_single(kb, case, variant, tau, tau_cgls, warm):
    """A batch of one runs exactly the kernels of sb_run: identical bits."""
    op, b, xt = case
    c = kb.SbConfig.from_gamma(0.1, 2.0, variant=variant, tau=tau, l_max=6, cgls=kb.CglsConfig(i_max=30, tau=tau_cgls),
                               warm_start=warm)
    (rb,) = kb.sb_run_batch(op, b, [c], x_true=xt)
    rs = kb.sb_run(op, b, c, x_true=xt)
    np.testing.assert_array_equal(rb.x, rs.x)
    assert (rb.outer_iters, rb.stop, rb.cgls_iters) == (rs.outer_iters, rs.stop, rs.cgls_iters)
    assert rb.rc_history == rs.rc_history and rb.re_history == rs.re_history


@pytest.mark.parametrize("variant", ["anisotropic", "isotropic"])
def test_batch_short_protocol_equals_single_runs(kb, case, variant):
    """SURVEY §8c (i) protocol (CGLS i_max=20, tau=0; l_max=5): per problem the
    batched run equals sb_run up to the split-K order of the stacked GEMMs."""
    op, b, xt = case
    lams = np.logspace(np.log10(0.03), np.log10(0.5), 7)
    cfgs = [kb.SbConfig.from_gamma(float(l), 2.0, variant=variant, tau=0.0, l_max=5,
                                   cgls=kb.CglsConfig(i_max=20, tau=0.0)) for l in lams]
    batch = kb.sb_run_batch(op, b, cfgs, x_true=xt)
    assert len(batch) == len(cfgs)
    for c, rb in zip(cfgs, batch):
        rs = kb.sb_run(op, b, c, x_true=xt)
        assert (rb.outer_iters, rb.stop, rb.cgls_iters) == (rs.outer_iters, rs.stop, rs.cgls_iters)
        assert _close(rb.x, rs.x, 1e-8), np.linalg.norm(rb.x - rs.x) / np.linalg.norm(rs.x)
        np.testing.assert_allclose(rb.re_history, rs.re_history, rtol=1e-8)


@pytest.mark.parametrize("variant", ["anisotropic", "isotropic"])
@pytest.mark.parametrize("warm", [False, True])
def test_batch_configured_protocol(kb, case, variant, warm):
    """Data-dependent stops (CGLS tau=1e-4, SB tau=2.6e-2): problems stop at
    different inner and outer iterations.  With the per-problem split-K
    (kb_sb_batch_exact) every problem is bit-identical to its own sb_run, which
    proves the masking; with the default stacked split-K the stagnating CGLS
    of the ill-conditioned problems may stop a few iterations apart (the same
    rounding sensitivity as GPU vs CPU, SURVEY §8c ii), RE within 1e-3."""
    from paper_2410_00233_b200 import _lib

    op, b, xt = case
    lams = np.logspace(np.log10(0.03), np.log10(0.5), 7)
    cfgs = [kb.SbConfig.from_gamma(float(l), 2.0, variant=variant, tau=2.6e-2, l_max=12,
                                   cgls=kb.CglsConfig(i_max=60, tau=1e-4), warm_start=warm) for l in lams]
    singles = [kb.sb_run(op, b, c, x_true=xt) for c in cfgs]
    lib = _lib.load()
    lib.kb_sb_batch_exact(1)
    try:
        exact = kb.sb_run_batch(op, b, cfgs, x_true=xt)
    finally:
        lib.kb_sb_batch_exact(0)
    for rs, rb in zip(singles, exact):
        np.testing.assert_array_equal(rb.x, rs.x)
        assert (rb.outer_iters, rb.stop, rb.cgls_iters, rb.re_history) == (rs.outer_iters, rs.stop, rs.cgls_iters,
                                                                            rs.re_history)
    assert len({r.outer_iters for r in exact}) > 1 or len({r.stop for r in exact}) > 1
    fast = kb.sb_run_batch(op, b, cfgs, x_true=xt)
    for rs, rb in zip(singles, fast):
        assert rb.outer_iters == rs.outer_iters and rb.stop == rs.stop
        np.testing.assert_allclose(rb.re_history, rs.re_history, rtol=1e-3)


def test_sweep_records_match_reference_semantics(kb, case):
    """sweep() through the batched path vs the oracle's sequential sb_run per grid point."""
    from oracle import sb as osb

    op, b, xt = case
    g = load_golden("sb_kat")
    recs = kb.sweep(op, b, gamma=2.0, lam_lo=0.05, lam_hi=0.5, count=4, x_true=xt, l_max=3,
                    cgls=kb.CglsConfig(i_max=15, tau=0.0), tau=0.0)
    assert len(recs) == 4
    korc = osb.KronOracle(list(g["n64_ax"]), list(g["n64_ay"]), 32, 32, 32, 32)
    for rec, lam in zip(recs, kb.lambda_grid(0.05, 0.5, 4)):
        assert rec["lam"] == pytest.approx(lam, rel=0, abs=0)
        assert rec["beta"] == pytest.approx(lam ** 2 / 2.0)
        ref = osb.sb_run(korc, b, float(lam), float(lam) ** 2 / 2.0, tau=0.0, l_max=3, i_max=15, tau_cgls=0.0,
                         x_true=xt)
        assert rec["outer_iters"] == 3 and rec["iota_total"] == 45
        assert rec["re"] == pytest.approx(ref.re_history[-1], rel=1e-8)
        assert np.isfinite(rec["isnr_db"])


def test_sweep_chunked_equals_unchunked(kb, case):
    op, b, xt = case
    kw = dict(gamma=2.0, lam_lo=0.05, lam_hi=0.5, count=5, x_true=xt, l_max=2, cgls=kb.CglsConfig(i_max=10, tau=1e-4))
    a = kb.sweep(op, b, batch=2, **kw)
    c = kb.sweep(op, b, **kw)
    for ra, rc in zip(a, c):
        assert ra["outer_iters"] == rc["outer_iters"] and ra["iota_total"] == rc["iota_total"]
        assert ra["re"] == pytest.approx(rc["re"], rel=1e-10)


def test_sweep_dense_operator_and_errors(kb):
    """The reference's own test case (test_splitbregman.py:192-211): dense A -> sequential path."""
    n = 8
    a = kb.build_blur_matrix(kb.Psf(np.ones((3, 3))), n)
    x_true = kb.vec(kb.make_test_image(n))
    b = a @ x_true
    records = kb.sweep(a, b, gamma=2.0, lam_lo=0.05, lam_hi=0.5, count=3, x_true=x_true, l_max=3)
    assert len(records) == 3
    for rec in records:
        assert rec["beta"] == pytest.approx(rec["lam"] ** 2 / 2.0)
        assert np.isfinite(rec["re"]) and rec["iota_total"] > 0
    records = kb.sweep(a, b, gamma=2.0, lam_lo=0.05, lam_hi=0.5, count=2, l_max=2)
    assert all(np.isnan(rec["re"]) for rec in records)
    with pytest.raises(kb.ValidationError):
        kb.sb_run_batch(a, b, [kb.SbConfig(0.1, 0.01), kb.SbConfig(0.1, 0.01, l_max=3)])
