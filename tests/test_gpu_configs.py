"""Parity at the BASELINE.json config sizes (SURVEY §8c protocol), CUDA path vs the CPU oracle:

* Kronecker factors of the eGKB runs (assembled operator on random vectors, sign-aligned
  leading factors within 1e-4; kronop.py:103-123) at n = 256, 512, 1024;
* the Kronecker apply at n = 512 / 1024 -- the banded split-K DMMA path the bench times --
  against the oracle's dense apply (kronop.py:58-84);
* split Bregman on the GPU's own factors against oracle.sb with the same factors
  (splitbregman.py:120-192): the strict 1e-9 short protocol at n = 256 / 512 (both
  variants) and n = 1024, and configs[1]'s isotropic protocol with the data-dependent
  CGLS stop next to the measured CPU-vs-CPU drift;
* configs[2]: RSVD (k=20, p=10, q=2, fp32) raises RankDeficiencyError at the reference's
  column (lowrank.py:332-372, linalg.py:183-197); TSVD-20 against the exact structured
  singular values.
"""

from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


_CACHE = {}


def _problem(name):
    from paper_2410_00233_b200 import datagen

    if name not in _CACHE:
        _CACHE[name] = datagen.make_problem(name)
    return _CACHE[name]


def _oracle_egkb(prob, kernel=None):
    from oracle import lowrank as olr
    from oracle import structured as ost

    n = prob.n
    k32 = (prob.psf / prob.psf.sum()).astype(np.float32)
    e = dict(dict(k_min=2, p=2, tau=1e-4) | prob.egkb)
    ocfg = SimpleNamespace(reorth=None, seed=0, break_tol=None, keep_basis=False, **e)
    return olr.egkb(lambda q: ost.ra_matvec(k32, n, q), lambda s: ost.ra_rmatvec(k32, n, s), (n * n, n * n),
                    np.float32, ocfg, kernel=kernel)


def _oracle_factors(u, s, v, n):
    """assemble (kronop.py:117-119): A_x,i = sigma_i unvec(u_i), A_y,i = unvec(v_i), fp64."""
    ax = [np.float64(s[i]) * u[:, i].astype(np.float64).reshape((n, n), order="F") for i in range(s.size)]
    ay = [v[:, i].astype(np.float64).reshape((n, n), order="F") for i in range(s.size)]
    return ax, ay


def _gpu_factors(kb, prob, arithmetic):
    svd, tr = kb.egkb(kb.RearrangedBlur(prob.psf, prob.n), kb.EgkbConfig(**prob.egkb), arithmetic=arithmetic)
    op = kb.assemble(svd, kb.BlockScheme.square_image(prob.n))
    return svd, tr, op


@pytest.mark.parametrize("name", ["n256", "n512", "n1024"])
@pytest.mark.parametrize("arithmetic", ["reference", "fast"])
def test_factor_parity(kb, name, arithmetic):
    """north_star: Kronecker factors up to sign within 1e-4 relative (the
    assembled operator on random vectors, a sign-aligned per-factor check for
    sigma_i >= 1e-3 sigma_1)."""
    from oracle import sb as osb

    prob = _problem(name)
    n = prob.n
    svd, tr, op = _gpu_factors(kb, prob, arithmetic)
    (u, s, v), otr = _oracle_egkb(prob)
    oax, oay = _oracle_factors(u, s, v, n)
    ref_op = osb.KronOracle(oax, oay, n, n, n, n)
    rng = np.random.default_rng(9)
    for _ in range(3):
        x = rng.standard_normal(n * n)
        want, got = ref_op.apply(x), op.apply(x)
        assert np.linalg.norm(got - want) <= 1e-4 * np.linalg.norm(want)
        want, got = ref_op.apply_t(x), op.apply_t(x)
        assert np.linalg.norm(got - want) <= 1e-4 * np.linalg.norm(want)
    ax, ay = op.ax, op.ay
    lead = [i for i in range(min(len(ax), len(oax))) if s[i] >= 1e-3 * s[0]]
    assert len(lead) >= 3
    for i in lead:
        sg = np.sign(np.sum(ay[i] * oay[i]))
        assert np.linalg.norm(ay[i] - sg * oay[i]) <= 1e-4 * np.linalg.norm(oay[i]), (name, i)
        assert np.linalg.norm(ax[i] - sg * oax[i]) <= 1e-4 * np.linalg.norm(oax[i]), (name, i)
    if arithmetic == "reference":
        assert (tr.chosen_k, tr.k_p) == (otr.chosen_k, otr.k_p)


@pytest.mark.parametrize("name", ["n512", "n1024"])
def test_kron_apply_banded_vs_oracle(kb, name):
    """The apply the bench times (banded G-stage tile skip + split-K F stage, DMMA) on the
    eGKB factors against the oracle's dense Sum_i A_y,i X A_x,i^T (kronop.py:58-84)."""
    from oracle import sb as osb

    prob = _problem(name)
    n = prob.n
    _, _, op = _gpu_factors(kb, prob, "fast")
    ref = osb.KronOracle(op.ax, op.ay, n, n, n, n)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(n * n)
    for got, want in ((op.apply(x), ref.apply(x)), (op.apply_t(x), ref.apply_t(x))):
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


def _sb_pair(kb, prob, op, variant, l_max, i_max, tau_cgls):
    from oracle import sb as osb
    from paper_2410_00233_b200 import datagen

    n = prob.n
    cfg = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=variant, tau=0.0, l_max=l_max,
                      cgls=kb.CglsConfig(i_max=i_max, tau=tau_cgls))
    res = kb.sb_run(op, prob.b, cfg, x_true=prob.x_true)
    oop = osb.KronOracle(op.ax, op.ay, n, n, n, n)
    ores = osb.sb_run(oop, prob.b, datagen.LAM, datagen.BETA, variant=variant, tau=0.0, l_max=l_max, i_max=i_max,
                      tau_cgls=tau_cgls, x_true=prob.x_true)
    return res, ores, oop


def _drift(prob, oop, variant, l_max, i_max, tau_cgls, ref_x):
    """CPU-vs-CPU self-drift (SURVEY §8c ii): the oracle with the Kronecker terms summed in
    reverse order."""
    from oracle import sb as osb
    from paper_2410_00233_b200 import datagen

    class Reassoc(osb.KronOracle):
        def apply(self, x):
            xm = osb._unvec(x, self.n2, self.n1)
            acc = np.zeros((self.m2, self.m1))
            for a, b in reversed(list(zip(self.ax, self.ay))):
                acc += b @ (xm @ a.T)
            return osb._vec(acc)

    op2 = Reassoc(oop.ax, oop.ay, oop.m1, oop.m2, oop.n1, oop.n2)
    x2 = osb.sb_run(op2, prob.b, datagen.LAM, datagen.BETA, variant=variant, tau=0.0, l_max=l_max, i_max=i_max,
                    tau_cgls=tau_cgls).x
    return np.linalg.norm(x2 - ref_x) / np.linalg.norm(ref_x)


@pytest.mark.parametrize("name,variant,l_max,i_max", [
    ("n256", "isotropic", 5, 20), ("n256", "anisotropic", 5, 20),
    ("n512", "isotropic", 5, 20), ("n512", "anisotropic", 5, 20),
    ("n1024", "isotropic", 1, 8),
])
def test_sb_short_protocol(kb, name, variant, l_max, i_max):
    """fixed CGLS counts (tau=0), the GPU's own eGKB factors, both sides
    given the same factors: final image within 1e-9 (or 10x the CPU re-association
    drift where that drift itself exceeds 1e-10), RE history to 1e-7."""
    prob = _problem(name)
    _, _, op = _gpu_factors(kb, prob, "fast")
    res, ores, oop = _sb_pair(kb, prob, op, variant, l_max, i_max, 0.0)
    gap = np.linalg.norm(res.x - ores.x) / np.linalg.norm(ores.x)
    if gap > 1e-9:
        drift = _drift(prob, oop, variant, l_max, i_max, 0.0, ores.x)
        assert drift > 1e-10 and gap <= 10 * drift, (gap, drift)
    assert res.cgls_iters == ores.cgls_iters
    np.testing.assert_allclose(res.re_history, ores.re_history, rtol=1e-7)


def test_sb_config1_protocol(kb):
    """configs[1] (n=256, isotropic, CglsConfig(100, 1e-4), tau=0) for 20 of its 200 outer
    iterations: the data-dependent CGLS stop, the GPU-vs-CPU gap reported next to the CPU
    self-drift, CGLS counts within +-2 per outer iteration, RE within 1e-3."""
    prob = _problem("n256")
    _, _, op = _gpu_factors(kb, prob, "fast")
    res, ores, oop = _sb_pair(kb, prob, op, "isotropic", 20, 100, 1e-4)
    gap = np.linalg.norm(res.x - ores.x) / np.linalg.norm(ores.x)
    drift = _drift(prob, oop, "isotropic", 20, 100, 1e-4, ores.x)
    print(f"configs[1] iso: gpu-cpu gap {gap:.2e}, cpu-cpu drift {drift:.2e}, "
          f"cgls {res.cgls_iters} vs {ores.cgls_iters}")
    assert gap <= max(1e-6, 10 * drift), (gap, drift)
    assert all(abs(a - b) <= 2 for a, b in zip(res.cgls_iters, ores.cgls_iters))
    np.testing.assert_allclose(res.re_history, ores.re_history, rtol=1e-3)


def test_rsvd_config2_rank_deficiency_column(kb):
    """configs[2]: RSVD k=20, p=10, q=2 in fp32 on the n=512 blur raises RankDeficiencyError
    at the same column as the reference's orthonormalize (linalg.py:183-197; the oracle
    raises at column 7 with both the SkylakeX and the Haswell OpenBLAS kernel)."""
    from oracle import lowrank as olr
    from oracle import structured as ost

    prob = _problem("n512")
    n = prob.n
    k32 = (prob.psf / prob.psf.sum()).astype(np.float32)
    mm = lambda F: np.stack([ost.ra_matvec(k32, n, F[:, j]) for j in range(F.shape[1])], axis=1)   # noqa: E731
    rm = lambda Y: np.stack([ost.ra_rmatvec(k32, n, Y[:, j]) for j in range(Y.shape[1])], axis=1)  # noqa: E731
    with pytest.raises(olr.OracleRankDeficiency) as oe:
        olr.rsvd(mm, rm, (n * n, n * n), np.float32, 20, 10, 2, 0)
    with pytest.raises(kb.RankDeficiencyError) as ge:
        kb.rsvd(kb.RearrangedBlur(prob.psf, n), kb.RsvdConfig(k=20, p=10, q=2, seed=0))
    assert ge.value.column == oe.value.column, (ge.value.column, oe.value.column)


def test_tsvd_config2(kb):
    """configs[2] TSVD-20: the structured SVD of R(A) against the exact fp64 structured
    singular values (the reference's svd_small(rearrange(A)) cannot run at n=512)."""
    from oracle import structured as ost

    prob = _problem("n512")
    svd = kb.tsvd(kb.RearrangedBlur(prob.psf, prob.n), 20)
    _, s_exact, _ = ost.structured_tsvd(prob.psf, prob.n, k=20)
    assert svd.k == 20
    assert np.all(np.abs(svd.sigma - s_exact) <= 1e-4 * s_exact + 1e-6 * s_exact[0]), (svd.sigma, s_exact)


def test_rsvd_gram_reduction_vs_host_svd(kb):
    """fp32 RSVD at a config size: the device reduction of the wide block H (Gram matrix +
    k_p x k_p host eigenproblem, lowrank._svd_wide_gram) against the reference's host
    LAPACK SVD of H (lowrank.py:368-371) -- same sigma, same factors up to sign."""
    from paper_2410_00233_b200 import lowrank

    prob = _problem("n512")
    n = prob.n
    blur = kb.RearrangedBlur(prob.psf, n)
    cfg = kb.RsvdConfig(k=4, p=2, q=2, seed=0)
    dev = kb.rsvd(blur, cfg)
    old = lowrank._RSVD_GRAM_MIN
    lowrank._RSVD_GRAM_MIN = 1 << 62          # force the host path
    try:
        host = kb.rsvd(blur, cfg)
    finally:
        lowrank._RSVD_GRAM_MIN = old
    s_d, s_h = np.asarray(dev.sigma, np.float64), np.asarray(host.sigma, np.float64)
    assert np.all(np.abs(s_d - s_h) <= 1e-5 * s_h + 2e-6 * s_h[0]), (s_d, s_h)
    _, s_exact, _ = __import__("oracle.structured", fromlist=["x"]).structured_tsvd(prob.psf, n, k=4)
    assert np.all(np.abs(s_d - s_exact) <= 1e-4 * s_exact + 5e-6 * s_exact[0])
    for i in range(3):   # leading vectors (sigma_i well above the fp32 floor)
        for a, b in ((dev.u[:, i], host.u[:, i]), (dev.v[:, i], host.v[:, i])):
            a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
            sg = np.sign(a @ b)
            assert np.linalg.norm(a - sg * b) <= 2e-4, i
