"""KroneckerSum.toeplitz_split (opt-in): the (k+1)-term operator with the zero-BC eGKB
structure made explicit -- k banded x banded terms (plus one dense x banded term when the
start vector's share is not at the rounding level; forced with dense_tol=0 here), both
GEMM stages skipping all-zero k tiles (kb_kron.fband / ndense).

* what the split drops is at the fp32 rounding level of the factors (SURVEY §8c factor bar:
  1e-4) and the split operator agrees with the original on random vectors;
* the split operator's apply (kronop.py:58-84) and a split-Bregman solve on it
  (splitbregman.py:120-192) match the CPU oracle run on the split operator's own factors
  (1e-12 / the strict 1e-9 short protocol).
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _op(kb, name):
    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem(name)
    svd, _ = kb.egkb(kb.RearrangedBlur(prob.psf, prob.n), kb.EgkbConfig(**prob.egkb))
    return prob, kb.assemble(svd, kb.BlockScheme.square_image(prob.n))


@pytest.mark.parametrize("name", ["n256", "n512", "n1024"])
def test_split_is_the_same_operator(kb, name):
    prob, op = _op(kb, name)
    n = prob.n
    sp, resid = op.toeplitz_split()
    assert sp.k == op.k           # the dense start-vector term is at the rounding level: dropped
    assert sp.split_dense_share < 2e-7 and resid < 1e-6, (sp.split_dense_share, resid)
    kept, resid1 = op.toeplitz_split(dense_tol=0.0)   # ... or kept as a (k + 1)-th term
    assert kept.k == op.k + 1 and resid1 <= resid
    rng = np.random.default_rng(2)
    for _ in range(2):
        x = rng.standard_normal(n * n)
        for a, b in ((sp.apply(x), op.apply(x)), (sp.apply_t(x), op.apply_t(x))):
            assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)


@pytest.mark.parametrize("dense_tol", [2e-7, 0.0])
@pytest.mark.parametrize("name", ["n256", "n512"])
def test_split_apply_vs_oracle(kb, name, dense_tol):
    from oracle import sb as osb

    prob, op = _op(kb, name)
    n = prob.n
    sp, _ = op.toeplitz_split(dense_tol=dense_tol)
    ref = osb.KronOracle(sp.ax, sp.ay, n, n, n, n)
    rng = np.random.default_rng(4)
    x = rng.standard_normal(n * n)
    for got, want in ((sp.apply(x), ref.apply(x)), (sp.apply_t(x), ref.apply_t(x))):
        assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("dense_tol", [2e-7, 0.0])
@pytest.mark.parametrize("variant", ["isotropic", "anisotropic"])
def test_split_sb_short_protocol(kb, variant, dense_tol):
    from oracle import sb as osb
    from paper_2410_00233_b200 import datagen

    prob, op = _op(kb, "n256")
    n = prob.n
    sp, _ = op.toeplitz_split(dense_tol=dense_tol)
    cfg = kb.SbConfig(lam=datagen.LAM, beta=datagen.BETA, variant=variant, tau=0.0, l_max=3,
                      cgls=kb.CglsConfig(i_max=10, tau=0.0))
    res = kb.sb_run(sp, prob.b, cfg)
    oop = osb.KronOracle(sp.ax, sp.ay, n, n, n, n)
    ores = osb.sb_run(oop, prob.b, datagen.LAM, datagen.BETA, variant=variant, tau=0.0, l_max=3, i_max=10,
                      tau_cgls=0.0)
    gap = np.linalg.norm(res.x - ores.x) / np.linalg.norm(ores.x)
    assert gap < 1e-9, gap
    # and the solve on the split operator stays close to the solve on the original one
    res0 = kb.sb_run(op, prob.b, cfg)
    assert np.linalg.norm(res.x - res0.x) <= 1e-4 * np.linalg.norm(res0.x)


def test_split_refuses_unstructured_factors(kb):
    """Reflexive BC adds Hankel families to the factors: not Toeplitz + one direction."""
    from paper_2410_00233_b200 import datagen

    n = 64
    psf = datagen.rotated_gaussian_psf(n)[16:49, 16:49]
    svd, _ = kb.egkb(kb.RearrangedBlur(psf, n, bc="reflexive"), kb.EgkbConfig(k_max=6, k_min=6, p=2, tau=1e300))
    op = kb.assemble(svd, kb.BlockScheme.square_image(n))
    with pytest.raises(kb.ValidationError):
        op.toeplitz_split()
    rng = np.random.default_rng(0)
    dense = kb.KroneckerSum([rng.standard_normal((n, n)) for _ in range(3)],
                            [rng.standard_normal((n, n)) for _ in range(3)], kb.BlockScheme.square_image(n))
    with pytest.raises(kb.ValidationError):
        dense.toeplitz_split()


def test_estimator_flag(kb):
    """KroneckerApproximator(toeplitz_split=True) fits the split operator (PSF input, n = 128)."""
    from paper_2410_00233_b200 import datagen

    n = 128
    psf = datagen.mixture_psf(n)
    est = kb.KroneckerApproximator(engine="egkb", k_max=12, precision="single", toeplitz_split=True)
    est.fit(kb.Psf(psf), side=n)
    ref = kb.KroneckerApproximator(engine="egkb", k_max=12, precision="single").fit(kb.Psf(psf), side=n)
    assert est.operator_.k == ref.operator_.k and est.operator_.split_residual < 1e-6
    x = np.random.default_rng(1).standard_normal(n * n)
    a, b = est.operator_.apply(x), ref.operator_.apply(x)
    assert np.linalg.norm(a - b) <= 1e-5 * np.linalg.norm(b)


@pytest.mark.parametrize("dense_tol", [2e-7, 0.0])
def test_term_sharded_split_world1(kb, dense_tol):
    """ShardedKroneckerSum over a Toeplitz-split operator carries the F band / dense-term
    count to kb_kron (world 1: this rank owns every term, no collective)."""
    from paper_2410_00233_b200.parallel import ShardedKroneckerSum

    prob, op = _op(kb, "n256")
    sp, _ = op.toeplitz_split(dense_tol=dense_tol)
    sh = ShardedKroneckerSum(sp)
    kr = sh.forward_struct().kron
    assert bool(kr.fband) and kr.ndense == (1 if dense_tol == 0.0 else 0)
    x = np.random.default_rng(8).standard_normal(prob.n * prob.n)
    assert np.array_equal(sh.apply(x), sp.apply(x))
    assert np.array_equal(sh.apply_t(x), sp.apply_t(x))


def test_batched_solve_on_split_operator(kb):
    """kb_sb_run_batch on a Toeplitz-split operator (its stacked GEMMs treat every F_i as
    dense -- zeros included): each problem equals sb_run of its own config."""
    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem("n64", n=64)
    svd, _ = kb.egkb(kb.RearrangedBlur(prob.psf, 64), kb.EgkbConfig(**prob.egkb))
    op = kb.assemble(svd, kb.BlockScheme.square_image(64), toeplitz_split=True)
    cfgs = [kb.SbConfig.from_gamma(float(l), 2.0, variant="isotropic", tau=0.0, l_max=4,
                                   cgls=kb.CglsConfig(i_max=15, tau=0.0)) for l in (0.05, 0.2, 0.4)]
    batch = kb.sb_run_batch(op, prob.b, cfgs)
    for c, rb in zip(cfgs, batch):
        rs = kb.sb_run(op, prob.b, c)
        assert np.linalg.norm(rb.x - rs.x) <= 1e-8 * np.linalg.norm(rs.x)
