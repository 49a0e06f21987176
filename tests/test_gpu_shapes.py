"""Image sides off the tiled kernels' envelope (n not a multiple of 128, n not dividing
128): the persistent / graph engines and the cooperative R(A) product against the
oracle, zero and reflexive BC (SURVEY §8c sigma bar; decisions above the noise floor)."""

from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


@pytest.mark.parametrize("n,bc", [(96, "zero"), (160, "zero"), (200, "zero"), (384, "zero"), (96, "reflexive"),
                                  (130, "reflexive")])
def test_odd_sides_vs_oracle(kb, n, bc):
    from oracle import lowrank as olr
    from oracle import structured as ost
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(n, seed=n)
    blur = kb.RearrangedBlur(psf, n, bc=bc)
    cfg = kb.EgkbConfig(k_max=12)
    svd, tr = kb.egkb(blur, cfg)
    k32 = blur.psf.kernel.astype(np.float32)
    ocfg = SimpleNamespace(k_max=12, p=2, tau=1e-4, k_min=2, reorth=None, seed=0, break_tol=None,
                           keep_basis=False)
    (_, os_, _), otr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q, bc), lambda s: ost.ra_rmatvec(k32, n, s, bc),
                                (n * n, n * n), np.float32, ocfg)
    assert tr.stop_reason == otr.stop_reason
    if not otr.breakdown:
        assert (tr.chosen_k, tr.k_p) == (otr.chosen_k, otr.k_p)
    m = min(svd.k, os_.size)
    ref = os_[:m].astype(np.float64)
    assert np.all(np.abs(svd.sigma[:m] - ref) <= 1e-4 * ref + 5e-6 * ref[0]), (svd.sigma, ref)
    # the standalone product on a random vector, both directions
    x = np.random.default_rng(n).standard_normal(n * n).astype(np.float32)
    for fwd, mv in ((True, ost.ra_matvec), (False, ost.ra_rmatvec)):
        got = np.asarray(blur.matvec(x) if fwd else blur.rmatvec(x), dtype=np.float64)
        want = mv(k32, n, x, bc).astype(np.float64)
        assert np.linalg.norm(got - want) <= 1e-6 * np.linalg.norm(want)
