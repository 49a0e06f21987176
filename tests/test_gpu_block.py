"""Zero-BC block products of R(A) (the RSVD products, lowrank.py:363-367; kb_ra_block.cu
k_rat_diag -> k_rat_w -> k_rat_z[_mma] -> k_rat_bcast, chained by programmatic dependent
launch) against the CPU oracle, every vector count of the three z kernels.  Back-to-back
products on DIFFERENT inputs, so a kernel that read its predecessor's output before the
dependency wait would see the previous product's data and fail here."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / np.linalg.norm(b))


@pytest.mark.parametrize("dtype,tol", [(np.float32, 2e-7), (np.float64, 1e-13)])
@pytest.mark.parametrize("n", [256, 512])
def test_back_to_back_block_products(kb, n, dtype, tol):
    from oracle import structured as ost
    from paper_2410_00233_b200 import datagen
    from paper_2410_00233_b200 import device as D
    from paper_2410_00233_b200.lowrank import _EngineOp

    psf = datagen.mixture_psf(n, seed=n + 1)
    blur = kb.RearrangedBlur(psf, n, dtype=dtype)
    kern = blur.psf.kernel.astype(dtype)
    op = _EngineOp(blur)
    rng = np.random.default_rng(11)
    for nv in (1, 2, 3, 4, 5, 7, 8, 9, 16):
        xs = [rng.standard_normal((nv, n * n)).astype(dtype) for _ in range(3)]
        xds = [D.to_device(x) for x in xs]
        outs = [(op.apply_block(xd, 0), op.apply_block(xd, 1)) for xd in xds]   # back to back, no sync
        for x, (yd, zd) in zip(xs, outs):
            y, z = D.to_host(yd), D.to_host(zd)
            for j in (0, nv - 1):
                assert _rel(y[j], ost.ra_matvec(kern, n, x[j]).astype(np.float64)) < tol, (nv, j)
                assert _rel(z[j], ost.ra_rmatvec(kern, n, x[j]).astype(np.float64)) < tol, (nv, j)


def test_rsvd_repeatable(kb):
    """RSVD in fp32 at configs[2]'s size: the same seed gives the same result (or the same
    RankDeficiencyError column) on every call."""
    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem("n512")
    blur = kb.RearrangedBlur(prob.psf, prob.n)
    seen = set()
    for _ in range(8):
        try:
            svd = kb.rsvd(blur, kb.RsvdConfig(k=4, p=2, q=2, seed=0))
            seen.add(("ok", np.asarray(svd.sigma).tobytes()))
        except kb.RankDeficiencyError as e:
            seen.add(("rank", e.column))
    assert len(seen) == 1, seen


@pytest.mark.parametrize("dtype,tol", [(np.float32, 3e-7), (np.float64, 1e-13)])
@pytest.mark.parametrize("n,shape", [(128, (129, 129)), (128, (255, 255)), (256, (511, 511)), (256, (33, 129)),
                                     (256, (1, 7)), (256, (257, 31)), (384, (385, 385)), (384, (767, 5))])
def test_dense_random_psf_shapes(kb, n, shape, dtype, tol):
    """Dense random PSFs (every entry significant, unlike the Gaussians): the tile skipping
    outside the support, the band edges, the partial last r chunk of the z kernels, the
    cluster sizes 1..8 and non-square supports, for every z kernel (1, 3, 6, 16 vectors)."""
    from oracle import structured as ost
    from paper_2410_00233_b200 import device as D
    from paper_2410_00233_b200.lowrank import _EngineOp

    rng = np.random.default_rng(n + shape[0] + 7 * shape[1])
    psf = rng.random(shape) + 0.1
    blur = kb.RearrangedBlur(psf, n, dtype=dtype)
    kern = blur.psf.kernel.astype(dtype)
    op = _EngineOp(blur)
    for nv in (1, 3, 6, 16):
        x = rng.standard_normal((nv, n * n)).astype(dtype)
        xd = D.to_device(x)
        y, z = D.to_host(op.apply_block(xd, 0)), D.to_host(op.apply_block(xd, 1))
        for j in sorted({0, nv - 1}):
            assert _rel(y[j], ost.ra_matvec(kern, n, x[j]).astype(np.float64)) < tol, (nv, j)
            assert _rel(z[j], ost.ra_rmatvec(kern, n, x[j]).astype(np.float64)) < tol, (nv, j)


def test_block_product_n2048(kb):
    """configs[4]'s side: the tiled chain (row chunks over a full cluster, 2049 diagonals)."""
    from oracle import structured as ost
    from paper_2410_00233_b200 import device as D
    from paper_2410_00233_b200.lowrank import _EngineOp

    n = 2048
    rng = np.random.default_rng(5)
    psf = rng.random((n + 1, n + 1)) + 0.1
    blur = kb.RearrangedBlur(psf, n)
    kern = blur.psf.kernel.astype(np.float32)
    op = _EngineOp(blur)
    for nv in (1, 16):
        x = rng.standard_normal((nv, n * n)).astype(np.float32)
        xd = D.to_device(x)
        y, z = D.to_host(op.apply_block(xd, 0)), D.to_host(op.apply_block(xd, 1))
        j = nv - 1
        assert _rel(y[j], ost.ra_matvec(kern, n, x[j]).astype(np.float64)) < 3e-7, nv
        assert _rel(z[j], ost.ra_rmatvec(kern, n, x[j]).astype(np.float64)) < 3e-7, nv
