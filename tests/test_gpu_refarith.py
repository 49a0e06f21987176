"""The reference-arithmetic eGKB engine (KB_ARITH_OPENBLAS_*) against the CPU oracle:
bit-identical sdot, traces, rank decisions and Krylov bases (lowrank.py:153-277).

The oracle runs the reference's algorithm with this host's numpy (its OpenBLAS
sdot kernel); the GPU engine is told to emulate the same kernel
(``host_blas_arithmetic()``).  The other x86-64 kernel is checked against the
oracle's numpy restatement of it (``oracle/blas.py``)."""

import ctypes as C
from types import SimpleNamespace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _sdot_gpu(lanes, x, y):
    import torch

    from paper_2410_00233_b200 import _lib
    from paper_2410_00233_b200 import device as D

    xd = D.to_device(x)
    yd = D.to_device(y) if y is not None else None
    out = D.empty((1,), np.float32)
    ws = D.empty((1024,), np.float32)
    _lib.check(_lib.load().kb_sdot_openblas(lanes, xd.data_ptr(), yd.data_ptr() if yd is not None else None,
                                             x.size, out.data_ptr(), ws.data_ptr(), 4096, D.stream_ptr()))
    torch.cuda.synchronize()
    return np.float32(out.cpu().numpy()[0])


@pytest.mark.parametrize("kernel,lanes", [("openblas-skx", 64), ("openblas-hsw", 32)])
def test_sdot_bitwise(kernel, lanes):
    from oracle import blas

    rng = np.random.default_rng(5)
    for n in [1, 31, 32, 33, 64, 96, 100, 1000, 4099, 65536, 65536 + 61, 1 << 20]:
        x = (rng.standard_normal(n) * 10.0 ** rng.uniform(-4, 4)).astype(np.float32)
        y = rng.standard_normal(n).astype(np.float32)
        assert _sdot_gpu(lanes, x, y) == blas.sdot(x, y, kernel), (kernel, n)
        assert _sdot_gpu(lanes, x, None) == blas.sdot(x, x, kernel), (kernel, n)


def _run_pair(kb, psf, n, egkb_kw, arithmetic, kernel=None, bc="zero"):
    from oracle import lowrank as olr
    from oracle import structured as ost

    cfg = kb.EgkbConfig(**egkb_kw, keep_basis=True)
    svd, tr = kb.egkb(kb.RearrangedBlur(psf, n, bc=bc), cfg, arithmetic=arithmetic)
    k32 = kb.RearrangedBlur(psf, n, bc=bc).psf.kernel.astype(np.float32)
    ocfg = SimpleNamespace(k_max=cfg.k_max, p=cfg.p, tau=cfg.tau, k_min=cfg.k_min, reorth=None, seed=0,
                           break_tol=None, keep_basis=True)
    (_, os_, _), otr = olr.egkb(lambda q: ost.ra_matvec(k32, n, q, bc), lambda s: ost.ra_rmatvec(k32, n, s, bc),
                                (n * n, n * n), np.float32, ocfg, kernel=kernel)
    return svd, tr, os_, otr


def _assert_identical(svd, tr, os_, otr):
    assert (tr.chosen_k, tr.k_p, tr.stop_reason, tr.breakdown) == (otr.chosen_k, otr.k_p, otr.stop_reason,
                                                                   otr.breakdown)
    # the whole trace, bit for bit (fp32 norms as Python floats, fp64 zeta / nu)
    assert tr.alphas == otr.alphas and tr.ts == otr.ts
    assert tr.zetas == otr.zetas and tr.nus == otr.nus
    # the Krylov bases: every stored vector bit-identical
    assert np.array_equal(tr.s_basis, otr.s_basis)
    assert np.array_equal(tr.q_basis, otr.q_basis)
    ref = os_.astype(np.float64)
    assert np.all(np.abs(svd.sigma - ref) <= 1e-6 * ref[0]), (svd.sigma, ref)


@pytest.mark.parametrize("name", ["n256", "n512", "n1024", "n2048"])
def test_config_runs_bit_identical(kb, name):
    """configs[1..4]: the automatic rank (n=256, n=2048 with cap 50) and the fixed-rank
    runs that end in a noise-floor breakdown (n=512: 20+2, n=1024: 30+2) take the
    reference's decisions, with the reference's trace and bases bit for bit."""
    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem(name)
    svd, tr, os_, otr = _run_pair(kb, prob.psf, prob.n, prob.egkb, "reference")
    _assert_identical(svd, tr, os_, otr)


@pytest.mark.parametrize("n,egkb_kw,bc", [
    (38, dict(k_max=8, k_min=8, p=2, tau=1e300), "zero"),      # n^2 = 1444: the 32-block and a tail of 4
    (37, dict(k_max=6), "zero"),                                # n^2 = 1369: tail of 25
    (40, dict(k_max=12, k_min=12, p=2, tau=1e300), "reflexive"),
])
def test_edge_lengths_bit_identical(kb, n, egkb_kw, bc):
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(n, seed=7)
    svd, tr, os_, otr = _run_pair(kb, psf, n, egkb_kw, "reference", bc=bc)
    _assert_identical(svd, tr, os_, otr)


@pytest.mark.parametrize("kernel", ["openblas-skx", "openblas-hsw"])
@pytest.mark.parametrize("n,seed", [(128, 101), (256, 104)])
def test_either_kernel_bit_identical(kb, kernel, n, seed):
    """Both x86-64 sdot kernels, whichever this host runs: against the oracle's
    restatement of that kernel (oracle/blas.py, pinned to numpy by test_oracle_blas)."""
    from paper_2410_00233_b200 import datagen

    psf = datagen.mixture_psf(n, seed=seed)
    svd, tr, os_, otr = _run_pair(kb, psf, n, dict(k_max=20, k_min=20, p=2, tau=1e300), kernel, kernel=kernel)
    _assert_identical(svd, tr, os_, otr)


def test_estimator_reference_arithmetic(kb):
    """KroneckerApproximator(arithmetic="reference") (estimators.py:95-139 + the extension):
    the fitted trace is the reference's, bit for bit."""
    from paper_2410_00233_b200 import datagen

    prob = datagen.make_problem("n256")
    est = kb.KroneckerApproximator(engine="egkb", k_max=20, precision="single", arithmetic="reference")
    est.fit(kb.Psf(prob.psf), side=prob.n)
    _, tr, _, otr = _run_pair(kb, prob.psf, prob.n, dict(k_max=20), "reference")
    assert (est.trace_.alphas, est.trace_.ts) == (otr.alphas, otr.ts)
    assert est.k_ == otr.chosen_k
