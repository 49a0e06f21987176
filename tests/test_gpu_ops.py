"""GPU parity of the operator / tall-skinny / GEMM kernels against the oracle."""

import numpy as np
import pytest

from conftest import load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def kb():
    import paper_2410_00233_b200 as kb

    return kb


def _rel(a, b):
    return float(np.linalg.norm(np.asarray(a, dtype=np.float64) - b) / max(np.linalg.norm(b), 1e-300))


class TestRearrangedBlur:
    def test_matches_reference_dense_rearrangement(self, kb):
        g = load_golden("ra_structured")
        for i in range(5):
            k, n = g[f"c{i}_psf"], int(g[f"c{i}_n"])
            op = kb.RearrangedBlur(k, n, dtype=np.float64)
            np.testing.assert_allclose(op.matvec(g[f"c{i}_q"]), g[f"c{i}_Rq"], rtol=0, atol=1e-14)
            np.testing.assert_allclose(op.rmatvec(g[f"c{i}_s"]), g[f"c{i}_RTs"], rtol=0, atol=1e-14)

    def test_padded_even_psf_fp32(self, kb):
        g = load_golden("ra_structured")
        k, n = g["pad_psf"], int(g["pad_n"])
        op = kb.RearrangedBlur(k, n)
        got = op.matvec(g["pad_q"].astype(np.float32))
        assert got.dtype == np.float32
        assert _rel(got, g["pad_Rq"]) < 1e-6
        assert _rel(op.rmatvec(g["pad_s"].astype(np.float32)), g["pad_RTs"]) < 1e-6

    @pytest.mark.parametrize("n", [64, 256, 1024])
    def test_large_sides_against_oracle(self, kb, n):
        from oracle import structured as ost
        from paper_2410_00233_b200 import datagen

        psf = datagen.mixture_psf(n)
        rng = np.random.default_rng(n)
        q = rng.standard_normal(n * n).astype(np.float32)
        k32 = psf.astype(np.float32)
        op = kb.RearrangedBlur(psf, n)
        assert _rel(op.matvec(q), ost.ra_matvec(k32, n, q)) < 2e-7
        assert _rel(op.rmatvec(q), ost.ra_rmatvec(k32, n, q)) < 2e-7
        op64 = kb.RearrangedBlur(psf, n, dtype=np.float64)
        q64 = q.astype(np.float64)
        assert _rel(op64.matvec(q64), ost.ra_matvec(psf, n, q64)) < 1e-13

    def test_adjoint_identity(self, kb):
        n = 96
        rng = np.random.default_rng(3)
        psf = rng.random((9, 13))
        op = kb.RearrangedBlur(psf, n, dtype=np.float64)
        x, y = rng.standard_normal(n * n), rng.standard_normal(n * n)
        assert op.matvec(x) @ y == pytest.approx(x @ op.rmatvec(y), rel=1e-12)

    def test_validation(self, kb):
        with pytest.raises(kb.ValidationError):
            kb.RearrangedBlur(np.ones((4, 3)), 8)
        with pytest.raises(kb.ValidationError):   # single reflection only (blurmodel.py:100-101)
            kb.RearrangedBlur(np.ones((17, 3)), 8, bc="reflexive")
        with pytest.raises(kb.ValidationError):
            kb.RearrangedBlur(np.ones((3, 3)), 8, bc="periodic")
        op = kb.RearrangedBlur(np.ones((3, 3)), 8)
        with pytest.raises(kb.ValidationError):
            op.matvec(np.ones(10, dtype=np.float32))


class TestDgemm:
    @pytest.mark.parametrize("ta,tb", [(0, 0), (0, 1), (1, 0), (1, 1)])
    @pytest.mark.parametrize("m,n,k", [(1, 1, 1), (7, 5, 3), (130, 70, 33), (256, 128, 64)])
    def test_against_numpy(self, kb, ta, tb, m, n, k):
        import ctypes as C

        import torch
        from paper_2410_00233_b200 import _lib, device as D

        rng = np.random.default_rng(m * 1000 + n * 10 + k + ta * 7 + tb * 3)
        nb, ns = 3, 2
        A = rng.standard_normal((nb, ns, k, m) if ta else (nb, ns, m, k))
        B = rng.standard_normal((nb, ns, n, k) if tb else (nb, ns, k, n))
        want = np.zeros((nb, m, n))
        for z in range(nb):
            for s in range(ns):
                a = A[z, s].T if ta else A[z, s]
                b = B[z, s].T if tb else B[z, s]
                want[z] += a @ b
        Ad, Bd = D.to_device(A), D.to_device(B)
        Cd = torch.zeros((nb, m, n), dtype=torch.float64, device="cuda")
        lda = m if ta else k
        ldb = k if tb else n
        _lib.check(_lib.load().kb_dgemm(ta, tb, m, n, k, Ad.data_ptr(), lda, ns * m * k, m * k,
                                        Bd.data_ptr(), ldb, ns * k * n, k * n, Cd.data_ptr(), n, m * n, nb, ns,
                                        0.0, D.stream_ptr()))
        np.testing.assert_allclose(D.to_host(Cd), want, rtol=1e-12, atol=1e-12)


class TestKronecker:
    @pytest.mark.parametrize("dims,k", [((3, 4, 2, 5), 3), ((2, 2, 2, 2), 1), ((5, 2, 3, 3), 4),
                                        ((64, 64, 64, 64), 10), ((33, 17, 9, 40), 5)])
    def test_apply_against_oracle(self, kb, dims, k):
        from oracle import sb as osb

        rng = np.random.default_rng(sum(dims) + k)
        m1, m2, n1, n2 = dims
        ax = [rng.standard_normal((m1, n1)) for _ in range(k)]
        ay = [rng.standard_normal((m2, n2)) for _ in range(k)]
        op = kb.KroneckerSum(ax, ay, kb.BlockScheme(*dims))
        ref = osb.KronOracle(ax, ay, *dims)
        x = rng.standard_normal(n1 * n2)
        y = rng.standard_normal(m1 * m2)
        assert _rel(op.apply(x), ref.apply(x)) < 1e-13
        assert _rel(op.apply_t(y), ref.apply_t(y)) < 1e-13
        if m1 * m2 * n1 * n2 <= 2 ** 20:
            np.testing.assert_allclose(op.apply(x), ref.materialize() @ x, atol=1e-11)

    @staticmethod
    def _apply_dense(op, v, transpose):
        """kb_kron_apply with the band cleared: every k tile of the G stage."""
        import ctypes as C

        import torch

        from paper_2410_00233_b200 import _lib
        from paper_2410_00233_b200 import device as D

        lib = _lib.load()
        kr = op.kron_struct()
        kr.band = None
        nb = C.c_size_t()
        _lib.check(lib.kb_kron_workspace_bytes(C.byref(kr), C.byref(nb)))
        ws = torch.empty(max(1, nb.value), dtype=torch.uint8, device=D.device())
        xd = D.to_device(np.ascontiguousarray(v, dtype=np.float64))
        m, n = op.shape
        y = torch.empty(n if transpose else m, dtype=torch.float64, device=D.device())
        _lib.check(lib.kb_kron_apply(C.byref(kr), xd.data_ptr(), y.data_ptr(), transpose, ws.data_ptr(),
                                     nb.value, D.stream_ptr()))
        return D.to_host(y)

    @pytest.mark.parametrize("dims,k,lo,hi", [((96, 200, 80, 160), 3, -7, 40), ((64, 256, 64, 256), 4, -59, 59),
                                              ((40, 130, 40, 300), 2, 100, 180), ((32, 64, 32, 64), 2, 0, 0)])
    def test_banded_g_skips_zero_tiles_bit_identically(self, kb, dims, k, lo, hi):
        m1, m2, n1, n2 = dims
        rng = np.random.default_rng(m2 + n2 + k)
        ax = [rng.standard_normal((m1, n1)) for _ in range(k)]
        a_idx, b_idx = np.meshgrid(np.arange(m2), np.arange(n2), indexing="ij")
        mask = ((a_idx - b_idx) >= lo) & ((a_idx - b_idx) <= hi)   # G[r][c] = ay[c][r], d = c - r
        ay = [np.where(mask, rng.standard_normal((m2, n2)), 0.0) for _ in range(k)]
        op = kb.KroneckerSum(ax, ay, kb.BlockScheme(*dims))
        x = rng.standard_normal(n1 * n2)
        y = rng.standard_normal(m1 * m2)
        got, got_t = op.apply(x), op.apply_t(y)
        band = op._band.cpu().numpy()
        nz = np.nonzero(np.any(np.stack(ay) != 0, axis=0))
        assert (band[0], band[1]) == ((nz[0] - nz[1]).min(), (nz[0] - nz[1]).max())
        np.testing.assert_array_equal(got, self._apply_dense(op, x, 0))
        np.testing.assert_array_equal(got_t, self._apply_dense(op, y, 1))

    def test_all_zero_g_gives_zero(self, kb):
        s = kb.BlockScheme(64, 64, 64, 64)
        rng = np.random.default_rng(3)
        op = kb.KroneckerSum([rng.standard_normal((64, 64))], [np.zeros((64, 64))], s)
        out = op.apply(rng.standard_normal(64 * 64))
        assert op._band.cpu().numpy()[0] > op._band.cpu().numpy()[1]
        np.testing.assert_array_equal(out, np.zeros(64 * 64))

    def test_egkb_factors_are_banded_and_skip_bit_identically(self, kb):
        """Zero BC: the v-side factors are banded Toeplitz (products of R(A)^T),
        so the apply skips most G tiles and still equals the dense apply."""
        from paper_2410_00233_b200 import datagen

        prob = datagen.make_problem("n256")
        n = prob.n
        svd, _ = kb.egkb(kb.RearrangedBlur(prob.psf.astype(np.float32), n), kb.EgkbConfig(k_max=20, k_min=20, p=2))
        op = kb.assemble(svd, kb.BlockScheme.square_image(n))
        rng = np.random.default_rng(1)
        x = rng.standard_normal(n * n)
        got, got_t = op.apply(x), op.apply_t(x)
        lo, hi = op._band.cpu().numpy()
        assert hi - lo < n // 2, (lo, hi)
        np.testing.assert_array_equal(got, self._apply_dense(op, x, 0))
        np.testing.assert_array_equal(got_t, self._apply_dense(op, x, 1))

    def test_materialize_and_factors_roundtrip(self, kb):
        rng = np.random.default_rng(0)
        s = kb.BlockScheme(3, 4, 2, 5)
        ax = [rng.standard_normal((3, 2)) for _ in range(2)]
        ay = [rng.standard_normal((4, 5)) for _ in range(2)]
        op = kb.KroneckerSum(ax, ay, s)
        dev = kb.KroneckerSum.from_device(op.f_dev, op.g_dev, s)
        for a, b in zip(dev.ax, ax):
            np.testing.assert_array_equal(a, b)
        np.testing.assert_allclose(dev.materialize(), sum(np.kron(a, b) for a, b in zip(ax, ay)))

    def test_assemble_matches_reference_rule(self, kb):
        g = load_golden("config_n64")
        n = 64
        svd = kb.TruncatedSvd(g["u"], g["sigma"], g["v"])
        op = kb.assemble(svd, kb.BlockScheme.square_image(n))
        for i in range(svd.k):
            want_ax = g["sigma"][i].astype(np.float64) * g["u"][:, i].astype(np.float64).reshape((n, n), order="F")
            np.testing.assert_array_equal(op.ax[i], want_ax)


class TestStencilsAndShrink:
    def test_diff_ops_against_oracle(self, kb):
        from oracle import sb as osb

        n = 37
        rng = np.random.default_rng(1)
        x = rng.standard_normal(n * n)
        w = rng.standard_normal(n * (n - 1))
        np.testing.assert_array_equal(kb.diff_x(x, n), osb.dx(x, n))
        np.testing.assert_array_equal(kb.diff_y(x, n), osb.dy(x, n))
        np.testing.assert_array_equal(kb.diff_x_t(w, n), osb.dx_t(w, n))
        np.testing.assert_array_equal(kb.diff_y_t(w, n), osb.dy_t(w, n))

    def test_shrink_updates(self, kb):
        from oracle import sb as osb

        rng = np.random.default_rng(2)
        cx, cy = rng.standard_normal(1000), rng.standard_normal(1000)
        cx[:5] = 0.0
        cy[:3] = 0.0
        for g in (0.5, 1.5, 19.0):
            dx, dy = kb.update_d_aniso(cx, cy, g, g)
            ex, ey = osb.d_aniso(cx, cy, g, g)
            np.testing.assert_array_equal(dx, ex)
            np.testing.assert_array_equal(dy, ey)
            dx, dy = kb.update_d_iso(cx, cy, g, g)
            ex, ey = osb.d_iso(cx, cy, g, g)
            np.testing.assert_allclose(dx, ex, rtol=1e-12, atol=1e-15)
            np.testing.assert_allclose(dy, ey, rtol=1e-12, atol=1e-15)
        dx, dy = kb.update_d_iso(np.array([3.0]), np.array([4.0]), 1.0, 1.0)
        assert dx[0] == pytest.approx(2.4) and dy[0] == pytest.approx(3.2)
        dx, dy = kb.update_d_iso(np.array([0.3]), np.array([0.4]), 1.0, 1.0)
        assert dx[0] == 0.0 and dy[0] == 0.0


class TestOrthonormalize:
    def test_against_reference_golden(self, kb):
        g = load_golden("rsvd_kat")
        q = kb.orthonormalize(g["orth_in"])
        assert np.abs(q - g["orth_out"]).max() < 1e-13
        q32 = kb.orthonormalize(g["orth_in"].astype(np.float32))
        assert q32.dtype == np.float32
        assert np.abs(q32 - g["orth32_out"]).max() < 1e-5

    def test_rank_deficiency_names_column(self, kb):
        rng = np.random.default_rng(0)
        m = rng.standard_normal((40, 6))
        m[:, 4] = m[:, 1] + 2 * m[:, 2]
        with pytest.raises(kb.RankDeficiencyError) as err:
            kb.orthonormalize(m)
        assert err.value.column == 4

    def test_too_many_columns(self, kb):
        with pytest.raises(kb.ValidationError):
            kb.orthonormalize(np.ones((3, 5)))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("side", [31, 513])
@pytest.mark.parametrize("order", ["C", "F"])
def test_device_psf_is_numpys_normalisation_bitwise(kb, dtype, side, order):
    """blurmodel.py:25-65: the device K is (k / k.sum()).astype(dtype) bit for bit, whichever
    upload path runs (host fp32 commit, staged raw fp64 + device cast, the small-PSF path,
    C- or Fortran-ordered input)."""
    from paper_2410_00233_b200 import device as D

    rng = np.random.default_rng(side)
    k = np.asarray(rng.random((side, side)) ** 3, order=order)
    blur = kb.RearrangedBlur(k, 1024 if side == 513 else 64, dtype=dtype)
    kd, kt = blur._device_kernels()
    want = (k / k.sum()).astype(dtype)
    assert np.array_equal(D.to_host(kd), want)
    assert np.array_equal(D.to_host(kt), want.T)
    # the staged copy is consumed once; a second operator from the same Psf uploads again
    blur2 = kb.RearrangedBlur(blur.psf, blur.n, dtype=dtype)
    assert np.array_equal(D.to_host(blur2._device_kernels()[0]), want)
    # a Psf built on its own
    blur3 = kb.RearrangedBlur(kb.Psf(k), blur.n, dtype=dtype)
    assert np.array_equal(D.to_host(blur3._device_kernels()[0]), want)
    # the caller's array may change after construction (the kernel is copied, blurmodel.py:33)
    k2 = np.array(k, order=order)
    blur4 = kb.RearrangedBlur(k2, blur.n, dtype=dtype)
    k2[:] = -1.0
    assert np.array_equal(D.to_host(blur4._device_kernels()[0]), want)
    assert np.array_equal(blur4.psf.kernel, k / k.sum())
