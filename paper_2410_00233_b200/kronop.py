"""Sum-of-Kronecker-products operator with device-resident fp64 factors.

Reference: pkg/src/kronblur/kronop.py.  ``apply`` computes
``vec(sum_i ay_i X ax_i^T)`` and ``apply_t`` ``vec(sum_i ay_i^T Y ax_i)``
(kronop.py:58-84) as two DMMA GEMMs each (kb_kron_apply): a batched stage
``P_i = X_r G_i`` and a segment-reduced stage ``Y_r = sum_i F_i^T P_i`` with
inner dimension k*n1, where F_i = ax_i^T and G_i = ay_i^T are stored as the
column-major vectors the SVD produced (so ``assemble`` is a pure cast/scale).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import ValidationError
from .metrics import FlopCounter
from .rearrange import BlockScheme

MATERIALIZE_CAP = 2 ** 24


def _forward_apply(fw, x, transpose: int, shape):
    from . import device as D

    host = not D.is_tensor(x)
    want = shape[0] if transpose else shape[1]
    if host:
        arr = np.asarray(x, dtype=np.float64)
        if arr.ndim == 2 and 1 in arr.shape:
            arr = arr.ravel()
        if arr.shape != (want,):
            raise ValidationError(
                f"{'apply_t' if transpose else 'apply'} expects a vector of length {want}, got {arr.shape}")
        xd = D.to_device(arr)
    else:
        xd = D.to_device(x, np.float64).reshape(-1)
        if xd.numel() != want:
            raise ValidationError(f"expected a vector of length {want}, got {xd.numel()}")
    rows_out = shape[1] if transpose else shape[0]
    y = D.empty(rows_out, np.float64)
    lib = _lib.load()
    nb = C.c_size_t()
    _lib.check(lib.kb_forward_workspace_bytes(C.byref(fw), C.byref(nb)))
    ws, wsb = D.WORKSPACE.get(nb.value)
    sharded = bool(fw.allreduce)
    if sharded:   # the allreduce hook maps the raw output pointer back to this tensor
        from .parallel import REGISTRY
        REGISTRY.add(y)
    try:
        _lib.check(lib.kb_forward_apply(C.byref(fw), xd.data_ptr(), y.data_ptr(), transpose, ws, wsb,
                                        D.stream_ptr()), "operator apply")
    finally:
        if sharded:
            REGISTRY.remove(y)
    return D.to_host(y) if host else y


class KroneckerSum:
    """k-term Kronecker-product sum with double-precision factors (kronop.py:28-100)."""

    def __init__(self, ax, ay, scheme: BlockScheme):
        from . import device as D

        if len(ax) != len(ay):
            raise ValidationError("ax and ay must hold the same number of terms")
        if len(ax) == 0:
            raise ValidationError("KroneckerSum needs at least one term")
        s = scheme
        ax = [np.ascontiguousarray(a, dtype=np.float64) for a in ax]
        ay = [np.ascontiguousarray(b, dtype=np.float64) for b in ay]
        for i, (a, b) in enumerate(zip(ax, ay)):
            if a.shape != (s.m1, s.n1):
                raise ValidationError(f"ax[{i}] has shape {a.shape}, expected {(s.m1, s.n1)}")
            if b.shape != (s.m2, s.n2):
                raise ValidationError(f"ay[{i}] has shape {b.shape}, expected {(s.m2, s.n2)}")
        self.scheme = s
        self._ax, self._ay = ax, ay
        f = np.stack([a.T.reshape(-1) for a in ax])   # F_i = ax_i^T  (n1 x m1 row-major)
        g = np.stack([b.T.reshape(-1) for b in ay])   # G_i = ay_i^T  (n2 x m2 row-major)
        self.f_dev = D.to_device(f)
        self.g_dev = D.to_device(g)
        self._band = None
        self._ft = None
        self._ndense, self._fband = None, None

    @classmethod
    def from_device(cls, f_dev, g_dev, scheme: BlockScheme) -> "KroneckerSum":
        obj = cls.__new__(cls)
        obj.scheme = scheme
        obj._ax = obj._ay = None
        obj.f_dev, obj.g_dev = f_dev, g_dev
        obj._band = None
        obj._ft = None
        obj._ndense, obj._fband = None, None
        return obj

    @property
    def ax(self) -> list:
        """Host factors A_x,i (m1 x n1, C order: kronop.py:42-43), transposed on the device
        and read back in one copy."""
        if self._ax is None:
            s = self.scheme
            f = self.f_dev.detach().view(-1, s.n1, s.m1).transpose(1, 2).contiguous().cpu().numpy()
            self._ax = [f[i] for i in range(f.shape[0])]
        return self._ax

    @property
    def ay(self) -> list:
        if self._ay is None:
            s = self.scheme
            g = self.g_dev.detach().view(-1, s.n2, s.m2).transpose(1, 2).contiguous().cpu().numpy()
            self._ay = [g[i] for i in range(g.shape[0])]
        return self._ay

    @property
    def k(self) -> int:
        return int(self.f_dev.shape[0])

    @property
    def shape(self) -> tuple[int, int]:
        return self.scheme.shape

    def kron_struct(self) -> _lib.KbKron:
        s = self.scheme
        kr = _lib.KbKron(s.m1, s.m2, s.n1, s.n2, self.k, self.f_dev.data_ptr(), self.g_dev.data_ptr())
        if self._band is None:
            # zero band of the G factors, found once on first use (stream-ordered,
            # no host sync): the G stage of every apply then skips all-zero tiles
            import torch

            from . import device as D

            band = torch.empty(2, dtype=torch.int32, device=self.g_dev.device)
            _lib.check(_lib.load().kb_kron_band(C.byref(kr), band.data_ptr(), D.stream_ptr()), "kron band")
            self._band = band
        kr.band = self._band.data_ptr()
        if self._ft is None:
            # F_i^T blocks (device transpose, once per operator): the reduced stage of the
            # transposed apply becomes one dense GEMM as well (structured: the dense terms only)
            s = self.scheme
            nd = self.k if self._ndense is None else self._ndense
            self._ft = self.f_dev[:max(nd, 1)].view(-1, s.n1, s.m1).transpose(1, 2).contiguous()
        if self._ndense is None or self._ndense > 0:   # (no dense F term: no cuBLAS stage, CGLS stays a graph)
            kr.ft = self._ft.data_ptr()
        if self._ndense is not None:
            if self._fband is None:   # zero band of the banded F blocks (same kernel as G's)
                import torch

                from . import device as D

                nd = self._ndense
                # kb_kron_band scans the "g" blocks (n2 x m2): here the stored n1 x m1 F blocks
                tmp = _lib.KbKron(s.m1, s.m1, s.n1, s.n1, self.k - nd, None, self.f_dev[nd:].data_ptr())
                fband = torch.empty(2, dtype=torch.int32, device=self.f_dev.device)
                _lib.check(_lib.load().kb_kron_band(C.byref(tmp), fband.data_ptr(), D.stream_ptr()), "kron band")
                self._fband = fband
            kr.ndense = self._ndense
            kr.fband = self._fband.data_ptr()
        return kr

    def toeplitz_split(self, drop: float = 3e-8, dense_tol: float = 2e-7, max_dropped: float = 1e-5):
        """The same operator with the structure of a zero-BC eGKB approximation made explicit.

        Every s-basis vector of the eGKB on R(A) is a combination of R(A) q products
        (constant along the diagonals of the n x n image: Toeplitz) and of the dense start
        vector, whose non-Toeplitz part is orthogonal to the range of R(A): the lifted
        F_i = T_i + a_i D + E_i with T_i Toeplitz (the diagonal means of F_i), D one dense
        matrix (the dominant direction of the non-Toeplitz parts) and both a_i D and E_i at
        the fp32 rounding level.  Returns (operator, dropped):

        * |a| <= ``dense_tol`` |F_1| (the case for every BASELINE config, 4e-8): the k-term
          operator sum_i T_i (x) G_i, every factor banded Toeplitz;
        * otherwise the (k + 1)-term operator D (x) (sum_i a_i G_i) + sum_i T_i (x) G_i.

        T_i diagonals below ``drop`` x max |T| and G entries below ``drop`` x max |G| are set
        to zero, so both GEMM stages of every product skip the all-zero k tiles
        (kb_kron.fband / band).  ``dropped`` is the relative Frobenius size of what the F
        side lost, max_i |F_i - F_i'| / |F_1|; above ``max_dropped`` (an operator without this
        structure: reflexive BC, sparse A, RSVD factors) a ValidationError is raised.  The
        split is an approximation of this operator (not of the reference's arithmetic):
        callers opt in.
        """
        import torch

        s = self.scheme
        if not (s.m1 == s.n1 == s.m2 == s.n2):
            raise ValidationError("toeplitz_split needs square factors of one size")
        n, k = s.n1, self.k
        f = self.f_dev.view(k, n, n)
        g = self.g_dev.view(k, n * n)
        # diagonal means: index d = col - row + n - 1 of the stored n1 x m1 blocks
        r = torch.arange(n, device=f.device)
        didx = (r[None, :] - r[:, None] + (n - 1)).reshape(-1)
        cnt = torch.zeros(2 * n - 1, dtype=torch.float64, device=f.device).index_add_(
            0, didx, torch.ones(n * n, dtype=torch.float64, device=f.device))
        fm = f.reshape(k, n * n)
        means = torch.zeros(k, 2 * n - 1, dtype=torch.float64, device=f.device).index_add_(1, didx, fm) / cnt
        non = fm - means[:, didx]                       # non-Toeplitz parts, rank one up to rounding
        gram = (non @ non.T).cpu().numpy()              # k x k: host eigh, no cuSOLVER start-up
        _, vecs = np.linalg.eigh(gram)
        d = torch.as_tensor(vecs[:, -1].copy(), device=f.device) @ non
        d = d / torch.linalg.norm(d)
        a = non @ d                                     # F_i ~ T_i + a_i D
        f1 = torch.linalg.norm(fm[0])
        dense_share = float(torch.linalg.norm(a) / f1)
        scale = means.abs().max()
        means = torch.where(means.abs() >= drop * scale, means, torch.zeros_like(means))
        t = means[:, didx]
        # the G side keeps its exact zeros; entries below drop x max |G| (the Gaussian tails
        # between the fp32 underflow and the rounding level) are dropped as well
        gt = torch.where(g.abs() >= drop * g.abs().max(), g, torch.zeros_like(g))
        if dense_share <= dense_tol:
            resid = torch.linalg.norm(fm - t, dim=1).max() / f1
            out = KroneckerSum.from_device(t.contiguous(), gt.contiguous(), s)
            out._ndense = 0
        else:
            resid = torch.linalg.norm(fm - t - a[:, None] * d[None, :], dim=1).max() / f1
            f2 = torch.cat([d[None, :], t], dim=0).contiguous()
            g2 = torch.cat([(a[:, None] * gt).sum(dim=0, keepdim=True), gt], dim=0).contiguous()
            out = KroneckerSum.from_device(f2, g2, s)
            out._ndense = 1
        if not float(resid) <= max_dropped:
            raise ValidationError(
                f"toeplitz_split would drop {float(resid):.2e} of the leading factor (limit {max_dropped:.1e}): "
                "the factors are not Toeplitz plus one dense direction")
        out.split_dense_share = dense_share             # |a| / |F_1|
        return out, float(resid)

    def forward_struct(self) -> _lib.KbForward:
        fw = _lib.KbForward()
        fw.kind = _lib.KB_FWD_KRON
        fw.m, fw.n = self.shape
        fw.a, fw.lda = None, 0
        fw.kron = self.kron_struct()
        return fw

    def apply(self, x, counter: FlopCounter | None = None):
        """A @ x for a vectorised image (kronop.py:58-70)."""
        out = _forward_apply(self.forward_struct(), x, 0, self.shape)
        if counter is not None:
            s = self.scheme
            counter.add_kp(s.m1, s.m2, s.n1, s.n2, self.k)
        return out

    def apply_t(self, y, counter: FlopCounter | None = None):
        """A.T @ y (kronop.py:72-84)."""
        out = _forward_apply(self.forward_struct(), y, 1, self.shape)
        if counter is not None:
            s = self.scheme
            counter.add_kp_transpose(s.m1, s.m2, s.n1, s.n2, self.k)
        return out

    def materialize(self, cap: int = MATERIALIZE_CAP) -> np.ndarray:
        """Dense sum_i kron(ax_i, ay_i) on the host (tests only, kronop.py:86-100)."""
        m, n = self.shape
        if m * n > cap:
            raise ValidationError(f"materializing a {m}x{n} matrix ({m * n} entries) exceeds the cap {cap}")
        out = np.zeros((m, n))
        for a, b in zip(self.ax, self.ay):
            out += np.kron(a, b)
        return out


def assemble(svd, scheme: BlockScheme, toeplitz_split: bool = False) -> KroneckerSum:
    """Truncated SVD of R(A) -> KroneckerSum (kronop.py:103-123).

    ax_i = sigma_i unvec(u_i, m1, n1), ay_i = unvec(v_i, m2, n2), promoted to
    fp64.  On the device this is one cast/scale kernel (kb_kron_assemble):
    F_i = ax_i^T is exactly sigma_i * u_i as stored.  ``toeplitz_split=True`` (an
    extension; zero-BC eGKB results) returns ``KroneckerSum.toeplitz_split()`` of that
    operator instead, with the dropped share in ``.split_residual``.
    """
    if toeplitz_split:
        op, resid = assemble(svd, scheme).toeplitz_split()
        op.split_residual = resid
        return op
    from . import device as D

    m_u, m_v = svd.shape
    if m_u != scheme.m1 * scheme.n1 or m_v != scheme.m2 * scheme.n2:
        raise ValidationError(
            f"SVD dimensions {m_u}x{m_v} do not match the rearranged shape {scheme.rearranged_shape}")
    k = svd.k
    f = D.empty((k, m_u), np.float64)
    g = D.empty((k, m_v), np.float64)
    sig = np.ascontiguousarray(svd.sigma.astype(np.float64))
    lazy = getattr(svd, "_lazy", None)
    if lazy is not None:            # eGKB result: factors straight from the Krylov bases
        lazy.assemble(sig, f, g)
        return KroneckerSum.from_device(f, g, scheme)
    u, v = svd.u_device, svd.v_device
    code = _lib.KB_F32 if str(u.dtype) == "torch.float32" else _lib.KB_F64
    _lib.check(_lib.load().kb_kron_assemble(code, u.data_ptr(), m_u, v.data_ptr(), m_v,
                                            sig.ctypes.data_as(C.POINTER(C.c_double)), k, m_u, m_v,
                                            f.data_ptr(), g.data_ptr(), D.stream_ptr()), "assemble")
    return KroneckerSum.from_device(f, g, scheme)
