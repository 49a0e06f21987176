"""PSF model, dense blur matrix (small n) and the matrix-free R(A) operator.

Reference: pkg/src/kronblur/blurmodel.py.  ``Psf``, ``NoiseSpec``,
``add_noise`` and ``build_blur_matrix`` keep the reference semantics (host
input construction).  :class:`RearrangedBlur` is the B200 extension named by
SURVEY §8(b): R(A) of a zero-BC blur applied matrix-free on the GPU, accepted
by :func:`egkb`, :func:`rsvd` and :func:`tsvd` wherever a dense ``b_mat`` is.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _lib
from .exceptions import NumericalError, ValidationError

BC_ZERO = "zero"
BC_REFLEXIVE = "reflexive"
BOUNDARY_CONDITIONS = (BC_ZERO, BC_REFLEXIVE)
DENSE_SIDE_CAP = 200   # blurmodel.py:22


_POOL = None


def _min(k: np.ndarray) -> float:
    """k.min() (order-independent, so large kernels are reduced by row blocks in parallel threads)."""
    if k.size < (1 << 18) or k.ndim != 2 or not k.flags.c_contiguous:
        return k.min()
    global _POOL
    if _POOL is None:
        from concurrent.futures import ThreadPoolExecutor

        _POOL = ThreadPoolExecutor(8)
    cuts = np.linspace(0, k.shape[0], 9).astype(int)
    parts = _POOL.map(lambda i: k[cuts[i]:cuts[i + 1]].min() if cuts[i + 1] > cuts[i] else np.inf, range(8))
    return min(parts)


_SCAN_MIN = 1 << 16
_HOST_THREADS = max(1, min(16, os.cpu_count() or 1))


# Recycled private-copy buffers (by shape): a fresh 8 MB array per Psf would pay its
# page faults on every construction; a Psf returns its copy here when it is dropped.
_RAW_POOL: dict = {}
_RAW_POOL_MAX = 2


def _raw_take(shape) -> np.ndarray:
    lst = _RAW_POOL.get(shape)
    return lst.pop() if lst else np.empty(shape, dtype=np.float64)


def _raw_give(arr: np.ndarray) -> None:
    lst = _RAW_POOL.setdefault(arr.shape, [])
    if len(lst) < _RAW_POOL_MAX:
        lst.append(arr)


def _scan(k: np.ndarray) -> tuple[float, np.float64, np.ndarray]:
    """min, numpy-exact sum and a private copy of ``k`` in one multithreaded pass."""
    lib = _lib.load()
    total, kmin = C.c_double(), C.c_double()
    own = _raw_take(k.shape)
    _lib.check(lib.kb_psf_scan(k.ctypes.data, k.size, _HOST_THREADS, C.byref(total), C.byref(kmin),
                               own.ctypes.data), "kb_psf_scan")
    return kmin.value, np.float64(total.value), own


class Psf:
    """Unit-sum, non-negative PSF with odd support (blurmodel.py:25-65).

    Like the reference, the kernel is copied at construction (later changes to
    the caller's array do not reach the operator); validation and the mass are
    computed eagerly, exactly as the reference (same checks, same pairwise sum
    over the C-ordered float64 array), in the same multithreaded pass as the
    copy.  The normalised float64 ``kernel`` is materialised on first access.
    """

    __slots__ = ("_raw", "_total", "_kernel", "_pooled")

    def __init__(self, kernel):
        k = np.asarray(kernel, dtype=np.float64)
        if k.ndim != 2:
            raise ValidationError("PSF kernel must be 2-D")
        if k.shape[0] % 2 == 0 or k.shape[1] % 2 == 0:
            raise ValidationError(f"PSF support must be odd in both dimensions, got {k.shape}")
        self._raw = None
        self._pooled = False
        if k.size >= _SCAN_MIN and k.flags.c_contiguous:
            # min, numpy's pairwise sum and the private copy in one multithreaded host pass
            # (kb_psf_scan: bit-identical to k.sum(), which is single-threaded)
            kmin, total, own = _scan(k)
            if not kmin >= 0 and np.any(own < 0):
                _raw_give(own)
                raise ValidationError("PSF kernel must be non-negative")
            k, self._pooled = own, True
        else:
            k = np.array(k)                           # the reference's private order-'K' copy
            if k.size == 0 or not _min(k) >= 0:      # one reduction; the exact test only when it fails
                if np.any(k < 0):
                    raise ValidationError("PSF kernel must be non-negative")
            total = k.sum()
        if total <= 0:
            if self._pooled:
                _raw_give(k)
            raise ValidationError("PSF kernel must have positive mass")
        self._raw, self._total, self._kernel = k, total, None

    def __del__(self):
        if getattr(self, "_pooled", False) and self._raw is not None:
            _raw_give(self._raw)

    @property
    def kernel(self) -> np.ndarray:
        if self._kernel is None:
            self._kernel = self._raw / self._total     # bitwise the reference's k / total
            if self._pooled:
                _raw_give(self._raw)
            self._raw = None
        return self._kernel

    def device_normalised(self, dtype):
        """The normalised kernel on the device in ``dtype``.  fp32: (k / total).astype(float32)
        on the host straight into pinned memory, 4 bytes per entry on the wire (bitwise
        numpy); fp64: the raw kernel uploaded and divided on the device (kb_div_cast)."""
        from . import device as D

        if self._kernel is not None:
            return D.upload(self._kernel, dtype)
        lib = _lib.load()
        src = self._raw if self._raw.flags.c_contiguous else np.ascontiguousarray(self._raw)
        if np.dtype(dtype) == np.float32:
            out = D.empty(self.shape, np.float32)
            _lib.check(lib.kb_psf_commit_f32(src.ctypes.data, src.size, float(self._total), out.data_ptr(),
                                             _HOST_THREADS, D.stream_ptr()), "PSF upload")
            return out
        raw = D.empty(self._raw.shape, np.float64)
        _lib.check(lib.kb_stage_upload(src.ctypes.data, src.nbytes, raw.data_ptr(), _HOST_THREADS,
                                       D.stream_ptr()), "kb_stage_upload")
        out = D.empty(self.shape, dtype)
        code = _lib.KB_F32 if np.dtype(dtype) == np.float32 else _lib.KB_F64
        _lib.check(lib.kb_div_cast(raw.data_ptr(), float(self._total), code, out.data_ptr(), raw.numel(),
                                   D.stream_ptr()), "kb_div_cast")
        return out

    def __repr__(self) -> str:
        return f"Psf(shape={self.shape})"

    @property
    def center(self) -> tuple[int, int]:
        return (self.shape[0] // 2, self.shape[1] // 2)

    @property
    def shape(self) -> tuple[int, int]:
        return (self._raw if self._kernel is None else self._kernel).shape

    def separability_ratio(self) -> float:
        s = np.linalg.svd(self.kernel, compute_uv=False)
        if s[0] == 0:
            raise NumericalError("PSF kernel has zero norm")
        return float(s[1] / s[0]) if s.size > 1 else 0.0


@dataclass(frozen=True)
class NoiseSpec:
    level: float
    seed: int = 0

    def __post_init__(self):
        if self.level < 0:
            raise ValidationError("noise level must be >= 0")


def add_noise(b_true, spec: NoiseSpec):
    """White noise with ||eta|| = level ||b_true|| (blurmodel.py:204-218)."""
    b_true = np.asarray(b_true, dtype=np.float64)
    if spec.level == 0.0:
        return b_true.copy(), np.zeros_like(b_true)
    zeta = np.random.default_rng(spec.seed).standard_normal(b_true.shape)
    znorm = np.linalg.norm(zeta.ravel())
    if znorm == 0.0:
        raise NumericalError("degenerate noise draw")
    eta = spec.level * (np.linalg.norm(b_true.ravel()) / znorm) * zeta
    return b_true + eta, eta


def _reflect(idx, n):
    out = np.where(idx < 0, -1 - idx, idx)
    return np.where(out >= n, 2 * n - 1 - out, out)


def build_blur_matrix(psf: Psf, n: int, bc: str = BC_ZERO, cap: int = DENSE_SIDE_CAP) -> np.ndarray:
    """Dense n^2 x n^2 convolution matrix (host; blurmodel.py:87-127).

    Only for small dense comparisons; the GPU path never forms A or R(A).
    """
    if bc not in BOUNDARY_CONDITIONS:
        raise ValidationError(f"boundary condition must be one of {BOUNDARY_CONDITIONS}, got {bc!r}")
    if n < 1:
        raise ValidationError("image side must be >= 1")
    if n > cap:
        raise ValidationError(f"image side {n} exceeds the dense cap {cap}")
    kh, kw = psf.shape
    if bc == BC_REFLEXIVE and (kh > 2 * n - 1 or kw > 2 * n - 1):
        raise ValidationError("PSF support too large for single reflection at this image size")
    cu, cv = psf.center
    rr, cc = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    out_idx = (cc * n + rr).ravel()
    a = np.zeros((n * n, n * n))
    for u in range(kh):
        for v in range(kw):
            wgt = psf.kernel[u, v]
            if wgt == 0.0:
                continue
            r_in, c_in = rr - u + cu, cc - v + cv
            if bc == BC_ZERO:
                ok = ((r_in >= 0) & (r_in < n) & (c_in >= 0) & (c_in < n)).ravel()
                a[out_idx[ok], (c_in * n + r_in).ravel()[ok]] += wgt
            else:
                a[out_idx, (_reflect(c_in, n) * n + _reflect(r_in, n)).ravel()] += wgt
    return a


def make_test_image(n: int) -> np.ndarray:
    """Deterministic piecewise-constant test image (blurmodel.py:186-201)."""
    if n < 8:
        raise ValidationError(f"test image side must be >= 8, got {n}")
    img = np.full((n, n), 0.05)
    img[n // 8 : n // 2, n // 8 : n // 2] = 0.9
    img[n // 2 :, 2 * n // 3 :] = 0.45
    rr, cc = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    img[(rr - 0.7 * n) ** 2 + (cc - 0.3 * n) ** 2 <= (0.16 * n) ** 2] = 0.7
    img[n // 12 : n // 6, :] = np.maximum(img[n // 12 : n // 6, :], 0.3)
    return img


class RearrangedBlur:
    """Matrix-free R(A) of a PSF blur on n x n images (zero or reflexive BC).

    R[c_in*n + c_out, r_in*n + r_out] = K[r_out - r_in + cu, c_out - c_in + cv]
    (closed form of rearrange.py:67-75 o blurmodel.py:106-121; SURVEY
    Appendix A).  For bc="reflexive" (blurmodel.py:80-84, 122-126) R =
    P_c K^T P_r^T where P also carries the two Hankel (reflected) index
    families; the same kernels run with the anti-diagonal terms enabled.  Shape (n^2, n^2); ``dtype`` is the working precision of the
    engines (float32 = the reference's "SP" path).  The PSF lives on the
    device; products run in the sm_100a kernels of libkronblur_b200.
    """

    def __init__(self, psf, n: int, bc: str = BC_ZERO, dtype=np.float32):
        if not isinstance(psf, Psf):
            psf = Psf(psf)
        if bc not in BOUNDARY_CONDITIONS:
            raise ValidationError(f"boundary condition must be one of {BOUNDARY_CONDITIONS}, got {bc!r}")
        if n < 1:
            raise ValidationError("image side must be >= 1")
        kh, kw = psf.shape
        if bc == BC_REFLEXIVE and (kh > 2 * n - 1 or kw > 2 * n - 1):   # blurmodel.py:100-101
            raise ValidationError("PSF support too large for single reflection at this image size")
        self.psf = psf
        self.n = int(n)
        self.bc = bc
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise ValidationError(f"unsupported dtype {self.dtype}; expected float32 or float64")
        self._k = None
        self._kt = None

    @property
    def shape(self) -> tuple[int, int]:
        return (self.n * self.n, self.n * self.n)

    @property
    def ndim(self) -> int:
        return 2

    def astype(self, dtype) -> "RearrangedBlur":
        return RearrangedBlur(self.psf, self.n, self.bc, dtype)

    def _device_kernels(self):
        from . import device as D

        if self._k is None:
            # one upload of the raw PSF; normalisation, cast and K^T on the device
            self._k = self.psf.device_normalised(self.dtype)
            kh, kw = self.psf.shape
            self._kt = D.empty((kw, kh), self.dtype)
            code = _lib.KB_F32 if self.dtype == np.float32 else _lib.KB_F64
            _lib.check(_lib.load().kb_transpose(code, self._k.data_ptr(), kh, kw, self._kt.data_ptr(),
                                                D.stream_ptr()), "kb_transpose")
        return self._k, self._kt

    def op_struct(self) -> _lib.KbOperator:
        k, kt = self._device_kernels()
        kh, kw = self.psf.shape
        op = _lib.KbOperator()
        op.kind = _lib.KB_OP_RA_ZERO if self.bc == BC_ZERO else _lib.KB_OP_RA_REFLEXIVE
        op.dtype = _lib.KB_F32 if self.dtype == np.float32 else _lib.KB_F64
        op.rows = op.cols = self.n * self.n
        op.a, op.lda = None, 0
        op.k, op.kt = k.data_ptr(), kt.data_ptr()
        op.kh, op.kw, op.side = kh, kw, self.n
        return op

    def _apply(self, x, transpose: int):
        from . import device as D

        host = not D.is_tensor(x)
        xd = D.to_device(x, self.dtype).reshape(-1)
        if xd.numel() != self.n * self.n:
            raise ValidationError(f"expected a vector of length {self.n * self.n}, got {xd.numel()}")
        y = D.empty(self.n * self.n, self.dtype)
        op = self.op_struct()
        lib = _lib.load()
        nb = C.c_size_t()
        _lib.check(lib.kb_op_workspace_bytes(C.byref(op), C.byref(nb)))
        ws, wsb = D.WORKSPACE.get(nb.value)
        _lib.check(lib.kb_op_apply(C.byref(op), xd.data_ptr(), y.data_ptr(), transpose, ws, wsb,
                                   D.stream_ptr()), "R(A) apply")
        return D.to_host(y) if host else y

    def matvec(self, q):
        """R(A) q  (replaces ``b_mat @ q``, lowrank.py:238)."""
        return self._apply(q, 0)

    def rmatvec(self, s):
        """R(A)^T s  (replaces ``b_mat.T @ s``, lowrank.py:211,250)."""
        return self._apply(s, 1)

    def __matmul__(self, x):
        return self.matvec(x)

    def to_dense(self) -> np.ndarray:
        """Dense R(A) (host, tiny n only; for tests)."""
        if self.n > 64:
            raise ValidationError("to_dense is for n <= 64")
        from .rearrange import BlockScheme, rearrange

        return rearrange(build_blur_matrix(self.psf, self.n), BlockScheme.square_image(self.n)).astype(self.dtype)
