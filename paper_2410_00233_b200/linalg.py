"""Precision control, vectorisation, truncated SVD container, small SVD and
the GPU orthonormalisation (reference: pkg/src/kronblur/linalg.py).

``TruncatedSvd`` keeps the reference's host-array surface (``u``, ``sigma``,
``v`` are numpy arrays, linalg.py:94-131) but may be *device-backed*: factors
produced on the GPU stay there (``u_device``/``v_device``, one singular vector
per row) and are copied to the host only when ``.u``/``.v`` are read.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import NumericalError, RankDeficiencyError, ValidationError

PRECISIONS = {"single": np.float32, "double": np.float64}
SVD_SMALL_LIMIT = 4096   # linalg.py:26


def dtype_for(precision: str) -> np.dtype:
    try:
        return np.dtype(PRECISIONS[precision])
    except KeyError:
        raise ValidationError(
            f"unknown precision {precision!r}; expected one of {sorted(PRECISIONS)}") from None


def precision_of(arr) -> str:
    """Precision name of a numpy array or torch tensor; rejects other dtypes."""
    dt = getattr(arr, "dtype", None)
    if dt is not None and not isinstance(dt, np.dtype):  # torch dtype
        dt = {"torch.float32": np.dtype(np.float32), "torch.float64": np.dtype(np.float64)}.get(str(dt))
    for name, want in PRECISIONS.items():
        if dt == want:
            return name
    raise ValidationError(f"unsupported dtype {getattr(arr, 'dtype', None)}; expected float32 or float64")


def eps_for(dtype_like) -> float:
    if isinstance(dtype_like, str):
        dtype_like = dtype_for(dtype_like)
    return float(np.finfo(dtype_like).eps)


def cast(arr, precision: str) -> np.ndarray:
    """Copy into the given precision (IEEE narrowing, linalg.py:54-63)."""
    dt = dtype_for(precision)
    with np.errstate(over="ignore"):
        return np.asarray(arr).astype(dt)


def fro_norm(mat) -> float:
    """Permutation-invariant Frobenius norm (sorted squares, linalg.py:66-73)."""
    sq = np.sort(np.square(np.asarray(mat, dtype=np.float64).ravel()))
    return float(np.sqrt(np.sum(sq)))


def vec(mat) -> np.ndarray:
    mat = np.asarray(mat)
    if mat.ndim != 2:
        raise ValidationError(f"vec expects a matrix, got ndim={mat.ndim}")
    return mat.reshape(-1, order="F")


def unvec(v, rows: int, cols: int) -> np.ndarray:
    v = np.asarray(v)
    if v.ndim != 1:
        raise ValidationError(f"unvec expects a vector, got ndim={v.ndim}")
    if v.size != rows * cols:
        raise ValidationError(f"cannot reshape length-{v.size} vector to {rows}x{cols}")
    return v.reshape((rows, cols), order="F")


class TruncatedSvd:
    """Rank-k factorisation ``u @ diag(sigma) @ v.T`` (linalg.py:94-131).

    Construct from host arrays (``TruncatedSvd(u, sigma, v)``) or, on the GPU
    path, from device tensors holding one singular vector per row
    (``TruncatedSvd.from_device(u_rows, sigma, v_rows)``).
    """

    def __init__(self, u, sigma, v):
        self._u = None if u is None else np.asarray(u)
        self._v = None if v is None else np.asarray(v)
        self.sigma = np.asarray(sigma)
        self._u_dev = None
        self._v_dev = None
        self._lazy = None
        if self._u is not None:
            self._validate(self._u.shape, self._v.shape)

    @classmethod
    def from_device(cls, u_rows, sigma, v_rows):
        obj = cls(None, sigma, None)
        obj._u_dev, obj._v_dev = u_rows, v_rows
        obj._validate((u_rows.shape[1], u_rows.shape[0]), (v_rows.shape[1], v_rows.shape[0]))
        return obj

    @classmethod
    def from_lift(cls, lazy, sigma):
        """Singular vectors kept as (Krylov basis, lift weights) on the device until
        first used; ``assemble`` then writes the fp64 Kronecker factors straight
        from the basis (kb_lift_assemble) without materialising u / v."""
        obj = cls(None, sigma, None)
        obj._lazy = lazy
        m, n = lazy.shape
        obj._validate((m, obj.sigma.size), (n, obj.sigma.size))
        return obj

    def _force(self):
        if self._lazy is not None:
            self._u_dev, self._v_dev = self._lazy.materialize()
            self._lazy = None

    def _validate(self, ushape, vshape):
        if len(ushape) != 2 or len(vshape) != 2 or self.sigma.ndim != 1:
            raise ValidationError("TruncatedSvd expects u, v matrices and a sigma vector")
        k = self.sigma.size
        if ushape[1] != k or vshape[1] != k:
            raise ValidationError(
                f"inconsistent rank: u has {ushape[1]} columns, v has {vshape[1]}, sigma has {k} entries")
        if k and np.any(np.diff(self.sigma) > 0):
            raise ValidationError("sigma must be non-increasing")
        if k and self.sigma[-1] < 0:
            raise ValidationError("sigma must be non-negative")

    @property
    def u(self) -> np.ndarray:
        self._force()
        if self._u is None:
            self._u = self._u_dev.detach().cpu().numpy().T
        return self._u

    @property
    def v(self) -> np.ndarray:
        self._force()
        if self._v is None:
            self._v = self._v_dev.detach().cpu().numpy().T
        return self._v

    @property
    def u_device(self):
        """u as a (k, m) CUDA tensor (uploads host factors on first use)."""
        self._force()
        if self._u_dev is None:
            from . import device as D
            self._u_dev = D.to_device(np.ascontiguousarray(self._u.T))
        return self._u_dev

    @property
    def v_device(self):
        self._force()
        if self._v_dev is None:
            from . import device as D
            self._v_dev = D.to_device(np.ascontiguousarray(self._v.T))
        return self._v_dev

    @property
    def k(self) -> int:
        return self.sigma.size

    @property
    def shape(self):
        if self._lazy is not None:
            return tuple(self._lazy.shape)
        m = self._u.shape[0] if self._u is not None else self._u_dev.shape[1]
        n = self._v.shape[0] if self._v is not None else self._v_dev.shape[1]
        return (m, n)

    def reconstruct(self) -> np.ndarray:
        return (self.u * self.sigma) @ self.v.T

    def truncate(self, k: int) -> "TruncatedSvd":
        if not 0 < k <= self.k:
            raise ValidationError(f"cannot truncate rank-{self.k} factorization to k={k}")
        self._force()
        if self._u is None:
            return TruncatedSvd.from_device(self._u_dev[:k], self.sigma[:k], self._v_dev[:k])
        return TruncatedSvd(self._u[:, :k], self.sigma[:k], self._v[:, :k])

    def __repr__(self):
        where = "device (lazy lift)" if self._lazy is not None else ("device" if self._u is None else "host")
        return f"TruncatedSvd(k={self.k}, shape={self.shape}, {where})"


def svd_small(mat) -> TruncatedSvd:
    """Full SVD of a small dense matrix on the host (LAPACK, linalg.py:134-153).

    The north star keeps the small bidiagonal / projected SVDs on the host;
    this is the reference's own call, used for C (eGKB) and H (RSVD).
    """
    mat = np.asarray(mat)
    if mat.ndim != 2:
        raise ValidationError(f"svd_small expects a matrix, got ndim={mat.ndim}")
    if min(mat.shape) > SVD_SMALL_LIMIT:
        raise ValidationError(
            f"matrix of shape {mat.shape} exceeds the small-problem bound {SVD_SMALL_LIMIT}")
    precision_of(mat)
    try:
        u, s, vt = np.linalg.svd(mat, full_matrices=False)
    except np.linalg.LinAlgError as exc:
        raise NumericalError(f"SVD failed to converge on shape {mat.shape}") from exc
    return TruncatedSvd(u, s, vt.T)


def orthonormalize_device(cols, drop_tol: float | None = None):
    """In-place CGS2 orthonormalisation of the rows of a (ncol, m) CUDA tensor
    with the reference drop test (linalg.py:156-199).  Raises
    RankDeficiencyError(j) / NumericalError like the reference."""
    from . import device as D

    ncol, m = cols.shape
    if ncol > m:
        raise ValidationError(f"cannot orthonormalize {ncol} columns in dimension {m}")
    dt = _lib.KB_F32 if str(cols.dtype) == "torch.float32" else _lib.KB_F64
    lib = _lib.load()
    nbytes = C.c_size_t()
    _lib.check(lib.kb_orth_workspace_bytes(m, ncol, C.byref(nbytes)))
    ws, wsb = D.WORKSPACE.get(nbytes.value)
    bad = C.c_int(-1)
    st = lib.kb_orthonormalize(dt, cols.data_ptr(), m, ncol, m, -1.0 if drop_tol is None else float(drop_tol),
                               C.byref(bad), ws, wsb, D.stream_ptr())
    if st == _lib.KB_ENUMERICAL:
        if bad.value >= 0:
            raise RankDeficiencyError(bad.value)
        if bad.value <= -2:
            raise NumericalError(f"non-finite column norm at column {-2 - bad.value}")
    _lib.check(st, "orthonormalize")
    return cols


def orthonormalize(mat, drop_tol: float | None = None) -> np.ndarray:
    """Orthonormalise the columns of ``mat`` on the GPU (linalg.py:156-199).

    Two classical Gram-Schmidt passes per column (CGS2) replace the
    reference's two MGS passes; the drop test and its default tolerance
    ``eps * sqrt(m) * max column norm`` are the reference's.
    """
    from . import device as D

    arr = np.asarray(mat)
    if arr.ndim != 2:
        raise ValidationError(f"orthonormalize expects a matrix, got ndim={arr.ndim}")
    m, n = arr.shape
    if n > m:
        raise ValidationError(f"cannot orthonormalize {n} columns in dimension {m}")
    precision_of(arr)
    if n == 0:
        return arr.copy()
    cols = D.to_device(np.ascontiguousarray(arr.T))
    orthonormalize_device(cols, drop_tol)
    return D.to_host(cols).T.copy()
