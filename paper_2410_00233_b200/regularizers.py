"""Halved first differences and the augmented system (reference: regularizers.py).

D_x x = vec(X L^T), D_y x = vec(L X) with L the (n-1) x n stencil [1, -1]/2
(regularizers.py:26-62).  The GPU forms these inside the fused CGLS passes;
the functions here expose the same kernels for direct calls.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import ValidationError
from .metrics import FlopCounter
from .operators import DenseOperator, as_operator


def first_difference_matrix(n: int) -> np.ndarray:
    if n < 2:
        raise ValidationError("first differences need n >= 2")
    l_mat = np.zeros((n - 1, n))
    idx = np.arange(n - 1)
    l_mat[idx, idx] = 0.5
    l_mat[idx, idx + 1] = -0.5
    return l_mat


def _diff(x, n: int, axis: int, transpose: int):
    from . import device as D

    if n < 2:
        raise ValidationError("first differences need n >= 2")
    want = n * n if not transpose else n * (n - 1)
    host = not D.is_tensor(x)
    xd = D.to_device(np.asarray(x, dtype=np.float64).ravel() if host else x, np.float64).reshape(-1)
    if xd.numel() != want:
        raise ValidationError(f"{'w' if transpose else 'x'} must have length {want}, got {xd.numel()}")
    out = D.empty(n * n if transpose else n * (n - 1), np.float64)
    _lib.check(_lib.load().kb_diff(xd.data_ptr(), out.data_ptr(), n, axis, transpose, 1.0, 0, D.stream_ptr()),
               "diff")
    return D.to_host(out) if host else out


def diff_x(x, n: int):
    """vec(0.5 (X[:, :-1] - X[:, 1:]))  (regularizers.py:37-39)."""
    return _diff(x, n, 0, 0)


def diff_y(x, n: int):
    """vec(0.5 (X[:-1, :] - X[1:, :]))  (regularizers.py:42-44)."""
    return _diff(x, n, 1, 0)


def diff_x_t(w, n: int):
    return _diff(w, n, 0, 1)


def diff_y_t(w, n: int):
    return _diff(w, n, 1, 1)


class AugmentedOp:
    """[A; lam_x D_x; lam_y D_y] (regularizers.py:65-117), applied on the GPU."""

    def __init__(self, forward, n: int, lam_x: float, lam_y: float):
        self.forward = as_operator(forward)
        if not hasattr(self.forward, "forward_struct"):
            raise ValidationError(
                f"{type(self.forward).__name__} has no device form; pass a dense matrix or a KroneckerSum")
        m, ncols = self.forward.shape
        if ncols != n * n:
            raise ValidationError(f"operator with {ncols} columns cannot act on {n}x{n} images")
        if n < 2:
            raise ValidationError("augmented system needs image side n >= 2")
        self.n = int(n)
        self.lam_x = float(lam_x)
        self.lam_y = float(lam_y)
        self.m = int(m)
        self.p_rows = n * (n - 1)
        self._dense = isinstance(self.forward, DenseOperator)

    @property
    def shape(self) -> tuple[int, int]:
        return (self.m + 2 * self.p_rows, self.n * self.n)

    def forward_struct(self):
        fw = self.forward.forward_struct()
        fw.augmented = 1
        fw.side = self.n
        fw.lam_x, fw.lam_y = self.lam_x, self.lam_y
        return fw

    def _count(self, counter, transpose):
        if counter is None:
            return
        if self._dense:
            counter.add_dense(self.shape[0], self.shape[1])
        elif hasattr(self.forward, "scheme"):
            s = self.forward.scheme
            (counter.add_kp_transpose if transpose else counter.add_kp)(s.m1, s.m2, s.n1, s.n2, self.forward.k)

    def apply(self, x, counter: FlopCounter | None = None):
        from .kronop import _forward_apply

        out = _forward_apply(self.forward_struct(), x, 0, self.shape)
        self._count(counter, 0)
        return out

    def apply_t(self, y, counter: FlopCounter | None = None):
        from .kronop import _forward_apply

        out = _forward_apply(self.forward_struct(), y, 1, self.shape)
        self._count(counter, 1)
        return out


def aug_rhs(b, dx, dy, gx, gy, lam_x: float, lam_y: float) -> np.ndarray:
    """[b; lam_x (dx - gx); lam_y (dy - gy)]  (regularizers.py:120-130)."""
    return np.concatenate([np.asarray(b), lam_x * (np.asarray(dx) - gx), lam_y * (np.asarray(dy) - gy)])
