"""Operator protocol (reference: operators.py:11-46).

Anything with ``apply``/``apply_t``/``shape`` is an operator; ndarrays are
wrapped in :class:`DenseOperator`, whose products run on the GPU (fp64).
"""

from __future__ import annotations

import numpy as np

from .exceptions import ValidationError


class DenseOperator:
    """A dense fp64 matrix held on the device."""

    def __init__(self, mat):
        from . import device as D

        if D.is_tensor(mat):
            if mat.ndim != 2:
                raise ValidationError("DenseOperator expects a matrix")
            self.dev = D.to_device(mat, np.float64)
        else:
            arr = np.asarray(mat, dtype=np.float64)
            if arr.ndim != 2:
                raise ValidationError("DenseOperator expects a matrix")
            self.dev = D.to_device(arr)
        self._shape = tuple(self.dev.shape)

    @property
    def shape(self):
        return self._shape

    @property
    def mat(self) -> np.ndarray:
        from . import device as D

        return D.to_host(self.dev)

    def forward_struct(self):
        from . import _lib

        fw = _lib.KbForward()
        fw.kind = _lib.KB_FWD_DENSE
        fw.m, fw.n = self._shape
        fw.a, fw.lda = self.dev.data_ptr(), self._shape[1]
        return fw

    def apply(self, x, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), x, 0, self._shape)

    def apply_t(self, y, counter=None):
        from .kronop import _forward_apply

        return _forward_apply(self.forward_struct(), y, 1, self._shape)


def as_operator(op):
    """Pass through anything with apply/apply_t/shape; wrap arrays."""
    from . import device as D

    if isinstance(op, np.ndarray) or D.is_tensor(op):
        return DenseOperator(op)
    for attr in ("apply", "apply_t", "shape"):
        if not hasattr(op, attr):
            raise ValidationError(f"object {type(op).__name__} lacks {attr}; not a linear operator")
    return op


def is_dense(op) -> bool:
    return isinstance(op, (DenseOperator, np.ndarray))
