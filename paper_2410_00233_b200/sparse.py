"""R(A) of an unstructured sparse A (rearrange.py:67-75).

The paper's premise is an arbitrary blur matrix A (not only a PSF
convolution).  ``rearrange`` only permutes entries:

    R[j*m1 + i, q*m2 + p] = A[i*m2 + p, j*n2 + q]          (rearrange.py:72-75)

so for a sparse A, R(A) is sparse with the same values.  ``RearrangedSparse``
applies that permutation to the nonzeros ONCE on the host, keeps CSR copies
of R and R^T on the device, and hands the engines (eGKB / RSVD) an operator of
kind ``KB_OP_SPARSE``: each product is a warp-per-row CSR kernel
(``k_csr_rows``, fixed-order reduction), HBM-bound at ~12 B per nonzero.
The values are cast to the working precision like ``cast(rearrange(A))``
(``linalg.py:54-63``).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .exceptions import ValidationError
from .rearrange import BlockScheme


def _coo(a):
    """(rows, cols, vals, shape) from a scipy sparse matrix, a COO triple or a dense array."""
    if isinstance(a, tuple) and len(a) == 4:
        r, c, v, shape = a
        return np.asarray(r, dtype=np.int64), np.asarray(c, dtype=np.int64), np.asarray(v), tuple(shape)
    if hasattr(a, "tocoo"):
        m = a.tocoo()
        return m.row.astype(np.int64), m.col.astype(np.int64), np.asarray(m.data), tuple(m.shape)
    d = np.asarray(a)
    if d.ndim != 2:
        raise ValidationError("A must be a 2-D matrix")
    r, c = np.nonzero(d)
    return r.astype(np.int64), c.astype(np.int64), d[r, c], d.shape


def _csr(rows, cols, vals, nrows):
    """CSR (row pointers int64, columns int32, values) of COO entries, duplicates summed."""
    order = np.lexsort((cols, rows))
    rows, cols, vals = rows[order], cols[order], vals[order]
    if rows.size:
        first = np.r_[True, (rows[1:] != rows[:-1]) | (cols[1:] != cols[:-1])]
        if not first.all():
            idx = np.cumsum(first) - 1
            vals = np.bincount(idx, weights=vals)
            rows, cols = rows[first], cols[first]
    rowptr = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(rows, minlength=nrows), out=rowptr[1:])
    return rowptr, cols.astype(np.int32), vals


class RearrangedSparse:
    """Matrix-free R(A) of a sparse A for the device engines (``egkb``, ``rsvd``)."""

    def __init__(self, a, scheme: BlockScheme, dtype=np.float32):
        r, c, v, shape = _coo(a)
        if shape != scheme.shape:
            raise ValidationError(f"matrix shape {shape} does not factor as "
                                  f"({scheme.m1}*{scheme.m2}, {scheme.n1}*{scheme.n2})")
        if r.size and (r.min() < 0 or c.min() < 0 or r.max() >= shape[0] or c.max() >= shape[1]):
            raise ValidationError("sparse entries out of range")
        self.dtype = np.dtype(dtype)
        if self.dtype not in (np.dtype(np.float32), np.dtype(np.float64)):
            raise ValidationError(f"unsupported dtype {self.dtype}; expected float32 or float64")
        v = np.asarray(v, dtype=np.float64)
        if not np.all(np.isfinite(v)):
            raise ValidationError("A has non-finite entries")
        m1, m2, n1, n2 = scheme.m1, scheme.m2, scheme.n1, scheme.n2
        i, p = np.divmod(r, m2)
        j, q = np.divmod(c, n2)
        rr, rc = j * m1 + i, q * m2 + p                  # rearrange.py:72-75
        self.scheme = scheme
        self.shape = scheme.rearranged_shape
        self._host = (rr, rc, v)
        self.nnz = None
        self._dev = None

    @property
    def ndim(self) -> int:
        return 2

    def _device(self):
        from . import device as D

        if self._dev is None:
            rr, rc, v = self._host
            rp, ci, va = _csr(rr, rc, v, self.shape[0])
            trp, tci, tva = _csr(rc, rr, v, self.shape[1])
            self.nnz = int(ci.size)
            self._dev = tuple(D.to_device(x) for x in (rp, ci)) + (D.to_device(va.astype(self.dtype)),) + \
                tuple(D.to_device(x) for x in (trp, tci)) + (D.to_device(tva.astype(self.dtype)),)
        return self._dev

    def op_struct(self) -> _lib.KbOperator:
        rp, ci, va, trp, tci, tva = self._device()
        op = _lib.KbOperator()
        op.kind = _lib.KB_OP_SPARSE
        op.dtype = _lib.KB_F32 if self.dtype == np.float32 else _lib.KB_F64
        op.rows, op.cols = self.shape
        op.sp_rowptr, op.sp_col, op.sp_val = rp.data_ptr(), ci.data_ptr(), va.data_ptr()
        op.spt_rowptr, op.spt_col, op.spt_val = trp.data_ptr(), tci.data_ptr(), tva.data_ptr()
        op.nnz = self.nnz
        return op

    @property
    def T(self) -> "RearrangedSparse":
        """R(A)^T as an operator (swaps the two CSR copies; no data movement)."""
        t = object.__new__(RearrangedSparse)
        t.dtype, t.scheme = self.dtype, self.scheme
        t.shape = (self.shape[1], self.shape[0])
        rr, rc, v = self._host
        t._host = (rc, rr, v)
        t._dev = None if self._dev is None else self._dev[3:] + self._dev[:3]
        t.nnz = self.nnz
        return t

    def astype(self, dtype) -> "RearrangedSparse":
        t = object.__new__(RearrangedSparse)
        t.dtype, t.scheme, t.shape, t._host, t.nnz, t._dev = np.dtype(dtype), self.scheme, self.shape, self._host, None, None
        return t

    def _apply(self, x, transpose: int):
        from . import device as D

        host = not D.is_tensor(x)
        n_in = self.shape[0] if transpose else self.shape[1]
        xd = D.to_device(x, self.dtype).reshape(-1)
        if xd.numel() != n_in:
            raise ValidationError(f"expected a vector of length {n_in}, got {xd.numel()}")
        y = D.empty(self.shape[1] if transpose else self.shape[0], self.dtype)
        op = self.op_struct()
        lib = _lib.load()
        nb = C.c_size_t()
        _lib.check(lib.kb_op_workspace_bytes(C.byref(op), C.byref(nb)))
        ws, wsb = D.WORKSPACE.get(nb.value)
        _lib.check(lib.kb_op_apply(C.byref(op), xd.data_ptr(), y.data_ptr(), transpose, ws, wsb, D.stream_ptr()),
                   "sparse R(A) apply")
        return D.to_host(y) if host else y

    def matvec(self, q):
        return self._apply(q, 0)

    def rmatvec(self, s):
        return self._apply(s, 1)

    def __matmul__(self, x):
        return self.matvec(x)

    def to_dense(self) -> np.ndarray:
        rr, rc, v = self._host
        out = np.zeros(self.shape)
        np.add.at(out, (rr, rc), v)
        return out
