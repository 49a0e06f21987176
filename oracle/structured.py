"""Matrix-free R(A) for a zero-boundary PSF blur (CPU oracle, test infra only).

Index conventions (reference ``pkg/src/kronblur/``):

* ``blurmodel.py:106-121``: A[c_out*n + r_out, c_in*n + r_in] += K[u, v] with
  r_in = r_out - u + cu, c_in = c_out - v + cv (zero BC drops out-of-range).
* ``rearrange.py:67-75`` with the square scheme ``rearrange.py:54-57``:
  R[j*n + i, q*n + p] = A[i*n + p, j*n + q].

Together:  R[c_in*n + c_out, r_in*n + r_out] =
K[r_out - r_in + cu, c_out - c_in + cv]  (zero when the K index is out of
range), i.e. R = W_c K^T W_r^T with 0/1 diagonal-indicator matrices W.

``ra_matvec``/``ra_rmatvec`` evaluate R q and R^T s in O(n^2 + kh*kw) work by
diagonal sums -> small K product -> Toeplitz broadcast.  ``ra_dense`` builds the
dense R for tiny n (used to pin the closed form against the reference).
``structured_tsvd`` is the exact SVD of R through D_c K^T D_r.
"""

from __future__ import annotations

import numpy as np

_OFFS_CACHE: dict[int, np.ndarray] = {}


def _offsets(n: int) -> np.ndarray:
    """offs[a*n + b] = b - a for an n-by-n row-major grid (cached per n)."""
    o = _OFFS_CACHE.get(n)
    if o is None:
        ar = np.arange(n, dtype=np.int64)
        o = (ar[None, :] - ar[:, None]).ravel()
        _OFFS_CACHE.clear()
        _OFFS_CACHE[n] = o
    return o


def _diag_sums(vec: np.ndarray, n: int, center: int, length: int) -> np.ndarray:
    """w[u] = sum_{a,b: b - a + center = u} vec[a*n + b], u in [0, length)."""
    idx = _offsets(n) + center
    keep = (idx >= 0) & (idx < length)
    return np.bincount(idx[keep], weights=vec[keep].astype(np.float64), minlength=length)


def _broadcast(z: np.ndarray, n: int, center: int, dtype) -> np.ndarray:
    """out[a*n + b] = z[b - a + center] (zero outside [0, len(z)))."""
    idx = _offsets(n) + center
    keep = (idx >= 0) & (idx < z.size)
    out = np.zeros(n * n, dtype=dtype)
    out[keep] = z[idx[keep]]
    return out


def ra_matvec(kernel: np.ndarray, n: int, q: np.ndarray) -> np.ndarray:
    """y = R(A) q.  q is indexed r_in*n + r_out, y is indexed c_in*n + c_out."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    w = _diag_sums(q, n, cu, kh)                       # over r_out - r_in
    z = np.asarray(kernel, dtype=np.float64).T @ w     # z[v] = sum_u K[u,v] w[u]
    return _broadcast(z, n, cv, q.dtype)


def ra_rmatvec(kernel: np.ndarray, n: int, s: np.ndarray) -> np.ndarray:
    """x = R(A)^T s.  s is indexed c_in*n + c_out, x is indexed r_in*n + r_out."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    w = _diag_sums(s, n, cv, kw)                       # over c_out - c_in
    z = np.asarray(kernel, dtype=np.float64) @ w       # z[u] = sum_v K[u,v] w[v]
    return _broadcast(z, n, cu, s.dtype)


def ra_dense(kernel: np.ndarray, n: int) -> np.ndarray:
    """Dense R(A) from the closed-form entry map (tiny n only)."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    offs = _offsets(n)
    ui = offs + cu           # per column index Q = r_in*n + r_out
    vi = offs + cv           # per row index J = c_in*n + c_out
    okr = (vi >= 0) & (vi < kw)
    okc = (ui >= 0) & (ui < kh)
    out = np.zeros((n * n, n * n))
    rows = np.nonzero(okr)[0]
    cols = np.nonzero(okc)[0]
    out[np.ix_(rows, cols)] = np.asarray(kernel, dtype=np.float64)[ui[cols][None, :], vi[rows][:, None]]
    return out


def diag_counts(n: int, center: int, length: int) -> np.ndarray:
    """Number of grid cells on each diagonal index u = b - a + center."""
    u = np.arange(length) - center
    return np.maximum(n - np.abs(u), 0).astype(np.float64)


def structured_tsvd(kernel: np.ndarray, n: int, k: int | None = None):
    """Exact SVD of R(A) (float64): R = (W^_c U) S (W^_r V)^T with
    M = D_c K^T D_r = U S V^T and D = diag(sqrt(diagonal counts)).

    Returns (u, sigma, v) with u: n^2 x k (s-space), v: n^2 x k (q-space).
    """
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    dr = np.sqrt(diag_counts(n, cu, kh))
    dc = np.sqrt(diag_counts(n, cv, kw))
    m = dc[:, None] * np.asarray(kernel, dtype=np.float64).T * dr[None, :]
    um, sm, vmt = np.linalg.svd(m, full_matrices=False)
    if k is None:
        k = sm.size
    um, sm, vm = um[:, :k], sm[:k], vmt[:k].T
    with np.errstate(divide="ignore", invalid="ignore"):
        uc = np.where(dc[:, None] > 0, um / dc[:, None], 0.0)
        vc = np.where(dr[:, None] > 0, vm / dr[:, None], 0.0)
    u = np.stack([_broadcast(uc[:, i], n, cv, np.float64) for i in range(k)], axis=1)
    v = np.stack([_broadcast(vc[:, i], n, cu, np.float64) for i in range(k)], axis=1)
    return u, sm, v
