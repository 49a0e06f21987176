"""Matrix-free R(A) for a PSF blur, zero or reflexive BC (CPU oracle, test infra only).

Index conventions (reference ``pkg/src/kronblur/``):

* ``blurmodel.py:106-121``: A[c_out*n + r_out, c_in*n + r_in] += K[u, v] with
  r_in = r_out - u + cu, c_in = c_out - v + cv (zero BC drops out-of-range).
* ``rearrange.py:67-75`` with the square scheme ``rearrange.py:54-57``:
  R[j*n + i, q*n + p] = A[i*n + p, j*n + q].

Together:  R[c_in*n + c_out, r_in*n + r_out] =
K[r_out - r_in + cu, c_out - c_in + cv]  (zero when the K index is out of
range), i.e. R = W_c K^T W_r^T with 0/1 diagonal-indicator matrices W.

``ra_matvec``/``ra_rmatvec`` evaluate R q and R^T s in O(n^2 + kh*kw) work by
diagonal sums -> small K product -> Toeplitz broadcast, every sum in fp64 in a
fixed sequential order (np.bincount's input order; kernel rows in index order),
then one rounding to the vector dtype.  ``ra_dense`` builds the
dense R for tiny n (used to pin the closed form against the reference).
``structured_tsvd`` is the exact SVD of R through D_c K^T D_r.

Reflexive BC (``blurmodel.py:80-84, 122-126``: out-of-range input indices
reflect as -1-i and 2n-1-i, one reflection).  R = P_c K^T P_r^T where cell
(a, b) of P hits u = b - a + c (Toeplitz) and also u = a + b + 1 + c and
u = a + b + c + 1 - 2n (Hankel).  The same three steps apply with the hits of
both families; the exact SVD goes through the Gram matrices G = P^T P
(``structured_tsvd(..., bc="reflexive")``).
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


_HITS_CACHE: dict = {}


def _hits(n: int, center: int, length: int, bc: str = "zero"):
    """(cells, u) incidence pairs of P, Toeplitz family first, then the two
    Hankel families (reflexive BC), in cell order within each family."""
    key = (n, center, length, bc)
    h = _HITS_CACHE.get(key)
    if h is None:
        ar = np.arange(n, dtype=np.int64)
        a = np.repeat(ar, n)
        b = np.tile(ar, n)
        fams = [b - a + center]
        if bc == "reflexive":
            fams += [a + b + 1 + center, a + b + center + 1 - 2 * n]
        elif bc != "zero":
            raise ValueError(f"unknown boundary condition {bc!r}")
        cells, us = [], []
        for u in fams:
            keep = (u >= 0) & (u < length)
            cells.append(np.nonzero(keep)[0])
            us.append(u[keep])
        h = (np.concatenate(cells), np.concatenate(us))
        _HITS_CACHE.clear()
        _HITS_CACHE[key] = h
    return h


def _diag_sums(vec: np.ndarray, n: int, center: int, length: int, bc: str = "zero") -> np.ndarray:
    """w[u] = sum of vec over the cells that hit u (P^T vec), u in [0, length)."""
    if bc == "zero":
        idx = _offsets(n) + center
        keep = (idx >= 0) & (idx < length)
        return np.bincount(idx[keep], weights=vec[keep].astype(np.float64), minlength=length)
    cells, us = _hits(n, center, length, bc)
    return np.bincount(us, weights=vec[cells].astype(np.float64), minlength=length)


def _broadcast(z: np.ndarray, n: int, center: int, dtype, bc: str = "zero") -> np.ndarray:
    """out = P z: out[a*n + b] = z[b - a + center] (+ Hankel terms, reflexive), fp64 sums."""
    if bc == "zero":
        idx = _offsets(n) + center
        keep = (idx >= 0) & (idx < z.size)
        out = np.zeros(n * n, dtype=dtype)
        out[keep] = z[idx[keep]]
        return out
    cells, us = _hits(n, center, z.size, bc)
    return np.bincount(cells, weights=np.asarray(z, dtype=np.float64)[us], minlength=n * n).astype(dtype)


def _kernel_product(kernel: np.ndarray, w: np.ndarray, transpose: bool) -> np.ndarray:
    """z = K^T w (z[v] = sum_u K[u,v] w[u]) or, transpose, z = K w (z[u] = sum_v K[u,v] w[v]).

    Every entry is a sequential fp64 sum of rounded fp64 products in index order
    (numpy's elementwise multiply and add, one kernel row / column at a time).  A
    fixed evaluation order instead of a BLAS dgemv, whose summation order depends
    on the host's OpenBLAS kernel and thread count; the device's reference-order
    product (kb_refarith.cu) repeats it bit for bit."""
    k64 = np.asarray(kernel, dtype=np.float64)
    if transpose:
        k64 = np.ascontiguousarray(k64.T)
    # numpy reduces axis 0 of a C-ordered array row by row: z = ((p_0 + p_1) + p_2) + ...,
    # the same bits as the explicit loop (pinned in tests/test_oracle_golden.py)
    return (k64 * w[:, None]).sum(axis=0)


def ra_matvec(kernel: np.ndarray, n: int, q: np.ndarray, bc: str = "zero") -> np.ndarray:
    """y = R(A) q.  q is indexed r_in*n + r_out, y is indexed c_in*n + c_out."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    w = _diag_sums(q, n, cu, kh, bc)                   # P_r^T q
    z = _kernel_product(kernel, w, False)              # z[v] = sum_u K[u,v] w[u]
    return _broadcast(z, n, cv, q.dtype, bc)


def ra_rmatvec(kernel: np.ndarray, n: int, s: np.ndarray, bc: str = "zero") -> np.ndarray:
    """x = R(A)^T s.  s is indexed c_in*n + c_out, x is indexed r_in*n + r_out."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    w = _diag_sums(s, n, cv, kw, bc)                   # P_c^T s
    z = _kernel_product(kernel, w, True)               # z[u] = sum_v K[u,v] w[v]
    return _broadcast(z, n, cu, s.dtype, bc)


def incidence(n: int, center: int, length: int, bc: str = "zero") -> np.ndarray:
    """Dense P (n^2 x length) with P[cell, u] = number of hits (tiny n only)."""
    cells, us = _hits(n, center, length, bc)
    p = np.zeros((n * n, length))
    np.add.at(p, (cells, us), 1.0)
    return p


def gram(n: int, center: int, length: int, bc: str = "zero") -> np.ndarray:
    """G = P^T P (length x length): co-hit counts of the index families."""
    cells, us = _hits(n, center, length, bc)
    order = np.argsort(cells, kind="stable")
    cells, us = cells[order], us[order]
    g = np.zeros((length, length))
    # every cell hits at most 3 indices: pair hits within each cell
    starts = np.flatnonzero(np.r_[True, cells[1:] != cells[:-1]])
    counts = np.diff(np.r_[starts, cells.size])
    for i in range(3):
        for j in range(3):
            sel = counts > max(i, j)
            ui, uj = us[starts[sel] + i], us[starts[sel] + j]
            g += np.bincount(ui * length + uj, minlength=length * length).reshape(length, length)
    return g


def ra_dense(kernel: np.ndarray, n: int, bc: str = "zero") -> np.ndarray:
    """Dense R(A) from the closed-form entry map (tiny n only)."""
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    if bc != "zero":
        return incidence(n, cv, kw, bc) @ np.asarray(kernel, dtype=np.float64).T @ incidence(n, cu, kh, bc).T
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


def _half_inverse_factor(g: np.ndarray):
    """(B, C) with B = E L^{1/2}, C = E L^{-1/2} over the positive eigenpairs of G = E L E^T."""
    lam, e = np.linalg.eigh(g)
    keep = lam > lam.max() * 1e-12
    lam, e = lam[keep], e[:, keep]
    return e * np.sqrt(lam)[None, :], e / np.sqrt(lam)[None, :]


def structured_tsvd(kernel: np.ndarray, n: int, k: int | None = None, bc: str = "zero"):
    """Exact SVD of R(A) (float64).

    Zero BC: R = (W^_c U) S (W^_r V)^T with M = D_c K^T D_r = U S V^T and
    D = diag(sqrt(diagonal counts)).  Reflexive BC: with G = P^T P = E L E^T,
    M = (E_c L_c^{1/2})^T K^T (E_r L_r^{1/2}) = U S V^T and the singular
    vectors are P_c E_c L_c^{-1/2} U, P_r E_r L_r^{-1/2} V.

    Returns (u, sigma, v) with u: n^2 x k (s-space), v: n^2 x k (q-space).
    """
    kh, kw = kernel.shape
    cu, cv = kh // 2, kw // 2
    kern = np.asarray(kernel, dtype=np.float64)
    if bc != "zero":
        br, cr = _half_inverse_factor(gram(n, cu, kh, bc))
        bcc, ccc = _half_inverse_factor(gram(n, cv, kw, bc))
        m = bcc.T @ kern.T @ br
        um, sm, vmt = np.linalg.svd(m, full_matrices=False)
        if k is None:
            k = sm.size
        uc = ccc @ um[:, :k]
        vc = cr @ vmt[:k].T
        u = np.stack([_broadcast(uc[:, i], n, cv, np.float64, bc) for i in range(k)], axis=1)
        v = np.stack([_broadcast(vc[:, i], n, cu, np.float64, bc) for i in range(k)], axis=1)
        return u, sm[:k], v
    dr = np.sqrt(diag_counts(n, cu, kh))
    dc = np.sqrt(diag_counts(n, cv, kw))
    m = dc[:, None] * kern.T * dr[None, :]
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
