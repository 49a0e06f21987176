"""eGKB / RSVD / orthonormalize restated over matvec callables (CPU oracle).

TEST INFRASTRUCTURE ONLY.  The reference (``pkg/src/kronblur/lowrank.py``)
needs a dense ``b_mat`` (``lowrank.py:187``), so it cannot run past n ~ 128.
This restatement takes ``matvec(q) -> B q`` and ``rmatvec(s) -> B^T s``
callables and performs the *same floating-point operations in the same
order*; with ``matvec = B.__matmul__`` it is bit-identical to the reference
(pinned by ``tests/test_oracle_golden.py``).

Algorithm map:
  * rule classification          lowrank.py:114-125
  * auto_rank                    lowrank.py:128-150
  * one-pass MGS                 lowrank.py:153-156
  * eGKB main loop               lowrank.py:187-277
  * C / bases / lift / truncate  lowrank.py:279-329
  * RSVD                         lowrank.py:332-372
  * orthonormalize (2-pass MGS)  linalg.py:156-199
  * svd_small (LAPACK gesdd)     linalg.py:134-153
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

NU_SENTINEL = 1e308


class OracleRankDeficiency(ArithmeticError):
    def __init__(self, column: int):
        super().__init__(f"column {column} collapsed")
        self.column = column


class OracleNumericalError(ArithmeticError):
    pass


class OracleValidationError(ValueError):
    pass


@dataclass
class OracleTrace:
    alphas: list = field(default_factory=list)
    ts: list = field(default_factory=list)
    zetas: list = field(default_factory=list)
    nus: list = field(default_factory=list)
    chosen_k: int = 0
    k_p: int = 0
    stop_reason: str = ""
    breakdown: bool = False
    s_basis: np.ndarray | None = None
    q_basis: np.ndarray | None = None
    c_mat: np.ndarray | None = None


def classify(nu_prev: float, nu_j: float, tau: float):
    """Rise beats dip (lowrank.py:114-125)."""
    if nu_j > nu_prev:
        return "rise"
    return "dip" if nu_j < tau else None


def auto_rank(nus, tau, k_min=2, k_max=None):
    """lowrank.py:128-150."""
    vals = [float(x) for x in nus]
    if not vals:
        raise OracleValidationError("empty")
    top = len(vals) if k_max is None else k_max
    if vals[0] < tau:
        return max(1, k_min), "nu_below_tol"
    for j in range(2, len(vals) + 1):
        ev = classify(vals[j - 2], vals[j - 1], tau)
        if ev == "rise":
            return max(j - 1, k_min), "nu_rose"
        if ev == "dip":
            return max(j, k_min), "nu_below_tol"
    return top, "hit_kmax"


def project_out(vec, basis, dot=None):
    """Sequential one-pass MGS (lowrank.py:153-156).  ``dot`` replaces numpy's
    ``b @ vec`` (e.g. ``oracle.blas.sdot`` of another OpenBLAS kernel)."""
    for b in basis:
        vec = vec - ((b @ vec) if dot is None else dot(b, vec)) * b
    return vec


def svd_small(mat):
    """LAPACK SVD in the matrix dtype (linalg.py:134-153)."""
    u, s, vt = np.linalg.svd(np.asarray(mat), full_matrices=False)
    return u, s, vt.T


def egkb(matvec, rmatvec, shape, dtype, cfg, y0=None, kernel=None):
    """Enlarged Golub-Kahan bidiagonalization (lowrank.py:159-329).

    ``cfg`` needs k_max, p, tau, k_min, reorth, seed, break_tol, keep_basis.
    ``kernel`` (fp32 only): compute every dot product and norm as that OpenBLAS
    kernel does (``oracle.blas``) instead of with this host's numpy -- the
    reference run on a host with that kernel.  Returns ((u, sigma, v), trace).
    """
    dtype = np.dtype(dtype)
    if kernel is not None:
        from . import blas

        dot = lambda a, b: blas.sdot(a, b, kernel)   # noqa: E731
        vnorm = lambda x: blas.norm(x, kernel)       # noqa: E731
    else:
        dot = None
        vnorm = lambda x: float(np.linalg.norm(x))   # noqa: E731
    one = dtype.type
    mbar, nbar = shape
    tol = cfg.break_tol if cfg.break_tol is not None else np.sqrt(float(np.finfo(dtype).eps))
    mode = cfg.reorth or ("full" if dtype == np.float32 else "one-sided")

    if y0 is None:
        y0 = np.random.default_rng(cfg.seed).standard_normal(mbar).astype(dtype)
    else:
        y0 = np.asarray(y0, dtype=dtype)
        if y0.shape != (mbar,):
            raise OracleValidationError("bad y0 length")
    t_first = vnorm(y0)
    if t_first == 0.0:
        raise OracleValidationError("zero y0")
    left = [y0 / one(t_first)]
    first_q = rmatvec(left[0])
    a_first = vnorm(first_q)
    if a_first == 0.0:
        raise OracleNumericalError("operator annihilates the starting vector")
    right = [first_q / one(a_first)]

    tr = OracleTrace()
    tr.alphas.append(a_first)
    tr.ts.append(t_first)
    tr.zetas.append(a_first * t_first)
    tr.nus.append(NU_SENTINEL)

    fired = None
    why = ""
    broke = False
    broke_on_t = False
    done = 1

    while done < ((fired + cfg.p + 1) if fired is not None else (cfg.k_max + 1)):
        u = matvec(right[-1])
        cand = u - one(tr.alphas[-1]) * left[-1]
        if mode == "full":
            cand = project_out(cand, left, dot)
        t_val = vnorm(cand)
        if t_val <= tol * vnorm(u):
            broke = broke_on_t = True
            break
        s_next = cand / one(t_val)

        back = rmatvec(s_next)
        back_norm = vnorm(back)
        back = back - one(t_val) * right[-1]
        back = project_out(back, right, dot)
        a_val = vnorm(back)
        if a_val <= tol * back_norm:
            broke = True
            left.append(s_next)
            tr.ts.append(t_val)
            break
        right.append(back / one(a_val))
        left.append(s_next)
        tr.ts.append(t_val)
        tr.alphas.append(a_val)
        zeta = a_val * t_val
        nu = float(np.sqrt(zeta * tr.zetas[-1]))
        tr.zetas.append(zeta)
        tr.nus.append(nu)
        done += 1
        if fired is None:
            ev = classify(tr.nus[-2], nu, cfg.tau)
            if ev == "rise":
                fired, why = max(done - 1, cfg.k_min), "nu_rose"
            elif ev == "dip":
                fired, why = max(done, cfg.k_min), "nu_below_tol"

    if broke:
        k_p = done
        rows = done if broke_on_t else done + 1
    else:
        k_p, rows = done - 1, done
    if fired is not None:
        chosen, reason = min(fired, k_p), why
    elif broke:
        chosen, reason = k_p, "breakdown"
    else:
        chosen, reason = min(cfg.k_max, k_p), "hit_kmax"
    if chosen < 1 or k_p < 1:
        raise OracleNumericalError("breakdown before any factor")

    c = np.zeros((rows, k_p), dtype=dtype)
    for i in range(k_p):
        c[i, i] = tr.alphas[i]
        if i + 1 < rows:
            c[i + 1, i] = tr.ts[i + 1]
    sb = np.column_stack(left[:rows])
    qb = np.column_stack(right[:k_p])
    cu_, cs_, cv_ = svd_small(c)
    u_full = sb @ cu_
    v_full = qb @ cv_
    tr.chosen_k, tr.k_p, tr.stop_reason, tr.breakdown = chosen, k_p, reason, broke
    if cfg.keep_basis:
        tr.s_basis, tr.q_basis, tr.c_mat = sb, qb, c
    return (u_full[:, :chosen], cs_[:chosen], v_full[:, :chosen]), tr


def orthonormalize(mat, drop_tol=None):
    """Two-pass MGS per column with a drop tolerance (linalg.py:156-199)."""
    mat = np.asarray(mat)
    m, ncol = mat.shape
    if drop_tol is None:
        scale = float(np.linalg.norm(mat, axis=0).max()) if ncol else 0.0
        drop_tol = float(np.finfo(mat.dtype).eps) * np.sqrt(m) * scale
    q = mat.copy()
    for j in range(ncol):
        col = q[:, j]
        for _ in range(2):
            for i in range(j):
                col -= (q[:, i] @ col) * q[:, i]
        nrm = np.linalg.norm(col)
        if not np.isfinite(nrm):
            raise OracleNumericalError(f"non-finite norm at column {j}")
        if nrm <= drop_tol:
            raise OracleRankDeficiency(j)
        q[:, j] = col / nrm
    return q


def rsvd(matmat, rmatmat, shape, dtype, k, p, q, seed, hmat=None):
    """Randomized SVD with q power iterations (lowrank.py:332-372).

    ``matmat(F) -> B F`` and ``rmatmat(Y) -> B^T Y`` on 2-D blocks;
    ``hmat(Y) -> Y^T B`` (defaults to ``rmatmat(Y).T``).  Handles the wide
    case by swapping the roles, as lowrank.py:352-354 does.
    """
    mbar, nbar = shape
    if mbar < nbar:
        u, s, v = rsvd(rmatmat, matmat, (nbar, mbar), dtype, k, p, q, seed)
        return v, s, u
    kp = k + p
    if kp > nbar:
        raise OracleValidationError("k + p exceeds the smaller dimension")
    f = np.random.default_rng(seed).standard_normal((nbar, kp)).astype(dtype)
    y = orthonormalize(matmat(f))
    for _ in range(q):
        z = orthonormalize(rmatmat(y))
        y = orthonormalize(matmat(z))
    h = hmat(y) if hmat is not None else rmatmat(y).T
    hu, hs, hv = svd_small(h)
    u = y @ hu
    if not np.all(np.isfinite(hs)):
        raise OracleNumericalError("non-finite sigma")
    return u[:, :k], hs[:k], hv[:, :k]
