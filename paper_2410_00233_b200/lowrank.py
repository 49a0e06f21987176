"""Truncated-SVD engines on the GPU: eGKB, RSVD and the structured TSVD.

Reference: pkg/src/kronblur/lowrank.py.  Same configs, same validation, same
return layout (``TruncatedSvd`` + ``EgkbTrace``).  ``b_mat`` may be a dense
float32/float64 matrix (numpy or CUDA tensor) exactly as in the reference, or
a matrix-free :class:`~paper_2410_00233_b200.blurmodel.RearrangedBlur`.

Division of labour (north star item 2): the Krylov loop, the operator
products, the full reorthogonalisation and the lifts run in sm_100a kernels
(``kb_egkb_run``, ``kb_lift_assemble``).  The bidiagonal SVD of C runs on the
host, in C++ inside ``kb_egkb_run`` (fp64 one-sided Jacobi), and its lift
weights go to the device stream-ordered.  The rank rule and the breakdown
tests run on the device inside the fused kernel (the same fp64 scalar
comparisons in every CTA), or on the host in the reference-arithmetic engine.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib, rng
from .blurmodel import RearrangedBlur
from .sparse import RearrangedSparse
from .exceptions import NumericalError, ValidationError
from .linalg import TruncatedSvd, eps_for, orthonormalize_device, precision_of, svd_small

NU_SENTINEL = 1e308

STOP_NU_ROSE = "nu_rose"
STOP_NU_BELOW_TOL = "nu_below_tol"
STOP_HIT_KMAX = "hit_kmax"
STOP_BREAKDOWN = "breakdown"

REORTH_ONE_SIDED = "one-sided"
REORTH_FULL = "full"


@dataclass
class EgkbConfig:
    """Settings for :func:`egkb` (lowrank.py:35-68)."""

    k_max: int
    p: int = 2
    tau: float = 1e-4
    k_min: int = 2
    reorth: str | None = None
    seed: int = 0
    break_tol: float | None = None
    keep_basis: bool = False

    def __post_init__(self):
        if self.k_max < 1:
            raise ValidationError("k_max must be >= 1")
        if self.p < 0:
            raise ValidationError("p must be >= 0")
        if self.k_min < 1:
            raise ValidationError("k_min must be >= 1")
        if self.reorth not in (None, REORTH_ONE_SIDED, REORTH_FULL):
            raise ValidationError(
                f"reorth must be {REORTH_ONE_SIDED!r} or {REORTH_FULL!r}, got {self.reorth!r}")


@dataclass
class EgkbTrace:
    """Per-iteration scalars of a bidiagonalisation run (lowrank.py:71-92)."""

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


@dataclass
class RsvdConfig:
    """Settings for :func:`rsvd` (lowrank.py:95-111)."""

    k: int
    p: int = 2
    q: int = 1
    seed: int = 0

    def __post_init__(self):
        if self.k < 1:
            raise ValidationError("k must be >= 1")
        if self.p < 0:
            raise ValidationError("p must be >= 0")
        if self.q < 0:
            raise ValidationError("q must be >= 0")


def _rule_event(nu_prev: float, nu_j: float, tau: float):
    """Rise first (smaller rank), then dip (lowrank.py:114-125)."""
    if nu_j > nu_prev:
        return "rise"
    if nu_j < tau:
        return "dip"
    return None


def auto_rank(nus, tau: float, k_min: int = 2, k_max: int | None = None):
    """Scan nu values for the first rise / dip (lowrank.py:128-150)."""
    nus = [float(v) for v in nus]
    if not nus:
        raise ValidationError("auto_rank needs at least one nu value")
    if k_max is None:
        k_max = len(nus)
    if nus[0] < tau:
        return max(1, k_min), STOP_NU_BELOW_TOL
    for j in range(2, len(nus) + 1):
        event = _rule_event(nus[j - 2], nus[j - 1], tau)
        if event == "rise":
            return max(j - 1, k_min), STOP_NU_ROSE
        if event == "dip":
            return max(j, k_min), STOP_NU_BELOW_TOL
    return k_max, STOP_HIT_KMAX


# ----------------------------------------------------------------- operators
class _EngineOp:
    """A b_mat prepared for the device engines (dense upload or R(A))."""

    def __init__(self, b_mat):
        from . import device as D

        self.keep = None
        if isinstance(b_mat, (RearrangedBlur, RearrangedSparse)):
            self.kind = "ra" if isinstance(b_mat, RearrangedBlur) else "sparse"
            self.blur = b_mat
            self.dtype = b_mat.dtype
            self.shape = b_mat.shape
            self.struct = b_mat.op_struct()
            return
        if D.is_tensor(b_mat):
            if b_mat.ndim != 2:
                raise ValidationError("expects a matrix")
            precision_of(b_mat)
            self.mat = D.to_device(b_mat)
            self.dtype = D.np_dtype(self.mat)
        else:
            arr = np.asarray(b_mat)
            if arr.ndim != 2:
                raise ValidationError("expects a matrix")
            precision_of(arr)
            self.dtype = arr.dtype
            self.mat = D.to_device(arr)
        self.kind = "dense"
        self.shape = tuple(self.mat.shape)
        op = _lib.KbOperator()
        op.kind = _lib.KB_OP_DENSE
        op.dtype = _lib.KB_F32 if self.dtype == np.float32 else _lib.KB_F64
        op.rows, op.cols = self.shape
        op.a, op.lda = self.mat.data_ptr(), self.shape[1]
        op.k = op.kt = None
        op.kh = op.kw = op.side = 0
        self.struct = op

    @property
    def code(self) -> int:
        return _lib.KB_F32 if self.dtype == np.float32 else _lib.KB_F64

    def apply(self, x, transpose: int, out):
        """out = B x or B^T x (device vectors)."""
        from . import device as D

        lib = _lib.load()
        nb = C.c_size_t()
        _lib.check(lib.kb_op_workspace_bytes(C.byref(self.struct), C.byref(nb)))
        ws, wsb = D.WORKSPACE.get(nb.value)
        _lib.check(lib.kb_op_apply(C.byref(self.struct), x.data_ptr(), out.data_ptr(), transpose, ws, wsb,
                                   D.stream_ptr()), "operator apply")
        return out

    def apply_block(self, X, transpose: int):
        """Rows of X are vectors; returns rows B x_i (or B^T x_i) (kb_op_apply_block)."""
        from . import device as D

        rows_out = self.shape[1] if transpose else self.shape[0]
        X = X.contiguous()
        out = D.empty((X.shape[0], rows_out), self.dtype)
        lib = _lib.load()
        nb = C.c_size_t()
        _lib.check(lib.kb_op_workspace_bytes(C.byref(self.struct), C.byref(nb)))
        ws, wsb = D.WORKSPACE.get(nb.value)
        _lib.check(lib.kb_op_apply_block(C.byref(self.struct), X.data_ptr(), X.shape[1], out.data_ptr(), rows_out,
                                         X.shape[0], transpose, ws, wsb, D.stream_ptr()), "block apply")
        return out


def _lift(code, basis, nrows, W, out_rows):
    """out_c = sum_i W[i, c] basis_i  (device; lowrank.py:317-318, 369)."""
    from . import device as D

    cols = W.shape[1]
    length = basis.shape[1]
    out = D.empty((cols, length), D.np_dtype(basis))
    wd = D.upload(np.ascontiguousarray(W[:nrows]), D.np_dtype(basis))   # pinned, stream-ordered
    _lib.check(_lib.load().kb_ts_lift(code, basis.data_ptr(), length, nrows, wd.data_ptr(), cols, out.data_ptr(),
                                      length, length, D.stream_ptr()), "lift")
    return out


# ----------------------------------------------------------------- eGKB
_BASES: dict = {}


def _bases_key(cap, mbar, nbar, dtype):
    from . import device as D

    return (cap, mbar, nbar, np.dtype(dtype).str, D.device().index)


class _LazyLift:
    """U = S W_u, V = Q W_v (lowrank.py:317-318) kept as (basis, weights) until used.

    ``materialize`` runs the working-precision lift (kb_ts_lift); ``assemble``
    writes the fp64 factors sigma_i u_i and v_i directly (kb_lift_assemble,
    kronop.py:117-119) -- the same bits as materialising then assembling.
    """

    def __init__(self, code, s_part, q_part, cols, shape, sigma, keep, sigma_ptr):
        # s_part / q_part: (basis, rows used, device pointer of the weights, row stride cols);
        # `keep` owns the weights and sigma (device); sigma: host fp64 copy
        self.code, self.cols, self.shape = code, cols, shape
        self.parts = [s_part, q_part]
        self._keep = keep
        self.sigma_host = np.asarray(sigma, dtype=np.float64)
        self.sigma_ptr = sigma_ptr

    def materialize(self):
        from . import device as D

        out = []
        for basis, nrows, wd in self.parts:
            length = basis.shape[1]
            rows_out = D.empty((self.cols, length), D.np_dtype(basis))
            _lib.check(_lib.load().kb_ts_lift(self.code, basis.data_ptr(), length, nrows, wd, self.cols,
                                              rows_out.data_ptr(), length, length, D.stream_ptr()), "lift")
            out.append(rows_out)
        self.parts = None
        return out[0], out[1]

    def assemble(self, sigma, f, g):
        from . import device as D

        if not np.array_equal(np.asarray(sigma, dtype=np.float64), self.sigma_host):
            raise ValidationError("lazy lift: sigma does not belong to this factorisation")
        for (basis, nrows, wd), out, scale in zip(self.parts, (f, g), (self.sigma_ptr, None)):
            length = basis.shape[1]
            _lib.check(_lib.load().kb_lift_assemble(self.code, basis.data_ptr(), length, nrows, wd,
                                                    self.cols, scale,
                                                    out.data_ptr(), length, length, D.stream_ptr()),
                       "lift+assemble")


def _bases(cap, mbar, nbar, dtype, key=None):
    """Krylov bases per shape, reused across calls while no result holds them
    (a lazily-lifted result owns its bases; the next call then takes fresh
    ones from the caching allocator)."""
    from . import device as D

    key = key if key is not None else _bases_key(cap, mbar, nbar, dtype)
    hit = _BASES.get(key)
    if hit is None:
        if len(_BASES) >= 4:
            _BASES.pop(next(iter(_BASES)))
        hit = (D.empty((cap, mbar), dtype), D.empty((cap, nbar), dtype))
        _BASES[key] = hit
    return hit


_ARITH_LANES = {"skylakex": "openblas-skx", "cooperlake": "openblas-skx", "sapphirerapids": "openblas-skx",
                "haswell": "openblas-hsw", "zen": "openblas-hsw"}


def host_blas_arithmetic() -> str:
    """The ``arithmetic`` that reproduces numpy's fp32 dot products on this host:
    OpenBLAS's x86-64 sdot kernel that numpy's OpenBLAS dispatches to here
    (threadpoolctl reports its core name; ``OPENBLAS_CORETYPE`` changes it)."""
    from threadpoolctl import threadpool_info

    for info in threadpool_info():
        if info.get("internal_api") == "openblas":
            arch = str(info.get("architecture", "")).lower()
            if arch in _ARITH_LANES:
                return _ARITH_LANES[arch]
            raise ValidationError(f"no reference-arithmetic emulation for OpenBLAS kernel {arch!r}")
    raise ValidationError("numpy is not using OpenBLAS: no reference-arithmetic emulation")


_ARITH_CODES = {"fast": 0, "openblas-skx": 1, "openblas-hsw": 2}


def egkb(b_mat, config: EgkbConfig, y0=None, reorth_passes: int = 1, *, arithmetic: str = "fast"):
    """Enlarged Golub-Kahan bidiagonalisation with automatic rank choice
    (lowrank.py:159-329), on the GPU.

    ``arithmetic`` selects the engine:

    * ``"fast"`` (default): one persistent fused kernel; projections as one
      classical pass with fp64-accumulated coefficients and exact fp64 norms.
      ``reorth_passes=2`` selects CGS2.
    * ``"reference"``: the reference's own fp32 operations in its order --
      sequential modified Gram-Schmidt (lowrank.py:153-156) with every dot
      product and norm computed as numpy's OpenBLAS sdot computes it on this
      host (``host_blas_arithmetic()``; or name the kernel:
      ``"openblas-skx"`` / ``"openblas-hsw"``).  The trace (alpha, t, zeta,
      nu), the rank decision and the Krylov bases are then bit-identical to
      the reference's, also past the fp32 numerical rank where the fast
      engine's more accurate sums let the recurrence run one or two steps
      longer before it breaks down.  Matrix-free fp32 operators only.
    """
    from . import device as D

    y0_early = None
    if y0 is None and isinstance(b_mat, RearrangedBlur):
        # the reference's start vector (lowrank.py:199-201) drawn on the device first, so the
        # draw runs while the host validates / normalises / uploads the PSF (op_struct)
        y0_early = rng.standard_normal(config.seed, b_mat.shape[0], b_mat.dtype)
    op = _EngineOp(b_mat)
    dtype = np.dtype(op.dtype)
    mbar, nbar = op.shape
    eps = eps_for(dtype)
    break_tol = config.break_tol if config.break_tol is not None else np.sqrt(eps)
    reorth = config.reorth
    if reorth is None:
        reorth = REORTH_FULL if dtype == np.float32 else REORTH_ONE_SIDED

    y0d = None
    if y0 is None:
        # the reference's draws (lowrank.py:199-201), generated on the device; launched
        # first, so the draw runs while the host prepares the eGKB launch
        y0d = y0_early if y0_early is not None else rng.standard_normal(config.seed, mbar, dtype)
    elif D.is_tensor(y0):
        y0d = D.to_device(y0, dtype)
        if tuple(y0d.shape) != (mbar,):
            raise ValidationError(f"y0 must have length {mbar}, got shape {tuple(y0d.shape)}")
    else:
        y0 = np.asarray(y0, dtype=dtype)
        if y0.shape != (mbar,):
            raise ValidationError(f"y0 must have length {mbar}, got shape {y0.shape}")
        y0d = D.to_device(y0)

    if arithmetic == "reference":
        arithmetic = host_blas_arithmetic()
    if arithmetic not in _ARITH_CODES:
        raise ValidationError(f"unknown arithmetic {arithmetic!r}")
    if arithmetic != "fast" and (dtype != np.float32 or op.kind == "dense"):
        raise ValidationError("arithmetic='reference' reproduces the fp32 recurrence on matrix-free operators")
    cfg = _lib.KbEgkbConfig(config.k_max, config.p, config.k_min, float(config.tau), float(break_tol),
                            1 if reorth == REORTH_FULL else 0, int(reorth_passes), _ARITH_CODES[arithmetic])
    lib = _lib.load()
    cap = lib.kb_egkb_capacity(C.byref(cfg))
    bkey = _bases_key(cap, mbar, nbar, dtype)
    s_basis, q_basis = _bases(cap, mbar, nbar, dtype, bkey)
    hist = np.zeros((7, cap), dtype=np.float64)
    dp = C.POINTER(C.c_double)
    st = _lib.KbEgkbState()
    st.s_basis, st.ld_s, st.q_basis, st.ld_q, st.capacity = s_basis.data_ptr(), mbar, q_basis.data_ptr(), nbar, cap
    st.alphas_host = hist[0].ctypes.data_as(dp)
    st.ts_host = hist[1].ctypes.data_as(dp)
    st.zetas_host = hist[2].ctypes.data_as(dp)
    st.nus_host = hist[3].ctypes.data_as(dp)
    st.s_scale_host = hist[4].ctypes.data_as(dp)
    st.q_scale_host = hist[5].ctypes.data_as(dp)
    # the small SVD of C (host, C++ Jacobi) and the lift weights are uploaded right after the
    # loop (kb_egkb_state.wu_dev): W_u, W_v (working dtype) and sigma (fp64) in one buffer
    esz = np.dtype(dtype).itemsize
    wbytes = (cap * cap * esz + 15) // 16 * 16
    svdbuf = D.empty(((2 * wbytes + 8 * cap) // 8,), np.float64)
    wu_ptr = svdbuf.data_ptr()
    wv_ptr = wu_ptr + wbytes
    st.wu_dev, st.wv_dev = wu_ptr, wv_ptr
    st.sigma_dev = C.cast(C.c_void_p(wu_ptr + 2 * wbytes), dp)
    st.sigma_host = hist[6].ctypes.data_as(dp)
    nb = C.c_size_t()
    _lib.check(lib.kb_egkb_workspace_bytes(C.byref(op.struct), cap, C.byref(nb)))
    ws, wsb = D.WORKSPACE.get(nb.value)
    status = lib.kb_egkb_run(C.byref(op.struct), C.byref(cfg), y0d.data_ptr(), C.byref(st), ws, wsb,
                             D.stream_ptr())
    _lib.check(status, "egkb")

    trace = EgkbTrace()
    trace.alphas = [float(v) for v in hist[0, : st.n_alphas]]
    trace.ts = [float(v) for v in hist[1, : st.n_ts]]
    trace.zetas = [float(v) for v in hist[2, : st.n_nus]]
    trace.nus = [float(v) for v in hist[3, : st.n_nus]]
    k_p, rows, chosen = st.k_p, st.rows, st.chosen_k

    sigma = hist[6, :chosen].copy()            # fp64 of the working-precision values
    if not np.all(np.isfinite(sigma)):
        raise NumericalError("bidiagonal SVD produced non-finite singular values")
    lazy = _LazyLift(op.code, (s_basis, rows, wu_ptr), (q_basis, k_p, wv_ptr), chosen, (mbar, nbar), sigma,
                     svdbuf, wu_ptr + 2 * wbytes)
    _BASES.pop(bkey, None)   # the result owns these bases now

    trace.chosen_k = chosen
    trace.k_p = k_p
    trace.stop_reason = _lib.KB_STOP[st.stop_reason]
    trace.breakdown = bool(st.breakdown)
    if config.keep_basis:
        c_mat = np.zeros((rows, k_p), dtype=dtype)
        for i in range(k_p):
            c_mat[i, i] = trace.alphas[i]
            if i + 1 < rows:
                c_mat[i + 1, i] = trace.ts[i + 1]
        # stored vectors x scale = the normalised basis (the fused engine defers the division)
        sc_s, sc_q = hist[4, :rows], hist[5, :k_p]
        sb = D.to_host(s_basis[:rows]).T
        qb = D.to_host(q_basis[:k_p]).T
        trace.s_basis = sb if np.all(sc_s == 1.0) else (sb.astype(np.float64) * sc_s).astype(dtype)
        trace.q_basis = qb if np.all(sc_q == 1.0) else (qb.astype(np.float64) * sc_q).astype(dtype)
        trace.c_mat = c_mat
    return TruncatedSvd.from_lift(lazy, sigma.astype(dtype)), trace


# ----------------------------------------------------------------- RSVD
def rsvd(b_mat, config: RsvdConfig) -> TruncatedSvd:
    """Randomised truncated SVD with q subspace iterations (lowrank.py:332-372).

    Block products and every orthonormalisation (with the reference's
    rank-deficiency test) run on the GPU; the SVD of the projected k+p row
    block H stays on the host (LAPACK, as the reference).
    """
    from . import device as D

    op = _EngineOp(b_mat)
    mbar, nbar = op.shape
    if mbar < nbar:
        if op.kind == "ra":
            raise ValidationError("wide matrix-free operators are not supported")
        inner = rsvd(op.blur.T if op.kind == "sparse" else op.mat.t().contiguous(), config)
        return TruncatedSvd.from_device(inner.v_device, inner.sigma, inner.u_device)
    k_p = config.k + config.p
    if k_p > nbar:
        raise ValidationError(f"k + p = {k_p} exceeds the smaller matrix dimension {nbar}")
    dtype = np.dtype(op.dtype)
    # the reference's test matrix (lowrank.py:361-362), drawn on the device, stored transposed
    fd = rng.standard_normal(config.seed, (nbar, k_p), dtype, transpose=True)
    y = orthonormalize_device(op.apply_block(fd, 0))
    for _ in range(config.q):
        z = orthonormalize_device(op.apply_block(y, 1))
        y = orthonormalize_device(op.apply_block(z, 0))
    hd = op.apply_block(y, 1)                 # rows: (B^T y_c)^T = y_c^T B  -> H (k_p x nbar)
    if dtype == np.float32 and k_p * nbar >= _RSVD_GRAM_MIN:
        small = _svd_wide_gram(op.code, hd, k_p, config.k)
        if small is not None:                 # H = U_H S V_H^T from its k_p x k_p Gram matrix
            u_h, sigma, v_rows = small
            u_rows = _lift(op.code, y, k_p, u_h, config.k)
            return TruncatedSvd.from_device(u_rows, sigma, v_rows)
    core = svd_small(D.to_host(hd))
    if not np.all(np.isfinite(core.sigma)):
        raise NumericalError("randomized SVD produced non-finite singular values")
    u_rows = _lift(op.code, y, k_p, core.u[:, : config.k], config.k)
    v_rows = D.to_device(np.ascontiguousarray(core.v[:, : config.k].T))
    return TruncatedSvd.from_device(u_rows, core.sigma[: config.k].copy(), v_rows)


_RSVD_GRAM_MIN = 1 << 18   # below this the host SVD of H costs less than it saves


def _svd_wide_gram(code, hd, k_p, k):
    """SVD of the wide fp32 block H (k_p x nbar, device) without moving it to the host:
    G = H H^T from k_p fp64-accumulated row-dot passes (kb_ts_dots), its k_p x k_p
    eigenproblem on the host (G = U_H S^2 U_H^T), and the right vectors as the lift
    V_H^T = S^-1 U_H^T H.  For fp32 data the fp64 Gram matrix carries sigma_i to
    1e-16 (sigma_1 / sigma_i)^2, far below the working precision; returns None (the
    caller then takes the reference's LAPACK path) when a wanted sigma_i is not safely
    above that floor.  (lowrank.py:368-371: svd_small(H), U = Y U_H.)"""
    from . import device as D

    lib = _lib.load()
    nbar = hd.shape[1]
    out = D.empty((k_p, k_p + 1), np.float64)
    nb = C.c_size_t()
    _lib.check(lib.kb_orth_workspace_bytes(nbar, k_p + 2, C.byref(nb)))   # covers kb_ts_dots with m = k_p
    ws, wsb = D.WORKSPACE.get(nb.value + 8 * (k_p + 64))
    for i in range(k_p):
        _lib.check(lib.kb_ts_dots(code, hd.data_ptr(), nbar, k_p, hd[i].data_ptr(), nbar, out[i].data_ptr(), ws, wsb,
                                  D.stream_ptr()), "gram")
    g = D.to_host(out)[:, :k_p]
    g = 0.5 * (g + g.T)
    lam, vec = np.linalg.eigh(g)
    order = np.argsort(lam)[::-1]
    lam, vec = lam[order], vec[:, order]
    if not np.all(np.isfinite(lam)):
        raise NumericalError("randomized SVD produced non-finite singular values")
    sig = np.sqrt(np.maximum(lam, 0.0))
    if sig[0] == 0.0 or sig[k - 1] <= 1e-6 * sig[0]:
        return None
    u_h = vec[:, :k]
    v_rows = _lift(code, hd, k_p, u_h / sig[None, :k], k)
    return u_h.astype(np.float32), sig[:k].astype(np.float32), v_rows


# ----------------------------------------------------------------- TSVD
def _ra_gram(n: int, center: int, length: int) -> np.ndarray:
    """G = P^T P for the reflexive-BC incidence P (length x length).

    Cell (a, b) hits u = b - a + c, a + b + 1 + c and a + b + c + 1 - 2n
    (each at most once); G counts co-hits: O(n^2) host work, done once per TSVD.
    """
    ar = np.arange(n, dtype=np.int64)
    a = np.repeat(ar, n)
    b = np.tile(ar, n)
    s = a + b + 1 + center
    fams = (b - a + center, s, s - 2 * n)
    valid = [(u >= 0) & (u < length) for u in fams]
    g = np.zeros(length * length)
    for i in range(3):
        for j in range(3):
            m = valid[i] & valid[j]
            g += np.bincount(fams[i][m] * length + fams[j][m], minlength=length * length)
    return g.reshape(length, length)


def _half_inverse_factor(g: np.ndarray):
    """(E L^1/2, E L^-1/2) over the positive eigenpairs of the Gram matrix G = E L E^T."""
    lam, e = np.linalg.eigh(g)
    keep = lam > lam.max() * 1e-12
    lam, e = lam[keep], e[:, keep]
    return e * np.sqrt(lam)[None, :], e / np.sqrt(lam)[None, :]


def tsvd(b_mat, k: int) -> TruncatedSvd:
    """Exact top-k SVD of R(A).

    For a :class:`RearrangedBlur` this is structured:
    R = (W^_c U) S (W^_r V)^T with M = D_c K^T D_r = U S V^T, a (kw x kh)
    host SVD, lifted to n^2-vectors by the Toeplitz-broadcast kernel.  The
    reflexive BC uses the Gram matrices G = P^T P of its Toeplitz + Hankel
    incidence instead of the diagonal D^2 (eigh on the host, same lift).  This
    replaces ``svd_small(rearrange(A)).truncate(k)`` (linalg.py:128-153),
    which the reference can only run for n <= 64.  Dense inputs take the
    reference route (``svd_small``).
    """
    from . import device as D

    if not isinstance(b_mat, RearrangedBlur):
        return svd_small(np.asarray(b_mat)).truncate(k)
    blur = b_mat
    n = blur.n
    kern = blur.psf.kernel
    kh, kw = kern.shape
    cu, cv = kh // 2, kw // 2
    refl = blur.bc == "reflexive"
    if not refl:
        dr = np.sqrt(np.maximum(n - np.abs(np.arange(kh) - cu), 0).astype(np.float64))
        dc = np.sqrt(np.maximum(n - np.abs(np.arange(kw) - cv), 0).astype(np.float64))
        m = dc[:, None] * kern.T * dr[None, :]
        um, sm, vmt = np.linalg.svd(m, full_matrices=False)
        if not 0 < k <= sm.size:
            raise ValidationError(f"cannot truncate rank-{sm.size} factorization to k={k}")
        with np.errstate(divide="ignore", invalid="ignore"):
            uc = np.where(dc[:, None] > 0, um[:, :k] / dc[:, None], 0.0).T    # (k, kw)
            vc = np.where(dr[:, None] > 0, vmt[:k].T / dr[:, None], 0.0).T    # (k, kh)
    else:
        # G = P^T P = E L E^T;  M = (E_c L_c^1/2)^T K^T (E_r L_r^1/2) = U S V^T;
        # singular vectors P (E L^-1/2 U)  (Toeplitz + Hankel broadcast on the device)
        br, cr = _half_inverse_factor(_ra_gram(n, cu, kh))
        bcc, ccc = _half_inverse_factor(_ra_gram(n, cv, kw))
        um, sm, vmt = np.linalg.svd(bcc.T @ kern.T @ br, full_matrices=False)
        if not 0 < k <= sm.size:
            raise ValidationError(f"cannot truncate rank-{sm.size} factorization to k={k}")
        uc = (ccc @ um[:, :k]).T
        vc = (cr @ vmt[:k].T).T
    dtype = blur.dtype
    code = _lib.KB_F32 if dtype == np.float32 else _lib.KB_F64
    lib = _lib.load()
    u_rows = D.empty((k, n * n), dtype)
    v_rows = D.empty((k, n * n), dtype)
    ucd = D.to_device(np.ascontiguousarray(uc), dtype)
    vcd = D.to_device(np.ascontiguousarray(vc), dtype)
    _lib.check(lib.kb_toeplitz_lift(code, ucd.data_ptr(), kw, kw, cv, k, n, int(refl), u_rows.data_ptr(), n * n,
                                    D.stream_ptr()), "toeplitz lift")
    _lib.check(lib.kb_toeplitz_lift(code, vcd.data_ptr(), kh, kh, cu, k, n, int(refl), v_rows.data_ptr(), n * n,
                                    D.stream_ptr()), "toeplitz lift")
    return TruncatedSvd.from_device(u_rows, sm[:k].astype(dtype), v_rows)
