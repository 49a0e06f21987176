"""Split Bregman TV deblurring on the GPU (reference: splitbregman.py).

``sb_run`` keeps the reference signature and result type; the outer loop,
the CGLS inner loop, the shrinkage / Bregman updates and the per-iteration
norms (rc, RE, ISNR) run in libkronblur_b200 (``kb_sb_run``), fp64.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cgls import CglsConfig, _device_forward
from .exceptions import ValidationError
from .metrics import FlopCounter

VARIANT_ANISOTROPIC = "anisotropic"
VARIANT_ISOTROPIC = "isotropic"
VARIANTS = (VARIANT_ANISOTROPIC, VARIANT_ISOTROPIC)
SB_CONVERGED = "converged"
SB_MAX_ITER = "max_iter"


def _shrink_pair(cx, cy, gamma_x, gamma_y, variant):
    from . import device as D

    host = not D.is_tensor(cx)
    a = D.to_device(np.atleast_1d(np.asarray(cx, dtype=np.float64)) if host else cx, np.float64).reshape(-1)
    b = D.to_device(np.atleast_1d(np.asarray(cy, dtype=np.float64)) if host else cy, np.float64).reshape(-1)
    if a.numel() != b.numel():
        raise ValidationError("cx and cy must have the same length")
    if gamma_x != gamma_y:
        # per-direction thresholds: run each direction with its own gamma
        dx1, _ = _shrink_pair(cx, cy, gamma_x, gamma_x, variant)
        _, dy2 = _shrink_pair(cx, cy, gamma_y, gamma_y, variant)
        return dx1, dy2
    dx = D.empty(a.numel(), np.float64)
    dy = D.empty(a.numel(), np.float64)
    code = _lib.KB_SB_ISOTROPIC if variant == VARIANT_ISOTROPIC else _lib.KB_SB_ANISOTROPIC
    _lib.check(_lib.load().kb_shrink_update(a.data_ptr(), b.data_ptr(), dx.data_ptr(), dy.data_ptr(), a.numel(),
                                            float(gamma_x), code, D.stream_ptr()), "shrink")
    if host:
        return D.to_host(dx), D.to_host(dy)
    return dx, dy


def shrink(w, v):
    """sign(w) max(|w| - v, 0) elementwise (splitbregman.py:32-35)."""
    w = np.asarray(w, dtype=np.float64)
    return np.sign(w) * np.maximum(np.abs(w) - v, 0.0)


def update_d_aniso(cx, cy, gamma_x: float, gamma_y: float):
    """Componentwise shrinkage, thresholds 1/gamma (GPU; splitbregman.py:38-40)."""
    return _shrink_pair(cx, cy, gamma_x, gamma_y, VARIANT_ANISOTROPIC)


def update_d_iso(cx, cy, gamma_x: float, gamma_y: float):
    """Coupled shrinkage on hypot(cx, cy) (GPU; splitbregman.py:43-56)."""
    return _shrink_pair(cx, cy, gamma_x, gamma_y, VARIANT_ISOTROPIC)


def update_g(gx, gy, x, dx, dy, n: int):
    from .regularizers import diff_x, diff_y

    return gx + diff_x(x, n) - dx, gy + diff_y(x, n) - dy


@dataclass
class SbConfig:
    """Split Bregman parameters (splitbregman.py:64-98)."""

    lam: float
    beta: float
    variant: str = VARIANT_ANISOTROPIC
    tau: float = 1e-3
    l_max: int = 50
    cgls: CglsConfig = field(default_factory=CglsConfig)
    warm_start: bool = False

    def __post_init__(self):
        if self.variant not in VARIANTS:
            raise ValidationError(f"variant must be one of {VARIANTS}, got {self.variant!r}")
        if self.lam <= 0 or self.beta <= 0:
            raise ValidationError("lam and beta must be positive")
        if self.l_max < 1:
            raise ValidationError("l_max must be >= 1")
        if self.tau < 0:
            raise ValidationError("tau must be >= 0")

    @property
    def gamma(self) -> float:
        return self.lam ** 2 / self.beta

    @classmethod
    def from_gamma(cls, lam: float, gamma: float, **kwargs) -> "SbConfig":
        if gamma <= 0:
            raise ValidationError("gamma must be positive")
        return cls(lam=lam, beta=lam ** 2 / gamma, **kwargs)


@dataclass
class SbResult:
    x: np.ndarray
    outer_iters: int
    stop: str
    rc_history: list = field(default_factory=list)
    re_history: list = field(default_factory=list)
    isnr_history: list = field(default_factory=list)
    cgls_iters: list = field(default_factory=list)

    @property
    def iota_total(self) -> int:
        return int(sum(self.cgls_iters))

    @property
    def converged(self) -> bool:
        return self.stop == SB_CONVERGED


def sb_run(op, b, config: SbConfig, x_true=None, counter: FlopCounter | None = None) -> SbResult:
    """Deblur ``b`` with split Bregman (splitbregman.py:120-192), on the GPU."""
    from . import device as D

    op = _device_forward(op)
    m_rows, n_cols = op.shape
    if m_rows != n_cols:
        raise ValidationError(f"operator must be square to start from the observed image, got {op.shape}")
    n = int(round(np.sqrt(n_cols)))
    if n * n != n_cols:
        raise ValidationError(f"operator size {n_cols} is not a perfect square")
    host = not D.is_tensor(b)
    bd = D.to_device(np.asarray(b, dtype=np.float64).ravel() if host else b, np.float64).reshape(-1)
    if bd.numel() != n_cols:
        raise ValidationError(f"b must have length {n_cols}, got {bd.numel()}")
    xtd = None
    if x_true is not None:
        xtd = D.to_device(np.asarray(x_true, dtype=np.float64).ravel() if not D.is_tensor(x_true) else x_true,
                          np.float64).reshape(-1)
        if xtd.numel() != n_cols:
            raise ValidationError(f"x_true must have length {n_cols}, got {xtd.numel()}")
    L = config.l_max
    rc, re, isnr = np.zeros(L), np.zeros(L), np.zeros(L)
    it = np.zeros(L, dtype=np.int32)
    dp = C.POINTER(C.c_double)
    st = _lib.KbSbState()
    st.lam, st.beta = float(config.lam), float(config.beta)
    st.variant = _lib.KB_SB_ISOTROPIC if config.variant == VARIANT_ISOTROPIC else _lib.KB_SB_ANISOTROPIC
    st.tau, st.l_max = float(config.tau), L
    st.i_max, st.tau_cgls = config.cgls.i_max, float(config.cgls.tau)
    st.warm_start = 1 if config.warm_start else 0
    st.rc_host, st.re_host, st.isnr_host = rc.ctypes.data_as(dp), re.ctypes.data_as(dp), isnr.ctypes.data_as(dp)
    st.cgls_iters_host = it.ctypes.data_as(C.POINTER(C.c_int))
    fw = op.forward_struct()
    x = D.empty(n_cols, np.float64)
    lib = _lib.load()
    nb = C.c_size_t()
    _lib.check(lib.kb_sb_workspace_bytes(C.byref(fw), C.byref(nb)))
    ws, wsb = D.WORKSPACE.get(nb.value)
    _lib.check(lib.kb_sb_run(C.byref(fw), bd.data_ptr(), None if xtd is None else xtd.data_ptr(), x.data_ptr(),
                             C.byref(st), ws, wsb, D.stream_ptr()), "sb_run")
    k = st.outer_iters
    res = SbResult(x=D.to_host(x) if host else x, outer_iters=k, stop=_lib.SB_STOPS[st.stop],
                   rc_history=[float(v) for v in rc[:k]], cgls_iters=[int(v) for v in it[:k]])
    if x_true is not None:
        res.re_history = [float(v) for v in re[:k]]
        res.isnr_history = [float(v) for v in isnr[:k]]
    if counter is not None and hasattr(op, "scheme"):
        s = op.scheme
        for ii in res.cgls_iters:
            for _ in range(ii + (1 if config.warm_start else 0)):
                counter.add_kp(s.m1, s.m2, s.n1, s.n2, op.k)
            for _ in range(ii + 1):
                counter.add_kp_transpose(s.m1, s.m2, s.n1, s.n2, op.k)
    return res


def lambda_grid(lam_lo: float, lam_hi: float, count: int = 100) -> np.ndarray:
    if lam_lo <= 0 or lam_hi <= lam_lo:
        raise ValidationError("need 0 < lam_lo < lam_hi")
    if count < 2:
        raise ValidationError("count must be >= 2")
    return np.logspace(np.log10(lam_lo), np.log10(lam_hi), count)


def sb_run_batch(op, b, configs, x_true=None) -> list:
    """Several SB solves of one observation in lock step (device, one launch per pass).

    ``configs`` are :class:`SbConfig` objects that may differ in ``lam`` /
    ``beta`` only.  Each result equals ``sb_run(op, b, config, x_true)`` of its
    config (splitbregman.py:120-192); the Kronecker products of all problems
    run as one pair of batched DMMA GEMMs (``kb_sb_run_batch``).  Dense
    operators are solved one after another with :func:`sb_run`.
    """
    from . import device as D

    configs = list(configs)
    if not configs:
        return []
    c0 = configs[0]
    for c in configs[1:]:
        if (c.variant, c.tau, c.l_max, c.cgls.i_max, c.cgls.tau, c.warm_start) != \
                (c0.variant, c0.tau, c0.l_max, c0.cgls.i_max, c0.cgls.tau, c0.warm_start):
            raise ValidationError("batched configs may differ in lam / beta only")
    op = _device_forward(op)
    fw = op.forward_struct()
    if fw.kind != _lib.KB_FWD_KRON:
        return [sb_run(op, b, c, x_true=x_true) for c in configs]
    m_rows, n_cols = op.shape
    if m_rows != n_cols:
        raise ValidationError(f"operator must be square to start from the observed image, got {op.shape}")
    n = int(round(np.sqrt(n_cols)))
    if n * n != n_cols:
        raise ValidationError(f"operator size {n_cols} is not a perfect square")
    host = not D.is_tensor(b)
    bd = D.to_device(np.asarray(b, dtype=np.float64).ravel() if host else b, np.float64).reshape(-1)
    if bd.numel() != n_cols:
        raise ValidationError(f"b must have length {n_cols}, got {bd.numel()}")
    xtd = None
    if x_true is not None:
        xtd = D.to_device(np.asarray(x_true, dtype=np.float64).ravel() if not D.is_tensor(x_true) else x_true,
                          np.float64).reshape(-1)
        if xtd.numel() != n_cols:
            raise ValidationError(f"x_true must have length {n_cols}, got {xtd.numel()}")
    B, L = len(configs), c0.l_max
    lam = np.array([float(c.lam) for c in configs])
    beta = np.array([float(c.beta) for c in configs])
    outer = np.zeros(B, dtype=np.int32)
    stop = np.zeros(B, dtype=np.int32)
    rc, re, isnr = np.zeros((B, L)), np.zeros((B, L)), np.zeros((B, L))
    it = np.zeros((B, L), dtype=np.int32)
    dp, ip = C.POINTER(C.c_double), C.POINTER(C.c_int)
    st = _lib.KbSbBatch()
    st.nprob = B
    st.lam_host, st.beta_host = lam.ctypes.data_as(dp), beta.ctypes.data_as(dp)
    st.variant = _lib.KB_SB_ISOTROPIC if c0.variant == VARIANT_ISOTROPIC else _lib.KB_SB_ANISOTROPIC
    st.tau, st.l_max = float(c0.tau), L
    st.i_max, st.tau_cgls = c0.cgls.i_max, float(c0.cgls.tau)
    st.warm_start = 1 if c0.warm_start else 0
    st.outer_iters_host, st.stop_host = outer.ctypes.data_as(ip), stop.ctypes.data_as(ip)
    st.rc_host, st.re_host, st.isnr_host = rc.ctypes.data_as(dp), re.ctypes.data_as(dp), isnr.ctypes.data_as(dp)
    st.cgls_iters_host = it.ctypes.data_as(ip)
    x = D.empty((B, n_cols), np.float64)
    lib = _lib.load()
    nb = C.c_size_t()
    _lib.check(lib.kb_sb_batch_workspace_bytes(C.byref(fw), B, C.byref(nb)))
    ws, wsb = D.WORKSPACE.get(nb.value)
    _lib.check(lib.kb_sb_run_batch(C.byref(fw), bd.data_ptr(), None if xtd is None else xtd.data_ptr(),
                                   x.data_ptr(), C.byref(st), ws, wsb, D.stream_ptr()), "sb_run_batch")
    xs = D.to_host(x) if host else x
    out = []
    for p in range(B):
        k = int(outer[p])
        res = SbResult(x=xs[p], outer_iters=k, stop=_lib.SB_STOPS[int(stop[p])],
                       rc_history=[float(v) for v in rc[p, :k]], cgls_iters=[int(v) for v in it[p, :k]])
        if x_true is not None:
            res.re_history = [float(v) for v in re[p, :k]]
            res.isnr_history = [float(v) for v in isnr[p, :k]]
        out.append(res)
    return out


def _batch_size(op, count: int) -> int:
    """Problems per batched launch: all of them, within ~24 GB of device workspace."""
    n_cols = op.shape[1]
    k = getattr(op, "k", 1)
    per = 8 * n_cols * (20 + 2 * k)   # stacked CGLS/SB state + Kronecker intermediate
    return max(1, min(count, int(24e9 // per)))


def sweep(op, b, gamma: float, lam_lo: float, lam_hi: float, count: int = 100, x_true=None, batch=None,
          **config_kwargs):
    """lambda sweep at fixed gamma (splitbregman.py:195-235).

    The grid points are independent SB problems sharing the factors; they run
    in lock step through :func:`sb_run_batch` (``batch`` problems per launch,
    default: as many as fit), so every Kronecker product is one batched GEMM
    pair over the whole grid instead of ``count`` small ones.
    """
    grid = lambda_grid(lam_lo, lam_hi, count)
    configs = [SbConfig.from_gamma(float(lam), gamma, **config_kwargs) for lam in grid]
    dop = _device_forward(op)
    step = int(batch) if batch else _batch_size(dop, len(configs))
    results = []
    for i in range(0, len(configs), step):
        results += sb_run_batch(dop, b, configs[i:i + step], x_true=x_true)
    records = []
    for config, res in zip(configs, results):
        records.append({
            "lam": float(config.lam), "beta": config.beta,
            "re": res.re_history[-1] if res.re_history else float("nan"),
            "isnr_db": res.isnr_history[-1] if res.isnr_history else float("nan"),
            "outer_iters": res.outer_iters, "iota_total": res.iota_total,
            "rc_final": res.rc_history[-1] if res.rc_history else float("nan"),
        })
    return records
