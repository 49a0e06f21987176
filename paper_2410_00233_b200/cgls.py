"""CGLS on the GPU (reference: cgls.py:25-116).

The whole iteration runs in libkronblur_b200 (``kb_cgls_run``): operator
products (DMMA GEMMs or dense GEMV), fused vector passes with on-device
scalars, and one host read-back per iteration for the stop tests.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .exceptions import ValidationError
from .metrics import FlopCounter
from .operators import as_operator

CGLS_CONVERGED = "converged"
CGLS_MAX_ITER = "max_iter"
CGLS_STALLED = "stalled"


@dataclass
class CglsConfig:
    i_max: int = 100
    tau: float = 1e-4

    def __post_init__(self):
        if self.i_max < 1:
            raise ValidationError("i_max must be >= 1")
        if self.tau < 0:
            raise ValidationError("tau must be >= 0")


@dataclass
class CglsResult:
    x: np.ndarray
    iters: int
    stop: str
    rc_history: list = field(default_factory=list)
    resnorms: list = field(default_factory=list)

    @property
    def converged(self) -> bool:
        return self.stop == CGLS_CONVERGED


def _device_forward(op):
    op = as_operator(op)
    if not hasattr(op, "forward_struct"):
        raise ValidationError(
            f"{type(op).__name__} has no device form; pass a dense matrix, a KroneckerSum or an AugmentedOp")
    return op


def cgls_solve(op, b, config: CglsConfig | None = None, x0=None, counter: FlopCounter | None = None):
    """Run CGLS on ``op x = b`` (cgls.py:50-116)."""
    from . import device as D

    op = _device_forward(op)
    if config is None:
        config = CglsConfig()
    m, n = op.shape
    host = not D.is_tensor(b)
    bd = D.to_device(np.asarray(b, dtype=np.float64).ravel() if host else b, np.float64).reshape(-1)
    if bd.numel() != m:
        raise ValidationError(f"b must have length {m}, got {bd.numel()}")
    x0d = None
    if x0 is not None:
        x0d = D.to_device(np.asarray(x0, dtype=np.float64).ravel() if not D.is_tensor(x0) else x0,
                          np.float64).reshape(-1)
        if x0d.numel() != n:
            raise ValidationError(f"x0 must have length {n}, got {x0d.numel()}")
    x = D.empty(n, np.float64)
    fw = op.forward_struct()
    rc = np.zeros(config.i_max + 1)
    res = np.zeros(config.i_max + 2)
    dp = C.POINTER(C.c_double)
    st = _lib.KbCglsState()
    st.i_max, st.tau = config.i_max, float(config.tau)
    st.rc_host, st.resnorm_host = rc.ctypes.data_as(dp), res.ctypes.data_as(dp)
    lib = _lib.load()
    nb = C.c_size_t()
    _lib.check(lib.kb_cgls_workspace_bytes(C.byref(fw), C.byref(nb)))
    ws, wsb = D.WORKSPACE.get(nb.value)
    _lib.check(lib.kb_cgls_run(C.byref(fw), bd.data_ptr(), None if x0d is None else x0d.data_ptr(),
                               x.data_ptr(), C.byref(st), ws, wsb, D.stream_ptr()), "cgls")
    stop = _lib.CGLS_STOPS[st.stop]
    if counter is not None:
        forwards = st.iters + (1 if stop == CGLS_STALLED else 0) + (1 if x0 is not None else 0)
        for _ in range(forwards):
            _count(op, counter, 0)
        for _ in range(st.iters + 1):
            _count(op, counter, 1)
    return CglsResult(x=D.to_host(x) if host else x, iters=st.iters, stop=stop,
                      rc_history=[float(v) for v in rc[: st.n_rc]],
                      resnorms=[float(v) for v in res[: st.n_res]])


def _count(op, counter, transpose):
    if hasattr(op, "_count"):
        op._count(counter, transpose)
    elif hasattr(op, "scheme"):
        s = op.scheme
        (counter.add_kp_transpose if transpose else counter.add_kp)(s.m1, s.m2, s.n1, s.n2, op.k)
