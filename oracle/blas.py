"""OpenBLAS x86-64 ``sdot`` restated in numpy (CPU oracle, TEST INFRASTRUCTURE ONLY).

The reference computes every fp32 dot product and norm of its eGKB recurrence
with numpy (``b @ v`` in ``_mgs_against``, ``np.linalg.norm`` = sqrt(x.dot(x));
``lowrank.py:153-156, 207-259``), i.e. with OpenBLAS's ``sdot`` (numpy's
bundled ``scipy_openblas`` 0.3.30, a DYNAMIC_ARCH build).  Its x86-64 kernel
(``kernel/x86_64/sdot.c``) runs one of two micro-kernels over the first
``n & -32`` elements and a scalar loop over the rest:

* SkylakeX / Cooperlake / SapphireRapids cores: four 512-bit fp32 FMA
  accumulators over blocks of 64 (lane l sums elements 64k+l in order), each
  folded to 256 bits (low half + high half), then a 256-bit loop for the
  remaining block of 32, then ((a0+a1)+a2)+a3, 128-bit halves added, and two
  horizontal adds;
* Haswell / Zen cores: four 256-bit accumulators over blocks of 32 (lane l
  sums 32k+l), each folded to 128 bits, then (f0+f1)+(f2+f3) and two
  horizontal adds.

The scalar tail adds the fp32 products ``x[i]*y[i]`` in double and returns the
sum rounded to float.  sdot is single-threaded at every length.  These
restatements are pinned bit-for-bit against numpy's own ``x @ y`` on the host
(``tests/test_oracle_blas.py``; the other kernel through ``OPENBLAS_CORETYPE``)
and are the checker for the device emulation (``kb_sdot_openblas``) and for
the reference-arithmetic eGKB engine on a kernel the host does not run.
"""

from __future__ import annotations

import numpy as np

KERNELS = {"openblas-skx": 64, "openblas-hsw": 32}


def _lanes(x: np.ndarray, y: np.ndarray, lanes: int) -> np.ndarray:
    """Per-lane fp32 FMA chains: lane l accumulates x[lanes*k+l]*y[lanes*k+l] in k order."""
    X = x.reshape(-1, lanes).astype(np.float64)
    Y = y.reshape(-1, lanes).astype(np.float64)
    acc = np.zeros(lanes, dtype=np.float32)
    for r in range(X.shape[0]):
        # fp32 FMA: the exact product (48 bits, exact in fp64) added, one rounding to fp32
        acc = (acc.astype(np.float64) + X[r] * Y[r]).astype(np.float32)
    return acc


def sdot(x, y, kernel: str = "openblas-skx") -> np.float32:
    """``x @ y`` for float32 vectors as OpenBLAS's ``kernel`` computes it."""
    x = np.ascontiguousarray(x, dtype=np.float32).ravel()
    y = np.ascontiguousarray(y, dtype=np.float32).ravel()
    n = x.size
    n1 = n & ~31
    f32 = np.float32
    if kernel == "openblas-skx":
        n64 = n1 & ~63
        acc = _lanes(x[:n64], y[:n64], 64) if n64 else np.zeros(64, np.float32)
        q = [(acc[16 * k:16 * k + 8] + acc[16 * k + 8:16 * k + 16]).astype(np.float32) for k in range(4)]
        if n1 > n64:   # the one remaining block of 32: one FMA into each 256-bit lane
            for k in range(4):
                xs = x[n64 + 8 * k:n64 + 8 * k + 8].astype(np.float64)
                ys = y[n64 + 8 * k:n64 + 8 * k + 8].astype(np.float64)
                q[k] = (q[k].astype(np.float64) + xs * ys).astype(np.float32)
        s = ((q[0] + q[1]) + q[2]) + q[3]
        h = (s[:4] + s[4:]).astype(np.float32)
        r = f32(f32(h[0] + h[1]) + f32(h[2] + h[3]))
    elif kernel == "openblas-hsw":
        acc = _lanes(x[:n1], y[:n1], 32) if n1 else np.zeros(32, np.float32)
        f = [(acc[8 * k:8 * k + 4] + acc[8 * k + 4:8 * k + 8]).astype(np.float32) for k in range(4)]
        t = ((f[0] + f[1]) + (f[2] + f[3])).astype(np.float32)
        r = f32(f32(t[0] + t[1]) + f32(t[2] + t[3]))
    else:
        raise ValueError(f"unknown kernel {kernel!r}")
    d = np.float64(r)
    for i in range(n1, n):   # scalar tail: fp32 products, double accumulator
        d = d + np.float64(f32(x[i] * y[i]))
    return f32(d)


def norm(x, kernel: str = "openblas-skx") -> float:
    """``float(np.linalg.norm(x))`` for a float32 vector on ``kernel``."""
    return float(np.sqrt(sdot(x, x, kernel)))
