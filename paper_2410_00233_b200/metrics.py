"""Quality metrics and flop accounting (reference: metrics.py:14-94).

The per-iteration norms inside ``sb_run`` are computed on the device by the
fused SB update pass; these host functions serve user calls on host arrays.
"""

from __future__ import annotations

import math

import numpy as np

from .exceptions import ValidationError


def snr_db(b_true, b) -> float:
    b_true = np.ravel(np.asarray(b_true, dtype=np.float64))
    b = np.ravel(np.asarray(b, dtype=np.float64))
    if b.size != b_true.size:
        raise ValidationError(f"b must have length {b_true.size}, got {b.size}")
    noise = np.linalg.norm(b_true - b)
    if noise == 0.0:
        return math.inf
    return float(10.0 * np.log10((np.linalg.norm(b_true) / noise) ** 2))


def relative_error(x, x_true) -> float:
    x, x_true = np.ravel(x), np.ravel(x_true)
    denom = np.linalg.norm(x_true)
    if denom == 0.0:
        raise ValidationError("relative_error is undefined for a zero reference")
    return float(np.linalg.norm(x - x_true) / denom)


def isnr_db(x, b, x_true) -> float:
    x, b, x_true = np.ravel(x), np.ravel(b), np.ravel(x_true)
    err = np.linalg.norm(x - x_true)
    obs = np.linalg.norm(b - x_true)
    if err == 0.0 and obs == 0.0:
        return 0.0
    if err == 0.0:
        return math.inf
    if obs == 0.0:
        return -math.inf
    return float(20.0 * np.log10(obs / err))


def relative_change(x_new, x_old) -> float:
    denom = np.linalg.norm(np.ravel(x_old))
    if denom == 0.0:
        raise ValidationError("relative_change is undefined for a zero previous iterate")
    return float(np.linalg.norm(np.ravel(x_new) - np.ravel(x_old)) / denom)


class FlopCounter:
    """Multiply-add tallies, 2*m*n*p per product (metrics.py:60-94)."""

    def __init__(self):
        self.kp_apply = 0
        self.dense_apply = 0

    def add_kp(self, m1, m2, n1, n2, k):
        self.kp_apply += 2 * (m2 * (n1 * n2) + (m1 * m2) * n1) * k

    def add_kp_transpose(self, m1, m2, n1, n2, k):
        self.kp_apply += 2 * (n2 * (m1 * m2) + (n1 * n2) * m1) * k

    def add_dense(self, rows, cols):
        self.dense_apply += 2 * rows * cols

    def merge(self, other):
        self.kp_apply += other.kp_apply
        self.dense_apply += other.dense_apply

    def as_dict(self):
        return {"kp_apply": int(self.kp_apply), "dense_apply": int(self.dense_apply)}

    def __repr__(self):
        return f"FlopCounter(kp_apply={self.kp_apply}, dense_apply={self.dense_apply})"


def kp_apply_flops(m1, m2, n1, n2, k) -> int:
    return 2 * (m2 * (n1 * n2) + (m1 * m2) * n1) * k
