"""Kronecker-sum apply, augmented operator, CGLS and split Bregman (CPU oracle).

TEST INFRASTRUCTURE ONLY.  Same floating-point operations, in the same order,
as the reference (``pkg/src/kronblur/``):

  * Kronecker apply / apply_t      kronop.py:58-84 (column-major unvec linalg.py:76-91)
  * halved first differences       regularizers.py:37-62
  * augmented operator             regularizers.py:97-117, rhs 120-130
  * CGLS                           cgls.py:50-116
  * shrinkage / d / g updates      splitbregman.py:32-61
  * split Bregman outer loop       splitbregman.py:120-192
  * relative change / error, ISNR  metrics.py:28-57
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


def _unvec(v, rows, cols):
    return np.asarray(v).reshape((rows, cols), order="F")


def _vec(m):
    return np.asarray(m).reshape(-1, order="F")


class KronOracle:
    """sum_i kron(ax_i, ay_i) with fp64 factors (kronop.py:28-100)."""

    def __init__(self, ax, ay, m1, m2, n1, n2):
        self.ax = [np.ascontiguousarray(a, dtype=np.float64) for a in ax]
        self.ay = [np.ascontiguousarray(b, dtype=np.float64) for b in ay]
        self.m1, self.m2, self.n1, self.n2 = m1, m2, n1, n2

    @property
    def shape(self):
        return (self.m1 * self.m2, self.n1 * self.n2)

    def apply(self, x):
        xm = _unvec(np.asarray(x, dtype=np.float64), self.n2, self.n1)
        acc = np.zeros((self.m2, self.m1))
        for a, b in zip(self.ax, self.ay):
            acc += b @ xm @ a.T
        return _vec(acc)

    def apply_t(self, y):
        ym = _unvec(np.asarray(y, dtype=np.float64), self.m2, self.m1)
        acc = np.zeros((self.n2, self.n1))
        for a, b in zip(self.ax, self.ay):
            acc += b.T @ ym @ a
        return _vec(acc)

    def materialize(self):
        out = np.zeros(self.shape)
        for a, b in zip(self.ax, self.ay):
            out += np.kron(a, b)
        return out


class DenseOracle:
    def __init__(self, mat):
        self.mat = np.asarray(mat, dtype=np.float64)

    @property
    def shape(self):
        return self.mat.shape

    def apply(self, x):
        return self.mat @ x

    def apply_t(self, y):
        return self.mat.T @ y


def dx(x, n):
    xm = _unvec(x, n, n)
    return _vec(0.5 * (xm[:, :-1] - xm[:, 1:]))


def dy(x, n):
    xm = _unvec(x, n, n)
    return _vec(0.5 * (xm[:-1, :] - xm[1:, :]))


def dx_t(w, n):
    wm = _unvec(w, n, n - 1)
    out = np.zeros((n, n))
    out[:, :-1] += 0.5 * wm
    out[:, 1:] -= 0.5 * wm
    return _vec(out)


def dy_t(w, n):
    wm = _unvec(w, n - 1, n)
    out = np.zeros((n, n))
    out[:-1, :] += 0.5 * wm
    out[1:, :] -= 0.5 * wm
    return _vec(out)


class AugOracle:
    """[A; lam_x Dx; lam_y Dy] (regularizers.py:65-117)."""

    def __init__(self, fwd, n, lam_x, lam_y):
        self.fwd, self.n, self.lx, self.ly = fwd, n, float(lam_x), float(lam_y)
        self.m = fwd.shape[0]
        self.p = n * (n - 1)

    @property
    def shape(self):
        return (self.m + 2 * self.p, self.n * self.n)

    def apply(self, x):
        return np.concatenate([self.fwd.apply(x), self.lx * dx(x, self.n), self.ly * dy(x, self.n)])

    def apply_t(self, y):
        out = self.fwd.apply_t(y[: self.m])
        out = out + self.lx * dx_t(y[self.m : self.m + self.p], self.n)
        out = out + self.ly * dy_t(y[self.m + self.p :], self.n)
        return out


@dataclass
class CglsOut:
    x: np.ndarray
    iters: int
    stop: str
    rc_history: list = field(default_factory=list)
    resnorms: list = field(default_factory=list)


def cgls(op, b, i_max=100, tau=1e-4, x0=None):
    """CGLS with the relative-change stop from the 2nd iteration (cgls.py:50-116)."""
    m, n = op.shape
    if x0 is None:
        x = np.zeros(n)
        r = b.copy()
    else:
        x = np.asarray(x0, dtype=np.float64).copy()
        r = b - op.apply(x)
    f = op.apply_t(r)
    w = f.copy()
    gam = float(f @ f)
    rcs, res = [], [float(np.linalg.norm(r))]
    stop, done = "max_iter", 0
    for it in range(i_max):
        z = op.apply(w)
        zz = float(z @ z)
        if zz == 0.0:
            stop = "stalled"
            break
        mu = gam / zz
        xn = float(np.linalg.norm(x))
        step = mu * float(np.linalg.norm(w))
        x = x + mu * w
        r = r - mu * z
        f = op.apply_t(r)
        gam_next = float(f @ f)
        if not np.isfinite(gam_next):
            raise ArithmeticError("CGLS produced non-finite residual quantities")
        w = f + (gam_next / gam) * w
        gam = gam_next
        done += 1
        res.append(float(np.linalg.norm(r)))
        if it >= 1:
            rc = step / xn if xn > 0 else np.inf
            rcs.append(rc)
            if rc < tau:
                stop = "converged"
                break
    return CglsOut(x, done, stop, rcs, res)


def shrink(w, v):
    w = np.asarray(w, dtype=np.float64)
    return np.sign(w) * np.maximum(np.abs(w) - v, 0.0)


def d_aniso(cx, cy, gx_, gy_):
    return shrink(cx, 1.0 / gx_), shrink(cy, 1.0 / gy_)


def d_iso(cx, cy, gx_, gy_):
    s = np.hypot(cx, cy)
    safe = np.where(s > 0, s, 1.0)
    fx = np.where(s > 0, np.maximum(s - 1.0 / gx_, 0.0) / safe, 0.0)
    fy = np.where(s > 0, np.maximum(s - 1.0 / gy_, 0.0) / safe, 0.0)
    return cx * fx, cy * fy


def rel_change(new, old):
    return float(np.linalg.norm(np.ravel(new) - np.ravel(old)) / np.linalg.norm(np.ravel(old)))


def rel_error(x, xt):
    return float(np.linalg.norm(x - xt) / np.linalg.norm(xt))


def isnr(x, b, xt):
    err = np.linalg.norm(x - xt)
    obs = np.linalg.norm(b - xt)
    if err == 0.0 and obs == 0.0:
        return 0.0
    if err == 0.0:
        return float("inf")
    if obs == 0.0:
        return float("-inf")
    return float(20.0 * np.log10(obs / err))


@dataclass
class SbOut:
    x: np.ndarray
    outer_iters: int
    stop: str
    rc_history: list = field(default_factory=list)
    re_history: list = field(default_factory=list)
    isnr_history: list = field(default_factory=list)
    cgls_iters: list = field(default_factory=list)


def sb_run(op, b, lam, beta, variant="anisotropic", tau=1e-3, l_max=50,
           i_max=100, tau_cgls=1e-4, warm_start=False, x_true=None, max_outer=None):
    """Split Bregman outer loop (splitbregman.py:120-192).

    ``max_outer`` truncates the run after that many outer iterations (used
    only by the bounded CPU baseline; None runs the reference semantics).
    """
    n = int(round(np.sqrt(op.shape[1])))
    gamma = lam ** 2 / beta
    aug = AugOracle(op, n, lam, lam)
    p = aug.p
    x_prev = np.asarray(b, dtype=np.float64).copy()
    ddx, ddy, ggx, ggy = np.zeros(p), np.zeros(p), np.zeros(p), np.zeros(p)
    out = SbOut(x=x_prev, outer_iters=0, stop="max_iter")
    limit = l_max if max_outer is None else min(l_max, max_outer)
    for _ in range(limit):
        rhs = np.concatenate([b, lam * (ddx - ggx), lam * (ddy - ggy)])
        inner = cgls(aug, rhs, i_max, tau_cgls, x0=x_prev if warm_start else None)
        x = inner.x
        cx = dx(x, n) + ggx
        cy = dy(x, n) + ggy
        if variant == "anisotropic":
            ddx, ddy = d_aniso(cx, cy, gamma, gamma)
        else:
            ddx, ddy = d_iso(cx, cy, gamma, gamma)
        ggx, ggy = cx - ddx, cy - ddy
        out.outer_iters += 1
        out.cgls_iters.append(inner.iters)
        rc = rel_change(x, x_prev)
        out.rc_history.append(rc)
        if x_true is not None:
            out.re_history.append(rel_error(x, x_true))
            out.isnr_history.append(isnr(x, b, x_true))
        x_prev = x
        if rc < tau:
            out.stop = "converged"
            break
    out.x = x_prev
    return out
