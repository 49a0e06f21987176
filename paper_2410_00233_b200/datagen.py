"""Seeded synthetic inputs for the five BASELINE.json configurations.

The reference ships no data for n >= 128 and the paper's IR-Tools PSFs and
images are not available, so these generators stand in for them:
same shapes, sizes and value distributions as BASELINE.json describes, fixed
seeds (image 1, PSF 2, noise 3, Krylov/sketch 0).  Everything is
generated on the host in numpy; GPU and CPU arms consume identical arrays.

Conventions follow the reference: images are n-by-n, vectorised column-major
(``linalg.py:76-91``); the PSF is zero-padded from n-by-n to (n+1)-by-(n+1) so
its support is odd and ``Psf.center == (n/2, n/2)`` (``blurmodel.py:40-51``,
SURVEY §7 hard part 4); noise follows ``add_noise`` (``blurmodel.py:204-218``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEED_IMAGE = 1
SEED_PSF = 2
SEED_NOISE = 3
SEED_KRYLOV = 0

LAM = 0.1150    # test_acceptance.py:236
BETA = 0.0066


def cartoon_image(n: int, seed: int = SEED_IMAGE) -> np.ndarray:
    """Sum of 12 axis-aligned rectangles then 6 disks, intensities U[0,1],
    clipped to [0,1] (BASELINE.json configs[0])."""
    rng = np.random.default_rng(seed)
    img = np.zeros((n, n))
    lo, hi = math.ceil(n / 32), math.ceil(n / 3)
    for _ in range(12):
        r0, c0 = rng.integers(0, n, size=2)
        h, w = rng.integers(lo, hi + 1, size=2)
        img[r0 : r0 + h, c0 : c0 + w] += rng.uniform(0.0, 1.0)
    rr, cc = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
    for _ in range(6):
        cr, ccen = rng.uniform(0.0, n, size=2)
        rad = rng.uniform(n / 32, n / 6)
        val = rng.uniform(0.0, 1.0)
        img[(rr - cr) ** 2 + (cc - ccen) ** 2 <= rad ** 2] += val
    return np.clip(img, 0.0, 1.0)


def _gauss(n: int, sig_a: float, sig_b: float, theta: float) -> np.ndarray:
    c = n // 2
    rr, cc = np.meshgrid(np.arange(n) - c, np.arange(n) - c, indexing="ij")
    a = rr * math.cos(theta) + cc * math.sin(theta)
    b = -rr * math.sin(theta) + cc * math.cos(theta)
    g = np.exp(-0.5 * ((a / sig_a) ** 2 + (b / sig_b) ** 2))
    return g / g.sum()


def pad_odd(kernel: np.ndarray) -> np.ndarray:
    """Append one zero row / column to an even-sized PSF (centre stays n/2)."""
    kh, kw = kernel.shape
    out = np.zeros((kh + (kh % 2 == 0), kw + (kw % 2 == 0)))
    out[:kh, :kw] = kernel
    return out / out.sum()


def rotated_gaussian_psf(n: int) -> np.ndarray:
    """configs[0]: sigma 3.5 along the 30 deg axis, 2 across, centred."""
    return pad_odd(_gauss(n, 3.5, 2.0, math.radians(30.0)))


def mixture_psf(n: int, sig_hi: float = 6.0, seed: int = SEED_PSF) -> np.ndarray:
    """configs[1..4]: 3 rotated anisotropic Gaussians, sigma in [1, sig_hi],
    angle U[0, pi), weight U[0.2, 1], each normalised, then normalised."""
    rng = np.random.default_rng(seed)
    acc = np.zeros((n, n))
    for _ in range(3):
        sa, sb = rng.uniform(1.0, sig_hi, size=2)
        th = rng.uniform(0.0, math.pi)
        wt = rng.uniform(0.2, 1.0)
        acc += wt * _gauss(n, sa, sb, th)
    return pad_odd(acc / acc.sum())


def blur(image: np.ndarray, psf: np.ndarray) -> np.ndarray:
    """Zero-BC convolution, 'same' size: equals build_blur_matrix(psf) @ vec(x)
    for an odd PSF (blurmodel.py:87-121; SURVEY probe p10)."""
    from scipy.signal import fftconvolve

    return fftconvolve(image, psf, mode="same")


def add_noise(b_true: np.ndarray, level: float, seed: int = SEED_NOISE) -> np.ndarray:
    """b + eta with ||eta|| = level * ||b|| (blurmodel.py:204-218)."""
    b_true = np.asarray(b_true, dtype=np.float64)
    if level == 0.0:
        return b_true.copy()
    zeta = np.random.default_rng(seed).standard_normal(b_true.shape)
    return b_true + level * (np.linalg.norm(b_true.ravel()) / np.linalg.norm(zeta.ravel())) * zeta


@dataclass
class Problem:
    """One configuration's inputs (all host arrays)."""

    name: str
    n: int
    psf: np.ndarray          # (n+1, n+1), unit sum
    x_true: np.ndarray       # length n^2, column-major vec
    b: np.ndarray            # noisy observation, column-major vec
    noise: float
    egkb: dict = field(default_factory=dict)
    sb: dict = field(default_factory=dict)


# configs[i] of BASELINE.json made concrete
CONFIGS = {
    "n64": dict(n=64, psf="rotated", noise=0.01,
                egkb=dict(k_max=10, k_min=10, p=2, tau=1e300),
                sb=dict(variant="anisotropic", tau=0.0, l_max=100)),
    "n256": dict(n=256, psf="mixture", sig_hi=6.0, noise=0.001,
                 egkb=dict(k_max=20),
                 sb=dict(variant="isotropic", tau=0.0, l_max=200)),
    "n512": dict(n=512, psf="mixture", sig_hi=6.0, noise=0.001,
                 egkb=dict(k_max=20, k_min=20, p=2, tau=1e300),
                 sb=dict(variant="both", tau=1e-3, l_max=50)),
    "n1024": dict(n=1024, psf="mixture", sig_hi=6.0, noise=0.01,
                  egkb=dict(k_max=30, k_min=30, p=2, tau=1e300),
                  sb=dict(variant="isotropic", tau=0.0, l_max=200)),
    "n2048": dict(n=2048, psf="mixture", sig_hi=12.0, noise=0.001,
                  egkb=dict(k_max=50),
                  sb=dict(variant="anisotropic", tau=0.0, l_max=300)),
}


def make_problem(name: str, n: int | None = None) -> Problem:
    """Build a configuration's inputs; ``n`` overrides the side (tests)."""
    spec = dict(CONFIGS[name])
    side = spec["n"] if n is None else n
    if spec["psf"] == "rotated":
        psf = rotated_gaussian_psf(side)
    else:
        psf = mixture_psf(side, spec.get("sig_hi", 6.0))
    img = cartoon_image(side)
    b_true = blur(img, psf)
    b = add_noise(b_true.reshape(-1, order="F"), spec["noise"])
    return Problem(name=name, n=side, psf=psf, x_true=img.reshape(-1, order="F"),
                   b=b, noise=spec["noise"], egkb=dict(spec["egkb"]), sb=dict(spec["sb"]))
