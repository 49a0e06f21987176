"""Randomised check of the tiled R(A) block product against the CPU oracle: 60 cases over
n in {128, 256, 384}, random odd PSF supports up to (2n-1)^2, fp32 / fp64, 1-16 vectors."""
import sys, numpy as np
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2410_00233_b200 as kb
from paper_2410_00233_b200 import device as D
from paper_2410_00233_b200.lowrank import _EngineOp
from oracle import structured as ost
rng = np.random.default_rng(2024)
bad = 0
for case in range(60):
    n = int(rng.choice([128, 256, 384]))
    kh = int(rng.integers(0, n)) * 2 + 1
    kw = int(rng.integers(0, n)) * 2 + 1
    kh, kw = min(kh, 2 * n - 1), min(kw, 2 * n - 1)
    dtype = np.float32 if rng.random() < 0.6 else np.float64
    nv = int(rng.choice([1, 2, 3, 4, 5, 8, 9, 13, 16]))
    psf = rng.random((kh, kw)) + 0.05
    blur = kb.RearrangedBlur(psf, n, dtype=dtype)
    kern = blur.psf.kernel.astype(dtype)
    op = _EngineOp(blur)
    x = rng.standard_normal((nv, n * n)).astype(dtype)
    xd = D.to_device(x)
    y, z = D.to_host(op.apply_block(xd, 0)), D.to_host(op.apply_block(xd, 1))
    tol = 4e-7 if dtype == np.float32 else 1e-13
    for j in {0, nv - 1}:
        wy = ost.ra_matvec(kern, n, x[j]).astype(np.float64); wz = ost.ra_rmatvec(kern, n, x[j]).astype(np.float64)
        ey = np.linalg.norm(y[j] - wy) / max(np.linalg.norm(wy), 1e-300); ez = np.linalg.norm(z[j] - wz) / max(np.linalg.norm(wz), 1e-300)
        if not (ey < tol and ez < tol):
            bad += 1
            print("FAIL", case, n, (kh, kw), dtype.__name__, nv, j, ey, ez)
print("cases done, failures:", bad)
