"""The C-ABI library builds for sm_100a, loads without a GPU and exports every
symbol include/kronblur_b200.h declares (no compute calls here)."""

import ctypes
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "kronblur_b200.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(kb_\w+)\s*\(", text, re.M)))


@pytest.fixture(scope="module")
def lib():
    from paper_2410_00233_b200 import _lib
    from paper_2410_00233_b200.build import build

    build()
    return _lib.load()


def test_header_declares_the_boundary():
    syms = declared_symbols()
    for must in ("kb_egkb_run", "kb_op_apply", "kb_kron_apply", "kb_sb_run", "kb_cgls_run", "kb_ts_lift",
                 "kb_orthonormalize", "kb_dgemm", "kb_toeplitz_lift"):
        assert must in syms


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name


def test_python_binding_covers_header():
    from paper_2410_00233_b200 import _lib

    assert set(declared_symbols()) == set(_lib.EXPORTED)


def test_struct_layouts_match_header():
    """Compile a C probe of sizeof/offsetof for the ABI structs and compare with ctypes."""
    from paper_2410_00233_b200 import _lib

    probe = r'''
#include <stdio.h>
#include <stddef.h>
#include "kronblur_b200.h"
#define P(T) printf(#T " %zu\n", sizeof(T));
int main(void){ P(kb_operator) P(kb_egkb_config) P(kb_egkb_state) P(kb_kron) P(kb_forward)
 P(kb_cgls_state) P(kb_sb_state)
 printf("kb_forward.lam_y %zu\n", offsetof(kb_forward, lam_y));
 printf("kb_sb_state.cgls_iters_host %zu\n", offsetof(kb_sb_state, cgls_iters_host));
 return 0; }
'''
    import tempfile

    with tempfile.TemporaryDirectory() as d:
        src = os.path.join(d, "p.c")
        exe = os.path.join(d, "p")
        open(src, "w").write(probe)
        subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), src, "-o", exe], check=True)
        out = subprocess.run([exe], check=True, capture_output=True, text=True).stdout
    sizes = dict(line.rsplit(" ", 1) for line in out.strip().splitlines())
    assert int(sizes["kb_operator"]) == ctypes.sizeof(_lib.KbOperator)
    assert int(sizes["kb_egkb_config"]) == ctypes.sizeof(_lib.KbEgkbConfig)
    assert int(sizes["kb_egkb_state"]) == ctypes.sizeof(_lib.KbEgkbState)
    assert int(sizes["kb_kron"]) == ctypes.sizeof(_lib.KbKron)
    assert int(sizes["kb_forward"]) == ctypes.sizeof(_lib.KbForward)
    assert int(sizes["kb_cgls_state"]) == ctypes.sizeof(_lib.KbCglsState)
    assert int(sizes["kb_sb_state"]) == ctypes.sizeof(_lib.KbSbState)
    assert int(sizes["kb_forward.lam_y"]) == _lib.KbForward.lam_y.offset
    assert int(sizes["kb_sb_state.cgls_iters_host"]) == _lib.KbSbState.cgls_iters_host.offset


def test_sass_is_sm100a(lib):
    from paper_2410_00233_b200._lib import LIB_PATH

    out = subprocess.run(["cuobjdump", "--list-elf", LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", LIB_PATH], capture_output=True, text=True).stdout
    assert "DMMA" in sass   # FP64 tensor-pipe GEMM for the Kronecker apply


def test_no_gpu_compute_without_device():
    """Importing the package and building configs works on a CPU-only host."""
    import paper_2410_00233_b200 as kb

    cfg = kb.EgkbConfig(k_max=3)
    assert cfg.p == 2
    with pytest.raises(kb.ValidationError):
        kb.EgkbConfig(k_max=0)
    with pytest.raises(kb.ValidationError):
        kb.SbConfig(lam=-1, beta=1)


@pytest.mark.parametrize("shape", [(1, 1), (3, 5), (33, 33), (129, 257), (513, 513), (1025, 1025), (2049, 7)])
def test_psf_scan_is_numpys_sum_and_min_bitwise(lib, shape):
    """kb_psf_scan restates numpy's pairwise summation (blurmodel.py:25-65 Psf: k.sum())
    on parallel subtrees: the sum must be bit-identical to k.sum(), the min exact.
    Host-only: runs without a GPU."""
    import numpy as np

    rng = np.random.default_rng(sum(shape))
    k = np.ascontiguousarray(rng.random(shape) ** 5 * 10.0 ** rng.uniform(-30, 30))
    total, kmin = ctypes.c_double(), ctypes.c_double()
    for threads in (1, 3, 8, 16):
        own = np.full_like(k, np.nan)
        assert lib.kb_psf_scan(k.ctypes.data, k.size, threads, ctypes.byref(total), ctypes.byref(kmin),
                               own.ctypes.data if threads != 3 else None) == 0
        assert total.value == k.sum(), (shape, threads)
        assert kmin.value == k.min()
        if threads != 3:
            assert np.array_equal(own, k)      # the private copy taken in the same pass


def test_psf_validation_uses_the_exact_scan():
    """Psf (blurmodel.py:25-65) on a large kernel: the same mass and checks as the reference."""
    import numpy as np
    from paper_2410_00233_b200.blurmodel import Psf
    from paper_2410_00233_b200.exceptions import ValidationError

    rng = np.random.default_rng(7)
    k = rng.random((513, 513))
    p = Psf(k)
    assert np.array_equal(p.kernel, k / k.sum())
    bad = k.copy()
    bad[100, 200] = -1e-300
    with pytest.raises(ValidationError):
        Psf(bad)
    with pytest.raises(ValidationError):
        Psf(np.zeros((513, 513)))


@pytest.mark.parametrize("side", [7, 301])
def test_psf_is_a_private_copy(side):
    """The reference's Psf copies the kernel (blurmodel.py:25-65, np.array(kernel)): changing
    the caller's array afterwards must not change the operator, on either the small
    (numpy) or the large (kb_psf_scan) construction path."""
    import numpy as np
    from paper_2410_00233_b200.blurmodel import Psf

    rng = np.random.default_rng(side)
    k = rng.random((side, side))
    want = k / k.sum()
    p = Psf(k)
    k[:] = -1.0
    assert np.array_equal(p.kernel, want)
