"""ctypes binding of ``libkronblur_b200.so`` (the C ABI in include/kronblur_b200.h).

This is the whole boundary between the Python host package and the sm_100a
kernels: plain pointers, sizes and a cudaStream_t.  The library is loaded on
first use and its absence is an error — there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

from .exceptions import KronblurError, NumericalError, ValidationError

LIB_NAME = "libkronblur_b200.so"
LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)

KB_OK, KB_EVALIDATION, KB_ENUMERICAL, KB_ERUNTIME = 0, 2, 3, 4
KB_F32, KB_F64 = 0, 1
KB_OP_DENSE, KB_OP_RA_ZERO, KB_OP_RA_REFLEXIVE, KB_OP_SPARSE = 0, 1, 2, 3
KB_STOP = {1: "nu_rose", 2: "nu_below_tol", 3: "hit_kmax", 4: "breakdown"}
KB_FWD_DENSE, KB_FWD_KRON = 0, 1
KB_ARITH_FAST, KB_ARITH_OPENBLAS_SKX, KB_ARITH_OPENBLAS_HSW = 0, 1, 2
KB_SB_ANISOTROPIC, KB_SB_ISOTROPIC = 0, 1
CGLS_STOPS = {0: "max_iter", 1: "converged", 2: "stalled"}
SB_STOPS = {0: "max_iter", 1: "converged"}

vp = C.c_void_p
i64 = C.c_int64
dp = C.POINTER(C.c_double)
ip = C.POINTER(C.c_int)


class KbOperator(C.Structure):
    _fields_ = [("kind", C.c_int), ("dtype", C.c_int), ("rows", i64), ("cols", i64),
                ("a", vp), ("lda", i64), ("k", vp), ("kt", vp),
                ("kh", C.c_int), ("kw", C.c_int), ("side", C.c_int),
                ("sp_rowptr", vp), ("sp_col", vp), ("sp_val", vp), ("spt_rowptr", vp), ("spt_col", vp),
                ("spt_val", vp), ("nnz", i64)]


class KbEgkbConfig(C.Structure):
    _fields_ = [("k_max", C.c_int), ("p", C.c_int), ("k_min", C.c_int), ("tau", C.c_double),
                ("break_tol", C.c_double), ("full_reorth", C.c_int), ("reorth_passes", C.c_int),
                ("arith", C.c_int)]


class KbEgkbState(C.Structure):
    _fields_ = [("s_basis", vp), ("ld_s", i64), ("q_basis", vp), ("ld_q", i64), ("capacity", C.c_int),
                ("alphas_host", dp), ("ts_host", dp), ("zetas_host", dp), ("nus_host", dp),
                ("s_scale_host", dp), ("q_scale_host", dp),
                ("n_alphas", C.c_int), ("n_ts", C.c_int), ("n_nus", C.c_int),
                ("chosen_k", C.c_int), ("k_p", C.c_int), ("rows", C.c_int),
                ("stop_reason", C.c_int), ("breakdown", C.c_int),
                ("wu_dev", vp), ("wv_dev", vp), ("sigma_dev", dp), ("sigma_host", dp)]


class KbKron(C.Structure):
    _fields_ = [("m1", C.c_int), ("m2", C.c_int), ("n1", C.c_int), ("n2", C.c_int), ("k", C.c_int),
                ("f", vp), ("g", vp), ("band", vp), ("ft", vp), ("ndense", C.c_int), ("fband", vp)]


ALLREDUCE_FN = C.CFUNCTYPE(None, vp, dp, i64, vp)


class KbForward(C.Structure):
    _fields_ = [("kind", C.c_int), ("m", i64), ("n", i64), ("a", vp), ("lda", i64), ("kron", KbKron),
                ("augmented", C.c_int), ("side", C.c_int), ("lam_x", C.c_double), ("lam_y", C.c_double),
                ("allreduce", ALLREDUCE_FN), ("allreduce_ctx", vp)]


class KbCglsState(C.Structure):
    _fields_ = [("i_max", C.c_int), ("tau", C.c_double), ("iters", C.c_int), ("stop", C.c_int),
                ("rc_host", dp), ("resnorm_host", dp), ("n_rc", C.c_int), ("n_res", C.c_int)]


class KbSbState(C.Structure):
    _fields_ = [("lam", C.c_double), ("beta", C.c_double), ("variant", C.c_int), ("tau", C.c_double),
                ("l_max", C.c_int), ("i_max", C.c_int), ("tau_cgls", C.c_double), ("warm_start", C.c_int),
                ("outer_iters", C.c_int), ("stop", C.c_int), ("rc_host", dp), ("re_host", dp),
                ("isnr_host", dp), ("cgls_iters_host", ip)]


class KbSbBatch(C.Structure):
    _fields_ = [("nprob", C.c_int), ("lam_host", dp), ("beta_host", dp), ("variant", C.c_int), ("tau", C.c_double),
                ("l_max", C.c_int), ("i_max", C.c_int), ("tau_cgls", C.c_double), ("warm_start", C.c_int),
                ("outer_iters_host", ip), ("stop_host", ip), ("rc_host", dp), ("re_host", dp), ("isnr_host", dp),
                ("cgls_iters_host", ip)]


P = C.POINTER
SZ = C.c_size_t
_SIGS = {
    "kb_last_error": (C.c_char_p, []),
    "kb_version": (C.c_int, []),
    "kb_prof_enable": (None, [C.c_int]),
    "kb_prof_query": (C.c_int, [C.c_int, dp, C.POINTER(C.c_longlong), dp, dp]),
    "kb_op_workspace_bytes": (C.c_int, [P(KbOperator), P(SZ)]),
    "kb_op_apply": (C.c_int, [P(KbOperator), vp, vp, C.c_int, vp, SZ, vp]),
    "kb_op_apply_block": (C.c_int, [P(KbOperator), vp, i64, vp, i64, C.c_int, C.c_int, vp, SZ, vp]),
    "kb_ts_dots": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, i64, vp, vp, SZ, vp]),
    "kb_ts_axpy": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, vp, i64, vp]),
    "kb_ts_lift": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, C.c_int, vp, i64, i64, vp]),
    "kb_lift_assemble": (C.c_int, [C.c_int, vp, i64, C.c_int, vp, C.c_int, vp, vp, i64, i64, vp]),
    "kb_orthonormalize": (C.c_int, [C.c_int, vp, i64, C.c_int, i64, C.c_double, ip, vp, SZ, vp]),
    "kb_orth_workspace_bytes": (C.c_int, [i64, C.c_int, P(SZ)]),
    "kb_egkb_capacity": (C.c_int, [P(KbEgkbConfig)]),
    "kb_egkb_run": (C.c_int, [P(KbOperator), P(KbEgkbConfig), vp, P(KbEgkbState), vp, SZ, vp]),
    "kb_sdot_openblas": (C.c_int, [C.c_int, vp, vp, i64, vp, vp, SZ, vp]),
    "kb_nccl_allreduce_f64": (None, [vp, dp, i64, vp]),
    "kb_nccl_available": (C.c_int, []),
    "kb_nccl_last_error": (C.c_int, [C.c_int]),
    "kb_shard_diag": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp]),
    "kb_shard_z": (C.c_int, [vp, C.c_int, C.c_int, vp, vp, vp]),
    "kb_shard_bcast_dots": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp, vp, i64, C.c_int, C.c_int, C.c_int,
                                      vp, vp, vp]),
    "kb_shard_update": (C.c_int, [vp, vp, i64, C.c_int, vp, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
    "kb_shard_normalize": (C.c_int, [vp, vp, vp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp]),
    "kb_shard_sqnorm": (C.c_int, [vp, C.c_int, C.c_int, C.c_int, vp, vp]),
    "kb_shard_limbs_value": (C.c_double, [vp]),
    "kb_egkb_workspace_bytes": (C.c_int, [P(KbOperator), C.c_int, P(SZ)]),
    "kb_transpose": (C.c_int, [C.c_int, vp, i64, i64, vp, vp]),
    "kb_div_cast": (C.c_int, [vp, C.c_double, C.c_int, vp, i64, vp]),
    "kb_psf_scan": (C.c_int, [vp, i64, C.c_int, dp, dp, vp]),
    "kb_stage_upload": (C.c_int, [vp, C.c_size_t, vp, C.c_int, vp]),
    "kb_psf_commit_f32": (C.c_int, [vp, C.c_size_t, C.c_double, vp, C.c_int, vp]),
    "kb_normal_pcg64": (C.c_int, [P(C.c_uint64), P(C.c_uint64), i64, C.c_int, i64, vp, vp, SZ, vp]),
    "kb_normal_workspace_bytes": (C.c_int, [i64, P(SZ)]),
    "kb_normal_test_entries": (None, [C.c_int]),
    "kb_toeplitz_lift": (C.c_int, [C.c_int, vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, i64, vp]),
    "kb_kron_workspace_bytes": (C.c_int, [P(KbKron), P(SZ)]),
    "kb_kron_apply": (C.c_int, [P(KbKron), vp, vp, C.c_int, vp, SZ, vp]),
    "kb_kron_band": (C.c_int, [P(KbKron), vp, vp]),
    "kb_kron_assemble": (C.c_int, [C.c_int, vp, i64, vp, i64, dp, C.c_int, i64, i64, vp, vp, vp]),
    "kb_dgemm": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, i64, i64, i64, vp, i64, i64,
                           i64, vp, i64, i64, C.c_int, C.c_int, C.c_double, vp]),
    "kb_forward_workspace_bytes": (C.c_int, [P(KbForward), P(SZ)]),
    "kb_forward_apply": (C.c_int, [P(KbForward), vp, vp, C.c_int, vp, SZ, vp]),
    "kb_cgls_workspace_bytes": (C.c_int, [P(KbForward), P(SZ)]),
    "kb_cgls_run": (C.c_int, [P(KbForward), vp, vp, vp, P(KbCglsState), vp, SZ, vp]),
    "kb_sb_workspace_bytes": (C.c_int, [P(KbForward), P(SZ)]),
    "kb_sb_run": (C.c_int, [P(KbForward), vp, vp, vp, P(KbSbState), vp, SZ, vp]),
    "kb_sb_batch_workspace_bytes": (C.c_int, [P(KbForward), C.c_int, P(SZ)]),
    "kb_sb_run_batch": (C.c_int, [P(KbForward), vp, vp, vp, P(KbSbBatch), vp, SZ, vp]),
    "kb_sb_batch_exact": (None, [C.c_int]),
    "kb_diff": (C.c_int, [vp, vp, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, vp]),
    "kb_shrink_update": (C.c_int, [vp, vp, vp, vp, i64, C.c_double, C.c_int, vp]),
}
EXPORTED = tuple(_SIGS)

_lock = threading.Lock()
_lib = None


def load(path: str = LIB_PATH):
    """Load the shared library (no CUDA call is made by loading)."""
    global _lib
    if _lib is not None:   # fast path (every launch goes through here)
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(path):
                raise KronblurError(
                    f"{LIB_NAME} is not built ({path} missing); run `python -c "
                    "'import __graft_entry__ as g; g.build()'` — there is no CPU fallback"
                )
            lib = C.CDLL(path)
            for name, (res, args) in _SIGS.items():
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def check(status: int, what: str = "") -> None:
    """Map a C status code to the reference's exception types."""
    if status == KB_OK:
        return
    msg = load().kb_last_error().decode(errors="replace")
    if what:
        msg = f"{what}: {msg}"
    if status == KB_EVALIDATION:
        raise ValidationError(msg)
    if status == KB_ENUMERICAL:
        raise NumericalError(msg)
    raise KronblurError(msg)


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args), name)
