/*
 * kronblur_b200 — C ABI of the B200 (sm_100a) hot path of arXiv 2410.00233.
 *
 * Drop-in boundary for the reference package `kronblur` (pure Python; its
 * hot path is numpy/OpenBLAS).  Every entry point below replaces one
 * reference call site, cited as pkg/src/kronblur/<file>:<line>.  The
 * Python host package `paper_2410_00233_b200` binds these with ctypes (see
 * INTEGRATION.md for the binding a kronblur maintainer would add).
 *
 * Conventions
 *  - All array arguments are DEVICE pointers owned by the caller (torch
 *    tensors on the Python side) unless the name ends in `_host`.
 *  - Every call is stream-ordered on the given cudaStream_t (pass the
 *    current torch stream) and returns an int status:
 *        KB_OK (0), KB_EVALIDATION (2), KB_ENUMERICAL (3), KB_ERUNTIME (4)
 *    matching the reference CLI exit codes (cli.py:584-595) for
 *    ValidationError / NumericalError / other failures.  kb_last_error()
 *    gives the message of the last failure on the calling thread.
 *  - Vectors are contiguous; a "basis" is `m` vectors of length `len`
 *    stored at stride `ld` (vector i at base + i*ld).
 *  - Reductions are deterministic: fixed-order tree reductions, no atomics
 *    on data (SPEC determinism).
 *  - dtype codes: KB_F32 (0), KB_F64 (1).
 */
#ifndef KRONBLUR_B200_H
#define KRONBLUR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* kb_stream_t; /* cudaStream_t */

#define KB_OK 0
#define KB_EVALIDATION 2
#define KB_ENUMERICAL 3
#define KB_ERUNTIME 4

#define KB_F32 0
#define KB_F64 1

/* Operator kinds for the low-rank engines. */
#define KB_OP_DENSE 0   /* b_mat given densely (lowrank.py:187)             */
#define KB_OP_RA_ZERO 1 /* matrix-free R(A) of a zero-BC PSF blur (new)      */
#define KB_OP_RA_REFLEXIVE 2 /* matrix-free R(A), reflexive BC (blurmodel.py:80-84,
                                122-126): Toeplitz + two Hankel index families */
#define KB_OP_SPARSE 3  /* R(A) of an unstructured sparse A (CSR of R and R^T)  */

/* eGKB stop reasons (lowrank.py:26-29) */
#define KB_STOP_NU_ROSE 1
#define KB_STOP_NU_BELOW_TOL 2
#define KB_STOP_HIT_KMAX 3
#define KB_STOP_BREAKDOWN 4

/* SB variants / stops (splitbregman.py:19-25), CGLS stops (cgls.py:15-17) */
#define KB_SB_ANISOTROPIC 0
#define KB_SB_ISOTROPIC 1
#define KB_SB_MAX_ITER 0
#define KB_SB_CONVERGED 1
#define KB_CGLS_MAX_ITER 0
#define KB_CGLS_CONVERGED 1
#define KB_CGLS_STALLED 2

const char* kb_last_error(void);
int kb_version(void);

/* Optional device timing per kernel class (CUDA events on the launching
 * stream): 0 reorth/normalise passes, 1 R(A) diagonal sums, 2 R(A)/dense
 * column sums + row dots, 3 FP64 GEMM, 4 SB/CGLS vector passes, 5 lifts,
 * 6 device Gaussian draws.
 * kb_prof_enable(1) clears the record; kb_prof_query sums a class. */
void kb_prof_enable(int on);
int kb_prof_query(int cls, double* ms, long long* launches, double* bytes, double* flops);

/* ------------------------------------------------------------------ */
/* Operators B for eGKB / RSVD                                        */
/* ------------------------------------------------------------------ */
typedef struct {
    int kind;          /* KB_OP_DENSE, KB_OP_RA_ZERO/_REFLEXIVE, KB_OP_SPARSE */
    int dtype;         /* KB_F32 / KB_F64: working precision               */
    int64_t rows;      /* mbar                                             */
    int64_t cols;      /* nbar                                             */
    const void* a;     /* DENSE: row-major rows x cols, leading dim lda    */
    int64_t lda;
    const void* k;     /* RA: PSF kernel kh x kw, row-major, dtype         */
    const void* kt;    /* RA: the same kernel transposed (kw x kh)         */
    int kh, kw;        /* RA: PSF support (odd; centre kh/2, kw/2)          */
    int side;          /* RA: image side n (rows = cols = n*n)             */
    /* SPARSE: R(A) of an unstructured sparse A as CSR of R (rows x cols)
     * and of R^T (cols x rows): row pointers (rows+1 / cols+1), int32 column
     * indices, values in dtype.  rearrange.py:67-75 applied to the nonzeros. */
    const int64_t* sp_rowptr;
    const int* sp_col;
    const void* sp_val;
    const int64_t* spt_rowptr;
    const int* spt_col;
    const void* spt_val;
    int64_t nnz;
} kb_operator;

/* Workspace for kb_op_apply / kb_egkb_run / kb_rsvd helpers. */
int kb_op_workspace_bytes(const kb_operator* op, size_t* bytes);

/* y = B x (transpose=0) or y = B^T x (transpose=1).
 * Replaces `b_mat @ q` / `b_mat.T @ s` (lowrank.py:211,238,250) and, for
 * KB_OP_RA_*, `rearrange(build_blur_matrix(psf, n, bc))` (rearrange.py:67-75,
 * blurmodel.py:87-121) without forming R(A). */
int kb_op_apply(const kb_operator* op, const void* x, void* y, int transpose,
                void* ws, size_t ws_bytes, kb_stream_t stream);

/* Block product Y = B X (or B^T X) for nv vectors (stride ldx / ldy): the
 * RSVD block products (lowrank.py:363-367).  For R(A) one cooperative kernel
 * per 16 vectors reads K once for the block. */
int kb_op_apply_block(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy,
                      int nv, int transpose, void* ws, size_t ws_bytes, kb_stream_t stream);

/* ------------------------------------------------------------------ */
/* Tall-skinny building blocks (reorthogonalisation, lift)            */
/* ------------------------------------------------------------------ */
/* out[i] = <S_i, v> for i < m, out[m] = <v, v>  (fp64 results, device). */
int kb_ts_dots(int dtype, const void* S, int64_t ld, int m, const void* v,
               int64_t len, double* out, void* ws, size_t ws_bytes, kb_stream_t stream);
/* v -= sum_i coef[i] S_i   (coef device fp64, length m). */
int kb_ts_axpy(int dtype, const void* S, int64_t ld, int m, const double* coef,
               void* v, int64_t len, kb_stream_t stream);
/* out_c = sum_{i<rows} W[i, c] S_i for c < cols; W row-major rows x cols in
 * dtype (device).  The eGKB lift U = S U_C, V = Q V_C (lowrank.py:317-318)
 * and the RSVD lift U = Y U_H (lowrank.py:369). */
int kb_ts_lift(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols,
               void* out, int64_t ld_out, int64_t len, kb_stream_t stream);
/* kb_ts_lift fused with kb_kron_assemble (kronop.py:117-119): out_c (fp64) =
 * scale[c] * (double)(sum_i W[i,c] S_i), the lift computed exactly as
 * kb_ts_lift does in dtype; scale (device, cols doubles) may be NULL (= 1).
 * Bit-identical to lift-then-assemble without materialising u / v. */
int kb_lift_assemble(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols,
                     const double* scale_dev, double* out, int64_t ld_out, int64_t len, kb_stream_t stream);
/* In-place two-pass Gram-Schmidt of ncol vectors with the drop test of
 * orthonormalize (linalg.py:156-199).  drop_tol < 0 selects the default
 * eps*sqrt(len)*max column norm.  Returns KB_ENUMERICAL and *bad_col=j
 * (RankDeficiencyError(j)) when column j collapses; *bad_col=-2 on a
 * non-finite norm. */
int kb_orthonormalize(int dtype, void* Q, int64_t ld, int ncol, int64_t len,
                      double drop_tol, int* bad_col, void* ws, size_t ws_bytes,
                      kb_stream_t stream);
int kb_orth_workspace_bytes(int64_t len, int ncol, size_t* bytes);

/* ------------------------------------------------------------------ */
/* eGKB (lowrank.py:159-329)                                           */
/* ------------------------------------------------------------------ */
typedef struct {
    int k_max, p, k_min;
    double tau;
    double break_tol;     /* < 0: sqrt(eps) of dtype (lowrank.py:194)          */
    int full_reorth;      /* 1: project s against S (lowrank.py:240-241)       */
    int reorth_passes;    /* 1: classical GS, 2: CGS2 (default)                */
    /* KB_ARITH_FAST: the fused persistent engine (fp64-accumulated sums).
     * KB_ARITH_OPENBLAS_SKX / _HSW: the reference's own fp32 operations in
     * its order -- sequential MGS (lowrank.py:153-156), norms and coefficients
     * as OpenBLAS's x86-64 sdot computes them (64 FMA lanes for the SkylakeX
     * kernel, 32 for the Haswell/Zen kernel) -- so the trace, the rank
     * decision and the bases are bit-identical to the reference run on a host
     * whose numpy uses that kernel.  fp32 only. */
    int arith;
} kb_egkb_config;

#define KB_ARITH_FAST 0
#define KB_ARITH_OPENBLAS_SKX 1
#define KB_ARITH_OPENBLAS_HSW 2

typedef struct {
    /* caller-allocated device bases: `capacity` vectors each */
    void* s_basis; int64_t ld_s;
    void* q_basis; int64_t ld_q;
    int capacity;
    /* caller-allocated host arrays of length `capacity` (trace, 1-based lists) */
    double* alphas_host; double* ts_host; double* zetas_host; double* nus_host;
    /* caller-allocated host arrays of length `capacity`: basis vector i is
     * stored scaled, the normalised vector is s_basis[i] * s_scale_host[i]
     * (the persistent kernel folds the normalisation into its consumers) */
    double* s_scale_host; double* q_scale_host;
    /* outputs */
    int n_alphas, n_ts, n_nus;
    int chosen_k, k_p, rows, stop_reason, breakdown;
    /* optional: the small SVD of C (lowrank.py:308-316) inside the call.  When
     * wu_dev != NULL the host computes it (fp64 one-sided Jacobi) right after
     * the loop and uploads, stream-ordered, W_u = U_C[:, :chosen] (rows x
     * chosen) to wu_dev and W_v = V_C[:, :chosen] (k_p x chosen) to wv_dev
     * (working dtype, row stride chosen; each block is capacity^2 elements,
     * all of which the library may write) and
     * sigma (fp64 of the working-precision values) to sigma_dev; sigma_host
     * (capacity doubles) gets the same values -- the caller's lift reads the
     * weights on the device without another host step. */
    void* wu_dev; void* wv_dev; double* sigma_dev; double* sigma_host;
} kb_egkb_state;

/* Minimum basis capacity for a config (vectors). */
int kb_egkb_capacity(const kb_egkb_config* cfg);
/* Runs the bidiagonalisation loop (lowrank.py:207-303) on the device; the
 * small SVD of C (lowrank.py:308-316) stays on the host, the lift is
 * kb_ts_lift.  y0 is a device vector of length op->rows in op->dtype. */
int kb_egkb_run(const kb_operator* op, const kb_egkb_config* cfg, const void* y0,
                kb_egkb_state* st, void* ws, size_t ws_bytes, kb_stream_t stream);
int kb_egkb_workspace_bytes(const kb_operator* op, int capacity, size_t* bytes);
/* *out_dev = sdot(x, y) as OpenBLAS's x86-64 kernel computes it (lanes = 64:
 * SkylakeX, 32: Haswell/Zen; y == NULL: sdot(x, x)), fp32, device pointers.
 * ws: >= 1024 bytes of device scratch.  The building block of KB_ARITH_OPENBLAS_*
 * (numpy's x @ y and np.linalg.norm on float32 vectors, lowrank.py:153-156, 207-259). */
int kb_sdot_openblas(int lanes, const float* x, const float* y, int64_t n, float* out_dev,
                     void* ws, size_t ws_bytes, kb_stream_t stream);

/* ------------------------------------------------------------------ */
/* Row-sharded eGKB steps (driven by parallel.sharded_egkb) */
/* ------------------------------------------------------------------ */
/* Vectors of length n^2 (index a*n + b), this shard owning image rows
 * [a0, a1) (a0 a multiple of 8).  Every cross-shard sum is accumulated as
 * three int64 limbs (weights 2^1, 2^-39, 2^-79) of per-chunk fp64 partials --
 * exact, so the callers' int64 sum-allreduce of the limb buffers gives a
 * result independent of the number of shards.  Limb buffers are added to
 * (zero them first).  lowrank.py:207-260 restated over the shards:
 *   |x|^2 of the own rows (lowrank.py:207) */
int kb_shard_sqnorm(const float* x, int n, int a0, int a1, long long* norm_limbs, kb_stream_t stream);
/* diagonal sums of x over the own rows (the input side of an R(A) product) */
int kb_shard_diag(const float* x, int n, int c, int len, int a0, int a1, long long* limbs, kb_stream_t stream);
/* z[o] = sum_i Mt[o][i] w[i] from the all-reduced diagonal limbs (Mt = K^T for R q, K for
 * R^T s; cols x rows row-major); z must hold rows + cols doubles (the decoded w is staged
 * behind z) */
int kb_shard_z(const float* Mt, int rows, int cols, const long long* w_limbs, double* z, kb_stream_t stream);
/* y = P z on the own rows, v = y - beta*prev (prev may be NULL), limbs of B_i . v (i < m),
 * |v|^2 and |y|^2 (3 (m + 2) limbs) */
int kb_shard_bcast_dots(const double* z, int n, int c, int len, const double* beta_dev, const float* prev,
                        const float* B, int64_t ld, int m, int a0, int a1, float* v, long long* limbs,
                        kb_stream_t stream);
/* v1 = v - sum_i h_i B_i (h from the all-reduced dot limbs), limbs of |v1|^2; scal[1] = |y| */
int kb_shard_update(float* v, const float* B, int64_t ld, int m, const long long* dot_limbs, int n, int a0,
                    int a1, long long* norm_limbs, double* scal, kb_stream_t stream);
/* t = |v1| (scal[0]), out = fl(v1 / t) on the own rows, and the diagonal limbs of out for the
 * next product (centre c, length len; diag_limbs may be NULL) */
int kb_shard_normalize(const float* v, const long long* norm_limbs, float* out, int n, int c, int len, int a0,
                       int a1, long long* diag_limbs, double* scal, kb_stream_t stream);
/* host decode of three limbs (the device's own formula) */
double kb_shard_limbs_value(const long long* limbs_host);

/* dst = (dtype)(src / divisor), device: the Psf normalisation k / k.sum()
 * (blurmodel.py:25-65) fused with the working-precision cast -- bitwise
 * numpy's (k / total).astype(dtype). */
int kb_div_cast(const double* src, double divisor, int dtype, void* dst, int64_t count, kb_stream_t stream);

/* Psf validation scan (blurmodel.py:25-65): *sum_out = k.sum() of the
 * C-ordered float64 kernel -- numpy's pairwise summation, bit for bit --
 * and *min_out = k.min(), using `threads` host threads.  When copy_to is not
 * NULL the n doubles are also copied there in the same pass: the private
 * copy the reference's Psf takes (np.array(kernel), "the kernel is copied").
 * Host only. */
int kb_psf_scan(const double* k, int64_t n, int threads, double* sum_out, double* min_out, double* copy_to);
/* (src / total).astype(float32) of the host PSF straight into a pinned buffer
 * and on to dst (stream-ordered): the fp32 path without a staged fp64 copy,
 * for callers that keep src unchanged until the upload is done. */
int kb_psf_commit_f32(const double* src, size_t count, double total, float* dst, int threads,
                      kb_stream_t stream);
/* bytes of host memory -> device `dst`, through a library-owned pinned
 * buffer filled by `threads` host threads, chunk-pipelined with the copies
 * (stream-ordered on `stream`; the host array may be reused on return). */
int kb_stage_upload(const void* src, size_t bytes, void* dst, int threads, kb_stream_t stream);

/* dst (cols x rows) = src (rows x cols)^T, row-major, device.  Builds the
 * PSF transpose K^T used by the R(A)^T products on the device (the host
 * uploads K once; blurmodel.py:25-65 Psf.kernel). */
int kb_transpose(int dtype, const void* src, int64_t rows, int64_t cols, void* dst, kb_stream_t stream);

/* ------------------------------------------------------------------ */
/* Gaussian draws on the device (lowrank.py:199-201, lowrank.py:361-362) */
/* ------------------------------------------------------------------ */
/* Writes the first `count` values of numpy's
 *     np.random.Generator(PCG64).standard_normal(count)
 * (PCG64 XSL-RR stream + numpy's 256-layer float64 ziggurat) for the PCG64
 * state {lo, hi} and increment {lo, hi} given on the host (numpy's
 * bit_generator.state["state"]), rounded to dtype (KB_F32 = the reference's
 * .astype(float32)).  cols > 0 writes the TRANSPOSE of the row-major
 * (count/cols, cols) draw matrix (the device layout of the RSVD test matrix,
 * lowrank.py:362).  Bit-identical to numpy for every fast-path and wedge
 * sample; tail samples (|x| > 3.654, ~3e-4) use CUDA's log1p (<= 1 ulp in
 * f64, identical after rounding to f32).  Replaces the host draws above. */
int kb_normal_pcg64(const uint64_t* pcg_state_host, const uint64_t* pcg_inc_host, int64_t count, int dtype,
                    int64_t cols, void* out, void* ws, size_t ws_bytes, kb_stream_t stream);
int kb_normal_workspace_bytes(int64_t count, size_t* bytes);
/* Test hook: speculate only `ne` (1..3) entry offsets per chunk (0 = default 4). */
void kb_normal_test_entries(int ne);

/* ------------------------------------------------------------------ */
/* Structured exact TSVD lift (new, replaces         */
/* svd_small(rearrange(A)) linalg.py:134-153 for blur operators)        */
/* ------------------------------------------------------------------ */
/* out_c[a*n+b] = coef[c*ldc + (b-a+center)] (0 outside [0,len_coef)), c<k;
 * reflexive != 0 adds the Hankel families coef[a+b+1+center] and
 * coef[a+b+center+1-2n] (reflexive BC, blurmodel.py:122-126). */
int kb_toeplitz_lift(int dtype, const void* coef, int64_t ldc, int len_coef, int center,
                     int k, int side, int reflexive, void* out, int64_t ld_out, kb_stream_t stream);

/* ------------------------------------------------------------------ */
/* Kronecker sum, fp64 (kronop.py:28-123)                               */
/* ------------------------------------------------------------------ */
typedef struct {
    int m1, m2, n1, n2, k;
    const double* f;  /* k x n1 x m1: F_i = ax_i^T = reshape(sigma_i u_i, (n1, m1)) */
    const double* g;  /* k x n2 x m2: G_i = ay_i^T = reshape(v_i, (n2, m2))         */
    const int* band;  /* optional device int[2] from kb_kron_band (NULL: dense G)    */
    const double* ft; /* optional k x m1 x n1: Ft_i = F_i^T.  With it the reduced
                       * stage of the transposed apply is one dense GEMM, like the
                       * forward one's (both then run on cuBLAS DGEMM, the faster
                       * library kernel for these dense shapes; NULL: DMMA k_dgemm). */
    /* optional structure of the F side (KroneckerSum.toeplitz_split): with fband set, only
     * the first ndense terms have dense F_i (ft then holds those ndense blocks); the others
     * share the zero band fband (device int[2], min/max of c - r over their nonzeros) and
     * the reduced stage skips the k tiles that only meet zeros.  NULL: every F_i dense. */
    int ndense;
    const int* fband;
} kb_kron;

/* band[0..1] = min/max of (c - r) over the nonzero entries G_i[r][c] of all
 * terms, stream-ordered on the device.  With it set in kb_kron, the G stage
 * of every apply skips the k tiles that only meet zeros (bit-identical
 * result for finite x; the v-side factors of a zero-BC approximation are banded Toeplitz).
 * The band must be recomputed if g changes. */
int kb_kron_band(const kb_kron* kr, int* band, kb_stream_t stream);

int kb_kron_workspace_bytes(const kb_kron* kr, size_t* bytes);
/* y = A x (transpose=0, kronop.py:58-70) or y = A^T x (kronop.py:72-84). */
int kb_kron_apply(const kb_kron* kr, const double* x, double* y, int transpose,
                  void* ws, size_t ws_bytes, kb_stream_t stream);
/* Factor assembly (kronop.py:103-123): F_i = sigma_i * u_i, G_i = v_i,
 * promoted to fp64 (u, v in dtype, vectors at stride ldu/ldv). */
int kb_kron_assemble(int dtype, const void* u, int64_t ldu, const void* v, int64_t ldv,
                     const double* sigma_host, int k, int64_t len_u, int64_t len_v,
                     double* f, double* g, kb_stream_t stream);
/* Generic fp64 GEMM used by the Kronecker apply:
 * C_z = sum_{s<nseg} op(A_{z,s}) op(B_{z,s}) (+ beta C_z), z < nbatch. */
int kb_dgemm(int trans_a, int trans_b, int m, int n, int k,
             const double* A, int64_t lda, int64_t sa_batch, int64_t sa_seg,
             const double* B, int64_t ldb, int64_t sb_batch, int64_t sb_seg,
             double* C, int64_t ldc, int64_t sc_batch, int nbatch, int nseg,
             double beta, kb_stream_t stream);

/* ------------------------------------------------------------------ */
/* Augmented system, CGLS, split Bregman (fp64)                         */
/* ------------------------------------------------------------------ */
#define KB_FWD_DENSE 0
#define KB_FWD_KRON 1
/* Sum-allreduce hook for term-sharded operators: when set, every
 * product of the forward operator is a rank-local partial sum (this rank's
 * Kronecker terms) and the hook is called on the n-vector result, stream-
 * ordered, before anything consumes it.  The host supplies it (NCCL over
 * NVLink through torch.distributed on a B200 box, gloo in CPU tests). */
typedef void (*kb_allreduce_fn)(void* ctx, double* buf, int64_t count, kb_stream_t stream);
/* A kb_allreduce_fn over NCCL: ctx is an ncclComm_t (e.g. torch's ProcessGroupNCCL
 * communicator); ncclAllReduce(sum, fp64) in place, stream-ordered.  The library
 * resolves ncclAllReduce from the already-loaded libnccl.so.2. */
void kb_nccl_allreduce_f64(void* comm, double* buf, int64_t count, kb_stream_t stream);
int kb_nccl_available(void);
/* last non-zero ncclResult_t of the hook since the previous reset (-1: NCCL not found) */
int kb_nccl_last_error(int reset);
typedef struct {
    int kind;            /* KB_FWD_DENSE / KB_FWD_KRON                       */
    int64_t m, n;        /* forward operator shape                           */
    const double* a;     /* DENSE: row-major m x n                           */
    int64_t lda;
    kb_kron kron;        /* KRON                                             */
    int augmented;       /* 1: [A; lam_x Dx; lam_y Dy] (regularizers.py:65)   */
    int side;            /* image side for the difference maps               */
    double lam_x, lam_y;
    kb_allreduce_fn allreduce;  /* NULL: the operator is complete on this rank  */
    void* allreduce_ctx;
} kb_forward;

int kb_forward_workspace_bytes(const kb_forward* fw, size_t* bytes);
int kb_forward_apply(const kb_forward* fw, const double* x, double* y, int transpose,
                     void* ws, size_t ws_bytes, kb_stream_t stream);

typedef struct {
    int i_max; double tau;
    /* outputs */
    int iters, stop;
    double* rc_host;        /* caller host array, capacity i_max               */
    double* resnorm_host;   /* caller host array, capacity i_max + 1           */
    int n_rc, n_res;
} kb_cgls_state;
int kb_cgls_workspace_bytes(const kb_forward* fw, size_t* bytes);
/* cgls.py:50-116.  x0 may be NULL (start from zero); x is the output. */
int kb_cgls_run(const kb_forward* fw, const double* b, const double* x0, double* x,
                kb_cgls_state* st, void* ws, size_t ws_bytes, kb_stream_t stream);

typedef struct {
    double lam, beta;
    int variant;         /* KB_SB_ANISOTROPIC / KB_SB_ISOTROPIC               */
    double tau;
    int l_max;
    int i_max; double tau_cgls;
    int warm_start;
    /* outputs (host arrays of capacity l_max, caller-owned) */
    int outer_iters, stop;
    double* rc_host; double* re_host; double* isnr_host; int* cgls_iters_host;
} kb_sb_state;
int kb_sb_workspace_bytes(const kb_forward* fw, size_t* bytes);
/* splitbregman.py:120-192.  fw must be the (non-augmented) square forward
 * operator; x_true may be NULL.  x (device, length n^2) receives the result. */
int kb_sb_run(const kb_forward* fw, const double* b, const double* x_true, double* x,
              kb_sb_state* st, void* ws, size_t ws_bytes, kb_stream_t stream);

/* Batched lambda sweep (splitbregman.py:195-235 `sweep`, cli.py:488-527):
 * nprob independent SB solves of the SAME observation b with the SAME
 * Kronecker operator and per-problem (lam, beta), run in lock step so every
 * Kronecker product is ONE pair of DMMA GEMMs over all problems (the images
 * are stacked along the GEMM M dimension) and every vector pass is one launch
 * over all problems.  Problems whose CGLS / SB loop has stopped are masked
 * out; each problem follows splitbregman.py:120-192 exactly as kb_sb_run. */
typedef struct {
    int nprob;
    const double* lam_host;   /* [nprob] */
    const double* beta_host;  /* [nprob] */
    int variant;              /* shared: KB_SB_*, tau, l_max, CGLS i_max / tau, warm start */
    double tau;
    int l_max;
    int i_max;
    double tau_cgls;
    int warm_start;
    int* outer_iters_host;    /* [nprob] out */
    int* stop_host;           /* [nprob] out */
    double* rc_host;          /* [nprob * l_max] out (row p = problem p) */
    double* re_host;          /* [nprob * l_max] out, if x_true */
    double* isnr_host;        /* [nprob * l_max] out, if x_true */
    int* cgls_iters_host;     /* [nprob * l_max] out */
} kb_sb_batch;
int kb_sb_batch_workspace_bytes(const kb_forward* fw, int nprob, size_t* bytes);
/* fw: plain square Kronecker forward operator (KB_FWD_KRON); x: nprob x n^2 (device). */
int kb_sb_run_batch(const kb_forward* fw, const double* b, const double* x_true, double* x,
                    kb_sb_batch* st, void* ws, size_t ws_bytes, kb_stream_t stream);
/* Test hook: split the stacked GEMMs per problem as kb_sb_run does (more
 * split-K partial traffic), making every problem bit-identical to its own run. */
void kb_sb_batch_exact(int on);

/* Elementwise pieces exposed for parity tests (splitbregman.py:32-61,
 * regularizers.py:37-62). */
int kb_diff(const double* x, double* out, int side, int axis, int transpose, double scale,
            int accumulate, kb_stream_t stream);
int kb_shrink_update(const double* cx, const double* cy, double* dx, double* dy,
                     int64_t len, double gamma, int variant, kb_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* KRONBLUR_B200_H */
