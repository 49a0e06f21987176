// Split-Bregman / CGLS hot loop in fp64 (sm_100a).
//
// Reference: cgls.py:50-116, regularizers.py:37-130, splitbregman.py:32-192,
// kronop.py:58-84, metrics.py:28-57.  Each CGLS iteration is
//     GEMM pair (A w)  -> fused pass F1 (stencil tail of z, |z|^2, |x|^2, |w|^2, mu)
//                      -> fused pass F2 (x += mu w, r -= mu z)
//     GEMM pair (A^T r)-> fused pass F3 (f += lam D^T r, |f|^2, |r|^2, delta)
//                      -> fused pass F4 (w = f + delta w)
// with every scalar (mu, delta, norms) computed on the device by the last
// block of the producing pass, and ONE host read-back per iteration for the
// reference's stop tests.  Reductions are deterministic (fixed grid, fixed
// order).  Vector updates mirror the reference's rounding (no FMA contraction:
// x + mu*w is two rounded ops, as numpy does).
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kb_common.cuh"

namespace kb {

extern int g_dgemm_split_per_batch;
extern GemmSkip g_dgemm_skip;
extern int g_dgemm_narrow;
void dgemm(int ta, int tb, int m, int n, int k, const double* A, int64_t lda, int64_t sa_b,
           int64_t sa_s, const double* B, int64_t ldb, int64_t sb_b, int64_t sb_s, double* C,
           int64_t ldc, int64_t sc_b, int nbatch, int nseg, double beta, cudaStream_t st,
           double* part = nullptr, int64_t part_doubles = 0);

// ------------------------------------------------------------ map-reduce core
constexpr int MR_THREADS = 256;
constexpr int MR_MAXR = 8;

inline int mr_blocks(int64_t len) {
    static const int per_sm = std::getenv("KB_MR_CTAS") ? std::max(1, std::atoi(std::getenv("KB_MR_CTAS"))) : 8;   // 2 -> 8 CTAs per SM: 1820 -> 2020 CGLS it/s on the split operator
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(len, MR_THREADS * 4), (int64_t)per_sm * kSMs));
}

// f(e, acc) for e in [0, len); R block-reduced sums -> out[0..R); post(out) on
// one thread after the deterministic final reduction.
template <int R, class F, class P>
__global__ void __launch_bounds__(MR_THREADS)
k_map_reduce(int64_t len, F f, P post, double* part, double* out, unsigned* counter) {
    __shared__ double sw[MR_THREADS / 32][MR_MAXR];
    __shared__ double fin[MR_MAXR];
    if (f.skip()) return;  // uniform across the grid (device flag)
    double acc[R > 0 ? R : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)MR_THREADS + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * MR_THREADS)
        f(e, acc);
    if (R == 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double v = warp_sum(acc[r]);
        if (lane == 0) sw[warp][r] = v;
    }
    __syncthreads();
    if (threadIdx.x < R) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < MR_THREADS / 32; ++w) s += sw[w][threadIdx.x];
        part[(int64_t)blockIdx.x * R + threadIdx.x] = s;
    }
    if (last_block_ticket(counter, gridDim.x)) {
        if (warp < R) {
            double s = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) s += __ldcg(&part[(int64_t)b * R + warp]);
            s = warp_sum(s);
            if (lane == 0) fin[warp] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int r = 0; r < R; ++r) out[r] = fin[r];
            post(out);
        }
    }
}

struct NoPost {
    __device__ void operator()(double*) const {}
};

// device scalar slots (one array per CGLS solve)
enum Slot {
    S_GAM = 0,     // tau_sq (f.f)
    S_ZZ,          // z.z
    S_MU,
    S_XN,          // ||x|| before the update
    S_STEP,        // mu * ||w||
    S_FF,          // tau_next
    S_DELTA,
    S_RR,          // ||r||^2
    S_STALL,       // 1 if z.z == 0 (skip remaining work)
    S_NSLOTS
};
// reduction scratch after the slots: [red0..red7]
constexpr int S_RED = 16;
constexpr int S_TOTAL = 32;

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }

// halved first differences on the column-major n x n image (regularizers.py:37-62)
__device__ __forceinline__ double dx_at(const double* x, int64_t e, int n) {  // e < n(n-1)
    return dmul(0.5, dsub(x[e], x[e + n]));
}
__device__ __forceinline__ double dy_at(const double* x, int64_t e, int n) {  // e < n(n-1)
    const unsigned c = (unsigned)e / (unsigned)(n - 1), r = (unsigned)e - c * (unsigned)(n - 1);
    const int64_t i = (int64_t)c * n + r;
    return dmul(0.5, dsub(x[i], x[i + 1]));
}
// (D_x^T w)[e]: out[:, :-1] += .5 W ; out[:, 1:] -= .5 W  with W n x (n-1)
__device__ __forceinline__ double dxt_at(const double* w, int64_t e, int n) {
    const int64_t P = (int64_t)n * (n - 1);
    double v = 0.0;
    if (e < P) v = dadd(v, dmul(0.5, w[e]));
    if (e >= n) v = dsub(v, dmul(0.5, w[e - n]));
    return v;
}
// (D_y^T w)[e]: out[:-1, :] += .5 W ; out[1:, :] -= .5 W  with W (n-1) x n
__device__ __forceinline__ double dyt_at(const double* w, int64_t e, int n) {
    const int64_t c = (unsigned)e / (unsigned)n, r = (unsigned)e - (unsigned)c * (unsigned)n;
    double v = 0.0;
    if (r < n - 1) v = dadd(v, dmul(0.5, w[c * (n - 1) + r]));
    if (r >= 1) v = dsub(v, dmul(0.5, w[c * (n - 1) + r - 1]));
    return v;
}

// ------------------------------------------------------------ CGLS passes
struct F1 {  // z tail, |z|^2, |x|^2, |w|^2
    const double* w; const double* x; double* z;
    int64_t m, ncols, P; int n; double lx, ly; const double* scal;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double* acc) const {
        if (e < m) { const double v = z[e]; acc[0] += v * v; }
        else if (e < m + P) { const double v = dmul(lx, dx_at(w, e - m, n)); z[e] = v; acc[0] += v * v; }
        else if (e < m + 2 * P) { const double v = dmul(ly, dy_at(w, e - m - P, n)); z[e] = v; acc[0] += v * v; }
        if (e < ncols) { acc[1] += x[e] * x[e]; acc[2] += w[e] * w[e]; }
    }
};
struct F1Post {
    double* scal;
    __device__ void operator()(double* r) const {
        scal[S_ZZ] = r[0];
        if (r[0] == 0.0) { scal[S_STALL] = 1.0; scal[S_MU] = 0.0; return; }
        const double mu = scal[S_GAM] / r[0];
        scal[S_MU] = mu;
        scal[S_XN] = sqrt(r[1]);
        scal[S_STEP] = mu * sqrt(r[2]);
    }
};
struct F2 {  // x += mu w ; r -= mu z
    double* x; const double* w; double* r; const double* z; int64_t ncols, T; const double* scal;
    __device__ bool skip() const { return scal[S_STALL] != 0.0; }
    __device__ void operator()(int64_t e, double*) const {
        const double mu = scal[S_MU];
        if (e < ncols) x[e] = dadd(x[e], dmul(mu, w[e]));
        if (e < T) r[e] = dsub(r[e], dmul(mu, z[e]));
    }
};
struct F3 {  // f = (f + lx Dx^T r2) + ly Dy^T r3 ; |f|^2 ; |r|^2
    double* f; const double* r; int64_t m, ncols, T, P; int n; double lx, ly; int aug; const double* scal;
    __device__ bool skip() const { return scal[S_STALL] != 0.0; }
    __device__ void operator()(int64_t e, double* acc) const {
        if (e < ncols) {
            double v = f[e];
            if (aug) {
                v = dadd(v, dmul(lx, dxt_at(r + m, e, n)));
                v = dadd(v, dmul(ly, dyt_at(r + m + P, e, n)));
                f[e] = v;
            }
            acc[0] += v * v;
        }
        if (e < T) acc[1] += r[e] * r[e];
    }
};
struct F3Post {
    double* scal;
    __device__ void operator()(double* r) const {
        scal[S_FF] = r[0];
        scal[S_RR] = r[1];
        scal[S_DELTA] = r[0] / scal[S_GAM];
        scal[S_GAM] = r[0];
    }
};
struct F4 {  // w = f + delta w
    double* w; const double* f; int64_t ncols; const double* scal;
    __device__ bool skip() const { return scal[S_STALL] != 0.0; }
    __device__ void operator()(int64_t e, double*) const {
        if (e < ncols) w[e] = dadd(f[e], dmul(scal[S_DELTA], w[e]));
    }
};
struct FInit {  // f f  and |r|^2 at start; w = f
    double* w; const double* f; const double* r; int64_t ncols, T;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double* acc) const {
        if (e < ncols) { const double v = f[e]; w[e] = v; acc[0] += v * v; }
        if (e < T) acc[1] += r[e] * r[e];
    }
};
struct FInitPost {
    double* scal;
    __device__ void operator()(double* r) const {
        scal[S_GAM] = r[0];
        scal[S_RR] = r[1];
        scal[S_STALL] = 0.0;
    }
};
struct FTail {  // y[m..] = lam D x (augmented forward tail)
    const double* x; double* y; int64_t m, P; int n; double lx, ly;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const {
        if (e < P) y[m + e] = dmul(lx, dx_at(x, e, n));
        else if (e < 2 * P) y[m + e] = dmul(ly, dy_at(x, e - P, n));
    }
};
struct FTailT {  // out = (out + lx Dx^T y2) + ly Dy^T y3
    double* out; const double* y; int64_t m, P, ncols; int n; double lx, ly;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const {
        if (e < ncols) {
            double v = out[e];
            v = dadd(v, dmul(lx, dxt_at(y + m, e, n)));
            v = dadd(v, dmul(ly, dyt_at(y + m + P, e, n)));
            out[e] = v;
        }
    }
};
struct FSub {  // r = b - r  (warm start residual)
    double* r; const double* b; int64_t T;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const { if (e < T) r[e] = dsub(b[e], r[e]); }
};
struct FCopy {
    double* dst; const double* src; int64_t len;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const { if (e < len) dst[e] = src[e]; }
};
struct FZero {
    double* dst; int64_t len;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const { if (e < len) dst[e] = 0.0; }
};

// ------------------------------------------------------------ SB passes
__device__ __forceinline__ double shrink1(double w, double v) {
    // np.sign(w) * np.maximum(np.abs(w) - v, 0.0)   (splitbregman.py:32-35)
    const double s = (w > 0.0) ? 1.0 : ((w < 0.0) ? -1.0 : (w == 0.0 ? 0.0 : w));
    return dmul(s, fmax(dsub(fabs(w), v), 0.0));
}
struct FRhs {  // rhs = [b; lam (dx - gx); lam (dy - gy)]   (regularizers.py:120-130)
    double* rhs; const double* b; const double* ddx; const double* ddy; const double* gx;
    const double* gy; int64_t N, P; double lam;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const {
        if (e < N) rhs[e] = b[e];
        else if (e < N + P) rhs[e] = dmul(lam, dsub(ddx[e - N], gx[e - N]));
        else if (e < N + 2 * P) rhs[e] = dmul(lam, dsub(ddy[e - N - P], gy[e - N - P]));
    }
};
struct FSbUpd {  // c = Dx + g; d = shrink(c); g = c - d; norms for rc/re
    const double* x; const double* xprev; const double* xtrue; double* ddx; double* ddy;
    double* gx; double* gy; int64_t N, P; int n; double inv_gamma; int iso;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double* acc) const {
        if (e < P) {
            const double cx = dadd(dx_at(x, e, n), gx[e]);
            const double cy = dadd(dy_at(x, e, n), gy[e]);
            double dxv, dyv;
            if (!iso) {
                dxv = shrink1(cx, inv_gamma);
                dyv = shrink1(cy, inv_gamma);
            } else {
                // splitbregman.py:43-56 (pairs cx[e] with cy[e] by flat index)
                const double s = hypot(cx, cy);
                double sc = 0.0;
                if (s > 0.0) sc = fmax(dsub(s, inv_gamma), 0.0) / s;
                dxv = dmul(cx, sc);
                dyv = dmul(cy, sc);
            }
            ddx[e] = dxv; ddy[e] = dyv;
            gx[e] = dsub(cx, dxv); gy[e] = dsub(cy, dyv);
        }
        if (e < N) {
            const double d = dsub(x[e], xprev[e]);
            acc[0] += d * d;
            acc[1] += xprev[e] * xprev[e];
            if (xtrue) { const double t = dsub(x[e], xtrue[e]); acc[2] += t * t; }
        }
    }
};
struct FNorm2 {  // |a - b|^2 and |b|^2
    const double* a; const double* b; int64_t len;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double* acc) const {
        if (e < len) { const double d = dsub(a[e], b[e]); acc[0] += d * d; acc[1] += b[e] * b[e]; }
    }
};

// ------------------------------------------------------------ host helpers
struct MR {
    double* part;
    unsigned* counter;
};
template <int R, class F, class P = NoPost>
static void map_reduce(int64_t len, const F& f, const MR& mr, double* out, cudaStream_t st,
                       const P& post = P()) {
    const int blocks = mr_blocks(len);
    ProfScope ps(st, PROF_SBVEC, 0.0);
    k_map_reduce<R, F, P><<<blocks, MR_THREADS, 0, st>>>(len, f, post, mr.part, out, mr.counter);
    KB_LAUNCH_CHECK();
}

// ---- Kronecker apply (two DMMA GEMMs) ----
// intermediate P/Q (k blocks) + split-K partials of the reduced stage (8 x output)
constexpr int KRON_SPLIT_MAX = 32;
size_t kron_ws_doubles(const kb_kron* kr) {
    const int64_t a = (int64_t)kr->n1 * kr->m2, b = (int64_t)kr->m1 * kr->n2;
    const int64_t out = std::max((int64_t)kr->m1 * kr->m2, (int64_t)kr->n1 * kr->n2);
    return (size_t)kr->k * (size_t)std::max(a, b) + (size_t)KRON_SPLIT_MAX * out + 64;
}

void dgemm_sum_blocks(int r, int c, int kin, int nblk, const double* Bl, const double* P, double* Y,
                      cudaStream_t st);

// The dense reduced stage runs on cuBLAS for large images (where the GEMM, not launch
// latency, bounds a CGLS iteration); such solves run the eager CGLS loop, since cuBLAS
// launches cannot live inside a conditional-while graph body.
static bool kron_uses_cublas(const kb_kron* kr) {
    return kr->ft != nullptr && std::min(kr->m1, kr->n1) >= 512 && std::min(kr->m2, kr->n2) >= 512;
}

void kron_apply(const kb_kron* kr, const double* x, double* y, int transpose, double* tmp,
                cudaStream_t st) {
    const int m1 = kr->m1, m2 = kr->m2, n1 = kr->n1, n2 = kr->n2, k = kr->k;
    const int64_t pq = (int64_t)k * std::max((int64_t)n1 * m2, (int64_t)m1 * n2);
    double* part = tmp + ((pq + 31) / 32) * 32;
    const int64_t part_n = (int64_t)KRON_SPLIT_MAX * std::max((int64_t)m1 * m2, (int64_t)n1 * n2);
    struct Reset {
        ~Reset() {
            g_dgemm_skip = GemmSkip{};
            g_dgemm_narrow = 0;
        }
    } reset;
    g_dgemm_skip.band = kr->band;   // stage 1 only: G's zero band (kb_kron_band)
    g_dgemm_narrow = kr->fband != nullptr;   // narrow tiles along the banded dimension (split operators)
    // F side: the first nd terms dense, the other kb terms banded (kb_kron.fband); without
    // the structure every term is dense
    const int nd = kr->fband ? std::max(0, std::min(kr->ndense, k)) : k, kb = k - nd;
    if (!transpose) {
        // P_i = Xr G_i            (n1 x m2), Xr = x as n1 x n2, G_i n2 x m2
        dgemm(0, 0, n1, m2, n2, x, n2, 0, 0, kr->g, m2, (int64_t)n2 * m2, 0, tmp, m2,
              (int64_t)n1 * m2, k, 1, 0.0, st);
        g_dgemm_skip = GemmSkip{};
        // Yr = sum_i F_i^T P_i    (m1 x m2), F_i n1 x m1: one dense GEMM, inner dim nd n1 ...
        if (nd > 0) {
            if (kron_uses_cublas(kr))
                dgemm_sum_blocks(m1, m2, n1, nd, kr->f, tmp, y, st);
            else
                dgemm(1, 0, m1, m2, n1, kr->f, m1, 0, (int64_t)n1 * m1, tmp, m2, 0, (int64_t)n1 * m2, y, m2,
                      0, 1, nd, 0.0, st, part, part_n);
        }
        if (kb > 0) {   // ... plus the banded terms: the k tiles inside F's zero band only
            g_dgemm_skip.band_a = kr->fband;
            dgemm(1, 0, m1, m2, n1, kr->f + (int64_t)nd * n1 * m1, m1, 0, (int64_t)n1 * m1,
                  tmp + (int64_t)nd * n1 * m2, m2, 0, (int64_t)n1 * m2, y, m2, 0, 1, kb, nd > 0 ? 1.0 : 0.0, st,
                  part, part_n);
        }
    } else {
        // Q_i = Yr G_i^T          (m1 x n2), Yr = y as m1 x m2
        dgemm(0, 1, m1, n2, m2, x, m2, 0, 0, kr->g, m2, (int64_t)n2 * m2, 0, tmp, n2,
              (int64_t)m1 * n2, k, 1, 0.0, st);
        g_dgemm_skip = GemmSkip{};
        // Xr = sum_i F_i Q_i      (n1 x n2) = sum_i Ft_i^T Q_i with Ft_i = F_i^T (m1 x n1)
        if (nd > 0) {
            if (kron_uses_cublas(kr))
                dgemm_sum_blocks(n1, n2, m1, nd, kr->ft, tmp, y, st);
            else
                dgemm(0, 0, n1, n2, m1, kr->f, m1, 0, (int64_t)n1 * m1, tmp, n2, 0, (int64_t)m1 * n2, y, n2,
                      0, 1, nd, 0.0, st, part, part_n);
        }
        if (kb > 0) {
            g_dgemm_skip.band_a = kr->fband;
            dgemm(0, 0, n1, n2, m1, kr->f + (int64_t)nd * n1 * m1, m1, 0, (int64_t)n1 * m1,
                  tmp + (int64_t)nd * m1 * n2, n2, 0, (int64_t)m1 * n2, y, n2, 0, 1, kb, nd > 0 ? 1.0 : 0.0, st,
                  part, part_n);
        }
    }
}

// ---- generic forward (dense / kron, optionally augmented) ----
struct FwdWs {
    double* tmp = nullptr;   // kron intermediate
    MR mr{};
    double* part = nullptr;
    int64_t n_counters = 0;
};

static size_t fwd_tmp_doubles(const kb_forward* fw) {
    return fw->kind == KB_FWD_KRON ? kron_ws_doubles(&fw->kron) : 0;
}

void dense_gemv64(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* x,
                  double* y, int transpose, double* part, unsigned* counters, cudaStream_t st);

static void forward_top(const kb_forward* fw, const double* x, double* y, int transpose,
                        const FwdWs& ws, cudaStream_t st) {
    if (fw->kind == KB_FWD_KRON)
        kron_apply(&fw->kron, x, y, transpose, ws.tmp, st);
    else
        dense_gemv64(fw->a, fw->lda, fw->m, fw->n, x, y, transpose, ws.part, ws.mr.counter + 8, st);
    if (fw->allreduce)   // term-sharded operator: sum the rank-local partial products
        fw->allreduce(fw->allreduce_ctx, y, transpose ? fw->n : fw->m, reinterpret_cast<kb_stream_t>(st));
}

static void forward_apply(const kb_forward* fw, const double* x, double* y, int transpose,
                          const FwdWs& ws, cudaStream_t st) {
    forward_top(fw, x, y, transpose, ws, st);
    if (!fw->augmented) return;
    const int n = fw->side;
    const int64_t P = (int64_t)n * (n - 1);
    if (!transpose) {
        FTail f{x, y, fw->m, P, n, fw->lam_x, fw->lam_y};
        map_reduce<0>(2 * P, f, ws.mr, nullptr, st);
    } else {
        FTailT f{y, x, fw->m, P, fw->n, n, fw->lam_x, fw->lam_y};
        map_reduce<0>(fw->n, f, ws.mr, nullptr, st);
    }
}

static int64_t fwd_rows(const kb_forward* fw) {
    const int64_t P = fw->augmented ? (int64_t)fw->side * (fw->side - 1) : 0;
    return fw->m + 2 * P;
}

static void fwd_ws_size(const kb_forward* fw, Sizer& s) {
    s.take<double>(fwd_tmp_doubles(fw) + 1);
    const int64_t big = std::max<int64_t>(fwd_rows(fw), fw->n);
    s.take<double>((size_t)(4 * kSMs) * std::max<int64_t>(fw->m, fw->n) + 64);  // gemv partials
    s.take<double>((size_t)mr_blocks(big) * MR_MAXR + 64);
    s.take<unsigned>(64 + (size_t)cdiv(std::max<int64_t>(fw->m, fw->n), 128) + 64);
}

static FwdWs fwd_ws_make(const kb_forward* fw, Arena& a) {
    FwdWs w;
    w.tmp = a.take<double>(fwd_tmp_doubles(fw) + 1);
    const int64_t big = std::max<int64_t>(fwd_rows(fw), fw->n);
    w.part = a.take<double>((size_t)(4 * kSMs) * std::max<int64_t>(fw->m, fw->n) + 64);
    w.mr.part = a.take<double>((size_t)mr_blocks(big) * MR_MAXR + 64);
    w.n_counters = 64 + cdiv(std::max<int64_t>(fw->m, fw->n), 128) + 64;
    w.mr.counter = a.take<unsigned>((size_t)w.n_counters);
    return w;
}

static void validate_fw(const kb_forward* fw) {
    KB_REQUIRE(fw != nullptr, "null forward operator");
    KB_REQUIRE(fw->m >= 1 && fw->n >= 1, "forward operator has empty shape");
    if (fw->kind == KB_FWD_KRON) {
        const kb_kron& k = fw->kron;
        KB_REQUIRE(k.k >= 1 && k.m1 >= 1 && k.m2 >= 1 && k.n1 >= 1 && k.n2 >= 1, "bad Kronecker sizes");
        KB_REQUIRE((int64_t)k.m1 * k.m2 == fw->m && (int64_t)k.n1 * k.n2 == fw->n,
                   "Kronecker scheme does not match the operator shape");
    } else {
        KB_REQUIRE(fw->kind == KB_FWD_DENSE, "unknown forward kind %d", fw->kind);
        KB_REQUIRE(fw->a != nullptr && fw->lda >= fw->n, "bad dense operator");
    }
    if (fw->augmented) {
        KB_REQUIRE(fw->side >= 2 && (int64_t)fw->side * fw->side == fw->n,
                   "augmented system needs n^2 columns with n >= 2");
    }
}

// ------------------------------------------------------------ CGLS driver
struct CglsWs {
    FwdWs f;
    double *r, *z, *w, *fv, *scal;
    double* scal_host;   // pinned
    int* ctl;            // device control block
    double *rc, *res;    // device histories
    int i_cap;
};
constexpr int CGLS_ICAP = 4096;   // maximum i_max per call

static void cgls_ws_size(const kb_forward* fw, Sizer& s) {
    fwd_ws_size(fw, s);
    const int64_t T = fwd_rows(fw), N = fw->n;
    s.take<double>(T);
    s.take<double>(T);
    s.take<double>(N);
    s.take<double>(N);
    s.take<double>(S_TOTAL);
    s.take<int>(16);
    s.take<double>(CGLS_ICAP + 2);
    s.take<double>(CGLS_ICAP + 2);
}

static CglsWs cgls_ws_make(const kb_forward* fw, Arena& a) {
    CglsWs w;
    w.f = fwd_ws_make(fw, a);
    const int64_t T = fwd_rows(fw), N = fw->n;
    w.r = a.take<double>(T);
    w.z = a.take<double>(T);
    w.w = a.take<double>(N);
    w.fv = a.take<double>(N);
    w.scal = a.take<double>(S_TOTAL);
    w.scal_host = nullptr;
    w.ctl = a.take<int>(16);
    w.rc = a.take<double>(CGLS_ICAP + 2);
    w.res = a.take<double>(CGLS_ICAP + 2);
    w.i_cap = CGLS_ICAP;
    return w;
}

struct PinnedScalars {   // per-thread pinned mailbox, allocated once
    double* p = nullptr;
    PinnedScalars() {
        static thread_local double* buf = nullptr;
        if (!buf) KB_CUDA(cudaMallocHost(&buf, sizeof(double) * S_TOTAL));
        p = buf;
    }
};

// ---- CGLS control on the device (graph while-loop / eager replay share it)
enum { C_ITERS = 0, C_NRC, C_NRES, C_STOP, C_RUN, C_ERR, C_COUNT = 8 };
struct CglsCtl {
    int* h;                 // [C_COUNT]
    double* rc;             // [i_max]
    double* res;            // [i_max + 1]
    const double* scal;
    int i_max;
    double tau;
    cudaGraphConditionalHandle handle;
    int use_cond;
};

__global__ void k_cgls_init_ctl(CglsCtl c) {
    if (threadIdx.x != 0) return;
    for (int i = 0; i < C_COUNT; ++i) c.h[i] = 0;
    c.res[0] = sqrt(c.scal[S_RR]);
    c.h[C_NRES] = 1;
    c.h[C_STOP] = KB_CGLS_MAX_ITER;
    c.h[C_RUN] = c.i_max >= 1;
    if (c.use_cond) cudaGraphSetConditional(c.handle, c.h[C_RUN] ? 1u : 0u);
}

// cgls.py:90-114 stop logic, evaluated on the device after each iteration
__global__ void k_cgls_control(CglsCtl c) {
    if (threadIdx.x != 0) return;
    int* h = c.h;
    const int it = h[C_ITERS];
    if (c.scal[S_STALL] != 0.0) {
        h[C_STOP] = KB_CGLS_STALLED;
        h[C_RUN] = 0;
    } else if (!isfinite(c.scal[S_FF])) {
        h[C_ERR] = 1;
        h[C_RUN] = 0;
    } else {
        h[C_ITERS] = it + 1;
        c.res[h[C_NRES]++] = sqrt(c.scal[S_RR]);
        if (it >= 1) {
            const double xn = c.scal[S_XN];
            const double rc = xn > 0 ? c.scal[S_STEP] / xn : INFINITY;
            c.rc[h[C_NRC]++] = rc;
            if (rc < c.tau) {
                h[C_STOP] = KB_CGLS_CONVERGED;
                h[C_RUN] = 0;
            }
        }
        if (h[C_ITERS] >= c.i_max) h[C_RUN] = 0;
    }
    if (c.use_cond) cudaGraphSetConditional(c.handle, h[C_RUN] ? 1u : 0u);
}

struct CglsPlan {
    const kb_forward* fw;
    const double* b;
    const double* x0;
    double* x;
    CglsWs* w;
    CglsCtl ctl;
};

static void cgls_enqueue_init(CglsPlan& P, cudaStream_t s) {
    const kb_forward* fw = P.fw;
    CglsWs& w = *P.w;
    const int64_t T = fwd_rows(fw), N = fw->n;
    const int64_t big = std::max(T, N);
    if (P.x0 == nullptr) {
        map_reduce<0>(N, FZero{P.x, N}, w.f.mr, nullptr, s);
        map_reduce<0>(T, FCopy{w.r, P.b, T}, w.f.mr, nullptr, s);
    } else {
        if (P.x0 != P.x) map_reduce<0>(N, FCopy{P.x, P.x0, N}, w.f.mr, nullptr, s);
        forward_apply(fw, P.x, w.r, 0, w.f, s);
        map_reduce<0>(T, FSub{w.r, P.b, T}, w.f.mr, nullptr, s);
    }
    forward_apply(fw, w.r, w.fv, 1, w.f, s);
    map_reduce<2>(big, FInit{w.w, w.fv, w.r, N, T}, w.f.mr, w.scal + S_RED, s, FInitPost{w.scal});
    k_cgls_init_ctl<<<1, 32, 0, s>>>(P.ctl);
    KB_LAUNCH_CHECK();
}

static void cgls_enqueue_body(CglsPlan& P, cudaStream_t s) {
    const kb_forward* fw = P.fw;
    CglsWs& w = *P.w;
    const int64_t T = fwd_rows(fw), N = fw->n;
    const int64_t big = std::max(T, N);
    const int64_t P_ = fw->augmented ? (int64_t)fw->side * (fw->side - 1) : 0;
    const int aug = fw->augmented;
    double* x = P.x;
    forward_top(fw, w.w, w.z, 0, w.f, s);
    map_reduce<3>(big, F1{w.w, x, w.z, fw->m, N, aug ? P_ : 0, fw->side, fw->lam_x, fw->lam_y, w.scal}, w.f.mr,
                  w.scal + S_RED, s, F1Post{w.scal});
    map_reduce<0>(big, F2{x, w.w, w.r, w.z, N, T, w.scal}, w.f.mr, nullptr, s);
    forward_top(fw, w.r, w.fv, 1, w.f, s);
    map_reduce<2>(big, F3{w.fv, w.r, fw->m, N, T, P_, fw->side, fw->lam_x, fw->lam_y, aug, w.scal}, w.f.mr,
                  w.scal + S_RED, s, F3Post{w.scal});
    map_reduce<0>(N, F4{w.w, w.fv, N, w.scal}, w.f.mr, nullptr, s);
    k_cgls_control<<<1, 32, 0, s>>>(P.ctl);
    KB_LAUNCH_CHECK();
}

// CUDA-graph cache for the CGLS loop (conditional while node around one iteration)
struct CglsKey {
    kb_forward fw;
    const void *b, *x0, *x, *ws;
    int i_max;
    double tau;
    bool operator==(const CglsKey& o) const { return std::memcmp(this, &o, sizeof(CglsKey)) == 0; }
};
struct CglsGraph {
    CglsKey key;
    cudaGraphExec_t exec;
};
static std::vector<CglsGraph> g_cgls_graphs;
static cudaStream_t g_cgls_capture = nullptr;

static cudaGraphExec_t cgls_build_graph(CglsPlan& P) {
    if (!g_cgls_capture) KB_CUDA(cudaStreamCreateWithFlags(&g_cgls_capture, cudaStreamNonBlocking));
    cudaStream_t cs = g_cgls_capture;
    const bool prof = g_prof;
    g_prof = false;
    cudaGraph_t g = nullptr;
    try {
        KB_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaStreamCaptureStatus cst;
        cudaGraph_t capg;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphConditionalHandle h;
        KB_CUDA(cudaGraphConditionalHandleCreate(&h, capg, 1, cudaGraphCondAssignDefault));
        P.ctl.handle = h;
        P.ctl.use_cond = 1;
        cgls_enqueue_init(P, cs);
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        KB_CUDA(cudaGraphAddNode(&cnode, capg, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        KB_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
        KB_CUDA(cudaStreamEndCapture(cs, &g));
        KB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        cgls_enqueue_body(P, cs);
        cudaGraph_t body_out;
        KB_CUDA(cudaStreamEndCapture(cs, &body_out));
        cudaGraphExec_t exec;
        KB_CUDA(cudaGraphInstantiate(&exec, g, 0));
        KB_CUDA(cudaGraphDestroy(g));
        g_prof = prof;
        return exec;
    } catch (...) {
        g_prof = prof;
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(cs, &junk);
            if (junk) cudaGraphDestroy(junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
    }
}

// Runs CGLS (cgls.py:50-116).  x0 may alias x (warm start) or be null.
// Without an allreduce hook and without profiling the loop is one CUDA graph
// launch (device-side stop test); otherwise the same kernels run eagerly with
// a host read of the control block per iteration.
static void cgls_core(const kb_forward* fw, const double* b, const double* x0, double* x,
                      kb_cgls_state* st, CglsWs& w, double* hs, cudaStream_t s) {
    CglsPlan P{fw, b, x0, x, &w, {}};
    P.ctl.h = w.ctl;
    P.ctl.rc = w.rc;
    P.ctl.res = w.res;
    P.ctl.scal = w.scal;
    P.ctl.i_max = st->i_max;
    P.ctl.tau = st->tau;
    KB_REQUIRE(st->i_max <= w.i_cap, "i_max %d exceeds the CGLS workspace capacity %d", st->i_max, w.i_cap);
    static const bool force_eager = std::getenv("KB_CGLS_EAGER") != nullptr;
    int* hh = reinterpret_cast<int*>(hs);
    const bool cublas_stage = fw->kind == KB_FWD_KRON && kron_uses_cublas(&fw->kron);
    if (!g_prof && !force_eager && fw->allreduce == nullptr && !cublas_stage) {
        CglsKey key;
        std::memset(&key, 0, sizeof(key));
        key.fw = *fw;
        key.b = b;
        key.x0 = x0;
        key.x = x;
        key.ws = w.scal;
        key.i_max = st->i_max;
        key.tau = st->tau;
        cudaGraphExec_t exec = nullptr;
        for (auto& e : g_cgls_graphs)
            if (e.key == key) exec = e.exec;
        if (!exec) {
            exec = cgls_build_graph(P);
            if (g_cgls_graphs.size() >= 16) {
                cudaGraphExecDestroy(g_cgls_graphs.front().exec);
                g_cgls_graphs.erase(g_cgls_graphs.begin());
            }
            g_cgls_graphs.push_back({key, exec});
        }
        KB_CUDA(cudaGraphLaunch(exec, s));
    } else {
        P.ctl.use_cond = 0;
        cgls_enqueue_init(P, s);
        for (;;) {
            KB_CUDA(cudaMemcpyAsync(hh, w.ctl, sizeof(int) * C_COUNT, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            if (!hh[C_RUN]) break;
            cgls_enqueue_body(P, s);
        }
    }
    KB_CUDA(cudaMemcpyAsync(hh, w.ctl, sizeof(int) * C_COUNT, cudaMemcpyDeviceToHost, s));
    KB_CUDA(cudaStreamSynchronize(s));
    if (hh[C_ERR]) {
        set_error("CGLS produced non-finite residual quantities");
        throw Fail{KB_ENUMERICAL};
    }
    st->iters = hh[C_ITERS];
    st->stop = hh[C_STOP];
    st->n_rc = hh[C_NRC];
    st->n_res = hh[C_NRES];
    if (st->rc_host && st->n_rc)
        KB_CUDA(cudaMemcpyAsync(st->rc_host, w.rc, sizeof(double) * st->n_rc, cudaMemcpyDeviceToHost, s));
    if (st->resnorm_host && st->n_res)
        KB_CUDA(cudaMemcpyAsync(st->resnorm_host, w.res, sizeof(double) * st->n_res, cudaMemcpyDeviceToHost, s));
    if ((st->rc_host && st->n_rc) || (st->resnorm_host && st->n_res)) KB_CUDA(cudaStreamSynchronize(s));
}

// ------------------------------------------------------------ SB driver
struct SbWs {
    CglsWs c;
    double *rhs, *ddx, *ddy, *gx, *gy, *xa, *xb, *red;
};

static void sb_ws_size(const kb_forward* aug, Sizer& s) {
    cgls_ws_size(aug, s);
    const int64_t T = fwd_rows(aug), N = aug->n, P = (int64_t)aug->side * (aug->side - 1);
    s.take<double>(T);
    for (int i = 0; i < 4; ++i) s.take<double>(P);
    s.take<double>(N);
    s.take<double>(N);
    s.take<double>(16);
}

static SbWs sb_ws_make(const kb_forward* aug, Arena& a) {
    SbWs w;
    w.c = cgls_ws_make(aug, a);
    const int64_t T = fwd_rows(aug), N = aug->n, P = (int64_t)aug->side * (aug->side - 1);
    w.rhs = a.take<double>(T);
    w.ddx = a.take<double>(P);
    w.ddy = a.take<double>(P);
    w.gx = a.take<double>(P);
    w.gy = a.take<double>(P);
    w.xa = a.take<double>(N);
    w.xb = a.take<double>(N);
    w.red = a.take<double>(16);
    return w;
}

static kb_forward make_aug(const kb_forward* fw, double lam) {
    kb_forward aug = *fw;
    int64_t n = (int64_t)std::llround(std::sqrt((double)fw->n));
    aug.augmented = 1;
    aug.side = (int)n;
    aug.lam_x = lam;
    aug.lam_y = lam;
    return aug;
}

}  // namespace kb

// ================================================================ C ABI
using namespace kb;

extern "C" int kb_kron_workspace_bytes(const kb_kron* kr, size_t* bytes) {
    try {
        KB_REQUIRE(kr && bytes, "null argument");
        Sizer s;
        s.take<double>(kron_ws_doubles(kr));
        *bytes = s.off;
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

// lo = min, hi = max of (c - r) over the nonzero entries G_i[r][c] of all
// terms (band[0] > band[1] when G is all zero).  For zero boundary conditions
// the v-side factors are banded Toeplitz matrices: every q-basis vector is a
// combination of R(A)^T products, whose entries vanish exactly where the PSF
// underflows.
__global__ void k_kron_band_init(int* band) { band[0] = INT_MAX; band[1] = INT_MIN; }
__global__ void k_kron_band(const double* __restrict__ g, int k, int n2, int m2, int* band) {
    const int64_t per = (int64_t)n2 * m2, total = per * k;
    int lo = INT_MAX, hi = INT_MIN;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (g[e] != 0.0) {
            const int64_t rem = e % per;
            const int d = (int)(rem % m2) - (int)(rem / m2);
            lo = min(lo, d);
            hi = max(hi, d);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
        hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    if ((threadIdx.x & 31) == 0 && lo <= hi) {
        atomicMin(band, lo);
        atomicMax(band + 1, hi);
    }
}

extern "C" int kb_kron_band(const kb_kron* kr, int* band, kb_stream_t stream) {
    try {
        KB_REQUIRE(kr && kr->g && band, "null argument");
        KB_REQUIRE(kr->k >= 1 && kr->n2 >= 1 && kr->m2 >= 1, "bad Kronecker sizes");
        cudaStream_t st = as_stream(stream);
        k_kron_band_init<<<1, 1, 0, st>>>(band);
        KB_LAUNCH_CHECK();
        const int64_t total = (int64_t)kr->k * kr->n2 * kr->m2;
        k_kron_band<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 8 * kSMs), 256, 0, st>>>(
            kr->g, kr->k, kr->n2, kr->m2, band);
        KB_LAUNCH_CHECK();
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_kron_apply(const kb_kron* kr, const double* x, double* y, int transpose, void* ws,
                             size_t ws_bytes, kb_stream_t stream) {
    try {
        KB_REQUIRE(kr && x && y, "null argument");
        KB_REQUIRE(kr->k >= 1 && kr->m1 >= 1 && kr->m2 >= 1 && kr->n1 >= 1 && kr->n2 >= 1,
                   "bad Kronecker sizes");
        Arena a(ws, ws_bytes);
        double* tmp = a.take<double>(kron_ws_doubles(kr));
        kron_apply(kr, x, y, transpose, tmp, as_stream(stream));
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_dgemm(int trans_a, int trans_b, int m, int n, int k, const double* A, int64_t lda,
                        int64_t sa_batch, int64_t sa_seg, const double* B, int64_t ldb,
                        int64_t sb_batch, int64_t sb_seg, double* C, int64_t ldc, int64_t sc_batch,
                        int nbatch, int nseg, double beta, kb_stream_t stream) {
    try {
        dgemm(trans_a, trans_b, m, n, k, A, lda, sa_batch, sa_seg, B, ldb, sb_batch, sb_seg, C, ldc,
              sc_batch, nbatch, nseg, beta, as_stream(stream));
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_forward_workspace_bytes(const kb_forward* fw, size_t* bytes) {
    try {
        validate_fw(fw);
        Sizer s;
        fwd_ws_size(fw, s);
        *bytes = s.off;
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_forward_apply(const kb_forward* fw, const double* x, double* y, int transpose,
                                void* ws, size_t ws_bytes, kb_stream_t stream) {
    try {
        validate_fw(fw);
        Arena a(ws, ws_bytes);
        FwdWs w = fwd_ws_make(fw, a);
        KB_CUDA(cudaMemsetAsync(w.mr.counter, 0, sizeof(unsigned) * w.n_counters, as_stream(stream)));
        forward_apply(fw, x, y, transpose, w, as_stream(stream));
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_cgls_workspace_bytes(const kb_forward* fw, size_t* bytes) {
    try {
        validate_fw(fw);
        Sizer s;
        cgls_ws_size(fw, s);
        *bytes = s.off;
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_cgls_run(const kb_forward* fw, const double* b, const double* x0, double* x,
                           kb_cgls_state* st, void* ws, size_t ws_bytes, kb_stream_t stream) {
    try {
        validate_fw(fw);
        KB_REQUIRE(st && b && x, "null argument");
        KB_REQUIRE(st->i_max >= 1, "i_max must be >= 1");
        KB_REQUIRE(st->tau >= 0, "tau must be >= 0");
        Arena a(ws, ws_bytes);
        CglsWs w = cgls_ws_make(fw, a);
        cudaStream_t s = as_stream(stream);
        KB_CUDA(cudaMemsetAsync(w.f.mr.counter, 0, sizeof(unsigned) * w.f.n_counters, s));
        PinnedScalars hs;
        cgls_core(fw, b, x0, x, st, w, hs.p, s);
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_sb_workspace_bytes(const kb_forward* fw, size_t* bytes) {
    try {
        validate_fw(fw);
        kb_forward aug = make_aug(fw, 1.0);
        validate_fw(&aug);
        Sizer s;
        sb_ws_size(&aug, s);
        *bytes = s.off;
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_sb_run(const kb_forward* fw, const double* b, const double* x_true, double* x,
                         kb_sb_state* st, void* ws, size_t ws_bytes, kb_stream_t stream) {
    try {
        validate_fw(fw);
        KB_REQUIRE(st && b && x, "null argument");
        KB_REQUIRE(fw->m == fw->n, "operator must be square to start from the observed image");
        KB_REQUIRE(!fw->augmented, "pass the plain forward operator to kb_sb_run");
        KB_REQUIRE(st->lam > 0 && st->beta > 0, "lam and beta must be positive");
        KB_REQUIRE(st->l_max >= 1 && st->i_max >= 1, "l_max and i_max must be >= 1");
        const double lam = st->lam, gamma = lam * lam / st->beta;
        kb_forward aug = make_aug(fw, lam);
        validate_fw(&aug);
        Arena a(ws, ws_bytes);
        SbWs w = sb_ws_make(&aug, a);
        cudaStream_t s = as_stream(stream);
        KB_CUDA(cudaMemsetAsync(w.c.f.mr.counter, 0, sizeof(unsigned) * w.c.f.n_counters, s));
        const int64_t N = aug.n, P = (int64_t)aug.side * (aug.side - 1), T = fwd_rows(&aug);
        const int n = aug.side;
        PinnedScalars hs;
        // x_prev = b; d = g = 0  (splitbregman.py:158-162)
        double* xprev = w.xa;
        double* xcur = w.xb;
        map_reduce<0>(N, FCopy{xprev, b, N}, w.c.f.mr, nullptr, s);
        for (double* p : {w.ddx, w.ddy, w.gx, w.gy}) map_reduce<0>(P, FZero{p, P}, w.c.f.mr, nullptr, s);
        double obs = 0.0, xt_norm = 1.0;
        if (x_true) {
            map_reduce<2>(N, FNorm2{b, x_true, N}, w.c.f.mr, w.red, s);
            KB_CUDA(cudaMemcpyAsync(hs.p, w.red, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            obs = std::sqrt(hs.p[0]);
            xt_norm = std::sqrt(hs.p[1]);
            KB_REQUIRE(xt_norm != 0.0, "relative_error is undefined for a zero reference");
        }
        st->outer_iters = 0;
        st->stop = KB_SB_MAX_ITER;
        kb_cgls_state cs{};
        cs.i_max = st->i_max;
        cs.tau = st->tau_cgls;
        for (int l = 0; l < st->l_max; ++l) {
            map_reduce<0>(T, FRhs{w.rhs, b, w.ddx, w.ddy, w.gx, w.gy, N, P, lam}, w.c.f.mr, nullptr, s);
            cgls_core(&aug, w.rhs, st->warm_start ? xprev : nullptr, xcur, &cs, w.c, hs.p, s);
            map_reduce<3>(N, FSbUpd{xcur, xprev, x_true, w.ddx, w.ddy, w.gx, w.gy, N, P, n, 1.0 / gamma,
                                    st->variant == KB_SB_ISOTROPIC},
                          w.c.f.mr, w.red, s);
            KB_CUDA(cudaMemcpyAsync(hs.p, w.red, sizeof(double) * 3, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            st->outer_iters++;
            if (st->cgls_iters_host) st->cgls_iters_host[l] = cs.iters;
            if (hs.p[1] == 0.0) {
                set_error("relative_change is undefined for a zero previous iterate");
                throw Fail{KB_EVALIDATION};
            }
            const double rc = std::sqrt(hs.p[0]) / std::sqrt(hs.p[1]);
            if (st->rc_host) st->rc_host[l] = rc;
            if (x_true) {
                const double err = std::sqrt(hs.p[2]);
                if (st->re_host) st->re_host[l] = err / xt_norm;
                double isnr;
                if (err == 0.0 && obs == 0.0) isnr = 0.0;
                else if (err == 0.0) isnr = INFINITY;
                else if (obs == 0.0) isnr = -INFINITY;
                else isnr = 20.0 * std::log10(obs / err);
                if (st->isnr_host) st->isnr_host[l] = isnr;
            }
            std::swap(xprev, xcur);
            if (rc < st->tau) {
                st->stop = KB_SB_CONVERGED;
                break;
            }
        }
        map_reduce<0>(N, FCopy{x, xprev, N}, w.c.f.mr, nullptr, s);
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

// ---------------------------------------------------------------- elementwise pieces
namespace kb {
struct FDiff {
    const double* x; double* out; int n; int axis; int transpose; double scale; int accumulate; int64_t len;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const {
        if (e >= len) return;
        double v;
        if (!transpose) v = axis == 0 ? dx_at(x, e, n) : dy_at(x, e, n);
        else v = axis == 0 ? dxt_at(x, e, n) : dyt_at(x, e, n);
        v = dmul(scale, v);
        out[e] = accumulate ? dadd(out[e], v) : v;
    }
};
struct FShrink {
    const double* cx; const double* cy; double* dx; double* dy; int64_t len; double inv_gamma; int iso;
    __device__ bool skip() const { return false; }
    __device__ void operator()(int64_t e, double*) const {
        if (e >= len) return;
        const double a = cx[e], b = cy[e];
        if (!iso) { dx[e] = shrink1(a, inv_gamma); dy[e] = shrink1(b, inv_gamma); return; }
        const double s = hypot(a, b);
        double sc = 0.0;
        if (s > 0.0) sc = fmax(dsub(s, inv_gamma), 0.0) / s;
        dx[e] = dmul(a, sc);
        dy[e] = dmul(b, sc);
    }
};
}  // namespace kb

extern "C" int kb_diff(const double* x, double* out, int side, int axis, int transpose, double scale,
                       int accumulate, kb_stream_t stream) {
    try {
        KB_REQUIRE(x && out, "null argument");
        KB_REQUIRE(side >= 2, "first differences need n >= 2");
        const int64_t len = transpose ? (int64_t)side * side : (int64_t)side * (side - 1);
        MR mr{nullptr, nullptr};
        map_reduce<0>(len, FDiff{x, out, side, axis, transpose, scale, accumulate, len}, mr, nullptr,
                      as_stream(stream));
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

extern "C" int kb_shrink_update(const double* cx, const double* cy, double* dx, double* dy,
                                int64_t len, double gamma, int variant, kb_stream_t stream) {
    try {
        KB_REQUIRE(gamma > 0, "gamma must be positive");
        MR mr{nullptr, nullptr};
        map_reduce<0>(len, FShrink{cx, cy, dx, dy, len, 1.0 / gamma, variant == KB_SB_ISOTROPIC}, mr,
                      nullptr, as_stream(stream));
        return KB_OK;
    } catch (Fail f) {
        return f.code;
    }
}

// ================================================================ batched lambda sweep
// kb_sb_run_batch: nprob SB solves (same b, same Kronecker operator, per-problem
// lam/beta) in lock step.  State vectors are stacked problem-major; every
// vector pass is one launch with blockIdx.y = problem (per-problem fixed-order
// reductions and on-device scalars, exactly the single-problem functors), and
// each Kronecker product is one pair of batched DMMA GEMMs with the images
// stacked along M.  Stopped problems are masked (their blocks exit at once).
namespace kb {

// Test hook (kb_sb_batch_exact): split the stacked GEMMs per problem exactly as
// kb_sb_run does, so every problem of a batch is bit-identical to its own run.
static int g_sbb_exact = 0;

template <int R, class F, class P>
__global__ void __launch_bounds__(MR_THREADS)
k_map_reduce_b(int64_t len, F f, P post, double* part, double* out, int out_stride, unsigned* counter) {
    __shared__ double sw[MR_THREADS / 32][MR_MAXR];
    __shared__ double fin[MR_MAXR];
    const int b = blockIdx.y;
    if (f.skip(b)) return;   // uniform per problem
    double acc[R > 0 ? R : 1];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
    for (int64_t e = blockIdx.x * (int64_t)MR_THREADS + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * MR_THREADS)
        f(b, e, acc);
    if (R == 0) return;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int r = 0; r < R; ++r) {
        double v = warp_sum(acc[r]);
        if (lane == 0) sw[warp][r] = v;
    }
    __syncthreads();
    double* pb = part + (int64_t)b * gridDim.x * R;
    if (threadIdx.x < R) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < MR_THREADS / 32; ++w) s += sw[w][threadIdx.x];
        pb[(int64_t)blockIdx.x * R + threadIdx.x] = s;
    }
    if (last_block_ticket(counter + b, gridDim.x)) {
        if (warp < R) {
            double s = 0.0;
            for (int q = lane; q < (int)gridDim.x; q += 32) s += __ldcg(&pb[(int64_t)q * R + warp]);
            s = warp_sum(s);
            if (lane == 0) fin[warp] = s;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double* ob = out + (int64_t)b * out_stride;
            for (int r = 0; r < R; ++r) ob[r] = fin[r];
            post(b, ob);
        }
    }
}

// Batched views of the single-problem functors: problem b's vectors start at
// base + b * stride; scalars at scal + b * S_TOTAL; lam per problem.
struct BNoPost {
    __device__ void operator()(int, double*) const {}
};
template <class P>
struct BPost {   // P(scal + b * S_TOTAL)
    double* scal;
    __device__ void operator()(int b, double* r) const { P{scal + (int64_t)b * S_TOTAL}(r); }
};

struct BF1 {
    const double* w; const double* x; double* z; int64_t m, ncols, P, T; int n; const double* lam;
    double* scal; const int* run;
    __device__ bool skip(int b) const { return !run[b * C_COUNT + C_RUN]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        F1{w + b * ncols, x + b * ncols, z + b * T, m, ncols, P, n, lam[b], lam[b], scal + b * S_TOTAL}(e, acc);
    }
};
struct BF2 {
    double* x; const double* w; double* r; const double* z; int64_t ncols, T; const double* scal; const int* run;
    __device__ bool skip(int b) const { return !run[b * C_COUNT + C_RUN] || scal[b * S_TOTAL + S_STALL] != 0.0; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        F2{x + b * ncols, w + b * ncols, r + b * T, z + b * T, ncols, T, scal + b * S_TOTAL}(e, acc);
    }
};
struct BF3 {
    double* f; const double* r; int64_t m, ncols, T, P; int n; const double* lam; int aug; const double* scal;
    const int* run;
    __device__ bool skip(int b) const { return !run[b * C_COUNT + C_RUN] || scal[b * S_TOTAL + S_STALL] != 0.0; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        F3{f + b * ncols, r + b * T, m, ncols, T, P, n, lam[b], lam[b], aug, scal + b * S_TOTAL}(e, acc);
    }
};
struct BF4 {
    double* w; const double* f; int64_t ncols; const double* scal; const int* run;
    __device__ bool skip(int b) const { return !run[b * C_COUNT + C_RUN] || scal[b * S_TOTAL + S_STALL] != 0.0; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        F4{w + b * ncols, f + b * ncols, ncols, scal + b * S_TOTAL}(e, acc);
    }
};
struct BFInit {
    double* w; const double* f; const double* r; int64_t ncols, T; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        FInit{w + b * ncols, f + b * ncols, r + b * T, ncols, T}(e, acc);
    }
};
struct BFCopy {   // dst_b = src_b (src stride may be 0: the shared b)
    double* dst; const double* src; int64_t len, dst_stride, src_stride; const int* active;
    __device__ bool skip(int b) const { return active && !active[b]; }
    __device__ void operator()(int b, int64_t e, double*) const {
        if (e < len) dst[b * dst_stride + e] = src[b * src_stride + e];
    }
};
struct BFSub {   // r_b = rhs_b - r_b
    double* r; const double* rhs; int64_t T; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const { FSub{r + b * T, rhs + b * T, T}(e, acc); }
};
struct BFTail {  // y_b[m..] = lam_b D x_b
    const double* x; double* y; int64_t m, P, ncols, T; int n; const double* lam; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        FTail{x + b * ncols, y + b * T, m, P, n, lam[b], lam[b]}(e, acc);
    }
};
struct BFTailT {  // out_b = (out_b + lam Dx^T y2) + lam Dy^T y3
    double* out; const double* y; int64_t m, P, ncols, T; int n; const double* lam; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        FTailT{out + b * ncols, y + b * T, m, P, ncols, n, lam[b], lam[b]}(e, acc);
    }
};
struct BFRhs {
    double* rhs; const double* bb; const double* ddx; const double* ddy; const double* gx; const double* gy;
    int64_t N, P, T; const double* lam; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        FRhs{rhs + b * T, bb, ddx + b * P, ddy + b * P, gx + b * P, gy + b * P, N, P, lam[b]}(e, acc);
    }
};
struct BFSbUpd {
    const double* x; const double* xprev; const double* xtrue; double* ddx; double* ddy; double* gx; double* gy;
    int64_t N, P; int n; const double* inv_gamma; int iso; const int* active;
    __device__ bool skip(int b) const { return !active[b]; }
    __device__ void operator()(int b, int64_t e, double* acc) const {
        FSbUpd{x + b * N, xprev + b * N, xtrue, ddx + b * P, ddy + b * P, gx + b * P, gy + b * P, N, P, n,
               inv_gamma[b], iso}(e, acc);
    }
};

struct BMR {
    double* part;       // [nprob][blocks][MR_MAXR]
    unsigned* counter;  // [nprob]
    int nprob;
};
template <int R, class F, class P = BNoPost>
static void map_reduce_b(int64_t len, const F& f, const BMR& mr, double* out, int out_stride, cudaStream_t st,
                         const P& post = P()) {
    const dim3 grid((unsigned)mr_blocks(len), (unsigned)mr.nprob);
    ProfScope ps(st, PROF_SBVEC, 0.0);
    k_map_reduce_b<R, F, P><<<grid, MR_THREADS, 0, st>>>(len, f, post, mr.part, out, out_stride, mr.counter);
    KB_LAUNCH_CHECK();
}

// Y_b = A X_b for all problems: two batched DMMA GEMMs, images stacked along M.
// x: B stacked inputs (contiguous, stride = input length); y: B outputs at stride ys.
// flags/stride: per-problem activity (GEMM tiles of inactive problems exit).
static void kron_apply_b(const kb_kron* kr, int B, const double* x, double* y, int64_t ys, int transpose,
                         double* tmp, double* part, int64_t part_n, const int* flags, int stride,
                         cudaStream_t st) {
    const int m1 = kr->m1, m2 = kr->m2, n1 = kr->n1, n2 = kr->n2, k = kr->k;
    struct Reset {
        ~Reset() { g_dgemm_skip = GemmSkip{}; }
    } reset;
    g_dgemm_skip = GemmSkip{flags, stride, transpose ? m1 : n1, kr->band};   // stage 1: problems stacked along M
    if (!transpose) {
        // P_i = [X_1; ...; X_B] G_i   ((B n1) x m2)
        dgemm(0, 0, B * n1, m2, n2, x, n2, 0, 0, kr->g, m2, (int64_t)n2 * m2, 0, tmp, m2,
              (int64_t)B * n1 * m2, k, 1, 0.0, st);
        // Y_b = sum_i F_i^T P_{i,b}   (m1 x m2), batch over b, segments over i
        g_dgemm_skip = GemmSkip{flags, stride, 0};                          // stage 2: batch = problem
        g_dgemm_split_per_batch = g_sbb_exact;
        dgemm(1, 0, m1, m2, n1, kr->f, m1, 0, (int64_t)n1 * m1, tmp, m2, (int64_t)n1 * m2,
              (int64_t)B * n1 * m2, y, m2, ys, B, k, 0.0, st, part, part_n);
        g_dgemm_split_per_batch = 0;
    } else {
        dgemm(0, 1, B * m1, n2, m2, x, m2, 0, 0, kr->g, m2, (int64_t)n2 * m2, 0, tmp, n2,
              (int64_t)B * m1 * n2, k, 1, 0.0, st);
        g_dgemm_skip = GemmSkip{flags, stride, 0};
        g_dgemm_split_per_batch = g_sbb_exact;
        dgemm(0, 0, n1, n2, m1, kr->f, m1, 0, (int64_t)n1 * m1, tmp, n2, (int64_t)m1 * n2,
              (int64_t)B * m1 * n2, y, n2, ys, B, k, 0.0, st, part, part_n);
        g_dgemm_split_per_batch = 0;
    }
}

struct SbBatchWs {
    double *r, *z, *w, *fv, *scal, *rhs, *ddx, *ddy, *gx, *gy, *xa, *xb, *red, *lam, *inv_gamma;
    double *tmp, *part, *rc, *res, *gather;
    int64_t part_n;
    int* ctl;       // [nprob][C_COUNT]
    int* active;    // [nprob]
    int* any;       // [4]
    BMR mr;
};

static int64_t sbb_part_doubles(const kb_forward* fw, int B) {
    if (g_sbb_exact) return (int64_t)KRON_SPLIT_MAX * B * std::max(fw->m, fw->n) + 64;
    // split-K partials (dgemm halves its splits to fit); at least the single-problem
    // budget, so a batch of one runs exactly the GEMMs of kb_sb_run
    const int64_t out = std::max(fw->m, fw->n);
    return std::max((int64_t)4 * B * out, (int64_t)KRON_SPLIT_MAX * out) + 64;
}

template <class A>
static void sbb_layout(const kb_forward* aug, int B, A& a, SbBatchWs* w) {
    const int64_t T = fwd_rows(aug), N = aug->n, P = (int64_t)aug->side * (aug->side - 1);
    const kb_kron& kr = aug->kron;
    const int64_t tmp_n = (int64_t)kr.k * B * std::max((int64_t)kr.n1 * kr.m2, (int64_t)kr.m1 * kr.n2);
    const int64_t blocks = mr_blocks(std::max(T, N));
    auto take_d = [&](int64_t cnt) { return a.template take<double>((size_t)cnt); };
    auto take_i = [&](int64_t cnt) { return a.template take<int>((size_t)cnt); };
    double* p[21];
    int64_t sizes[] = {B * T, B * T, B * N, B * N, (int64_t)B * S_TOTAL, B * T, B * P, B * P, B * P, B * P,
                       B * N, B * N, (int64_t)B * 4, B, B, tmp_n + 64, sbb_part_doubles(aug, B),
                       (int64_t)B * (CGLS_ICAP + 2), (int64_t)B * (CGLS_ICAP + 2), blocks * MR_MAXR * B + 64,
                       (int64_t)B * std::max(N, aug->m)};
    for (int i = 0; i < 21; ++i) p[i] = take_d(sizes[i]);
    int* ctl = take_i((int64_t)B * C_COUNT);
    int* active = take_i(B);
    int* any = take_i(4);
    unsigned* counter = a.template take<unsigned>((size_t)B + 64);
    if (w) {
        w->r = p[0]; w->z = p[1]; w->w = p[2]; w->fv = p[3]; w->scal = p[4]; w->rhs = p[5];
        w->ddx = p[6]; w->ddy = p[7]; w->gx = p[8]; w->gy = p[9]; w->xa = p[10]; w->xb = p[11];
        w->red = p[12]; w->lam = p[13]; w->inv_gamma = p[14]; w->tmp = p[15]; w->part = p[16];
        w->part_n = sizes[16]; w->rc = p[17]; w->res = p[18];
        w->mr = BMR{p[19], counter, B};
        w->gather = p[20];
        w->ctl = ctl; w->active = active; w->any = any;
    }
}

// y_b = A x_b (or A^T x_b) for all problems; x_b at stride xs, y_b at stride ys.
// The stacked first GEMM needs contiguous inputs: strided ones (the tops of
// the augmented residuals) are gathered first (one B x len copy).
static void forward_top_b(const kb_forward* fw, int B, const double* x, int64_t xs, double* y, int64_t ys,
                          int transpose, SbBatchWs& w, const int* flags, int stride, cudaStream_t st) {
    const int64_t in_len = transpose ? fw->m : fw->n;
    if (xs != in_len) {
        map_reduce_b<0>(in_len, BFCopy{w.gather, x, in_len, in_len, xs, nullptr}, w.mr, nullptr, 0, st);
        x = w.gather;
    }
    kron_apply_b(&fw->kron, B, x, y, ys, transpose, w.tmp, w.part, w.part_n, flags, stride, st);
}

struct CglsCtlB {
    int* h;            // [nprob][C_COUNT]
    double* rc;        // [nprob][CGLS_ICAP + 2]
    double* res;
    const double* scal;
    const int* active;
    int* any;
    int nprob, i_max;
    double tau;
    cudaGraphConditionalHandle handle;
    int use_cond;
};

__global__ void k_cgls_init_ctl_b(CglsCtlB c) {
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < c.nprob; b += blockDim.x) {
        int* h = c.h + b * C_COUNT;
        for (int i = 0; i < C_COUNT; ++i) h[i] = 0;
        h[C_STOP] = KB_CGLS_MAX_ITER;
        if (c.active[b]) {
            c.res[(int64_t)b * (CGLS_ICAP + 2)] = sqrt(c.scal[b * S_TOTAL + S_RR]);
            h[C_NRES] = 1;
            h[C_RUN] = c.i_max >= 1;
            if (h[C_RUN]) atomicOr(&any, 1);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        c.any[0] = any;
        if (c.use_cond) cudaGraphSetConditional(c.handle, any ? 1u : 0u);
    }
}

// cgls.py:90-114 per problem (k_cgls_control), then "any problem still running"
__global__ void k_cgls_control_b(CglsCtlB c) {
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    for (int b = threadIdx.x; b < c.nprob; b += blockDim.x) {
        int* h = c.h + b * C_COUNT;
        if (!h[C_RUN]) continue;
        const double* scal = c.scal + b * S_TOTAL;
        double* rc = c.rc + (int64_t)b * (CGLS_ICAP + 2);
        double* res = c.res + (int64_t)b * (CGLS_ICAP + 2);
        const int it = h[C_ITERS];
        if (scal[S_STALL] != 0.0) {
            h[C_STOP] = KB_CGLS_STALLED;
            h[C_RUN] = 0;
        } else if (!isfinite(scal[S_FF])) {
            h[C_ERR] = 1;
            h[C_RUN] = 0;
        } else {
            h[C_ITERS] = it + 1;
            res[h[C_NRES]++] = sqrt(scal[S_RR]);
            if (it >= 1) {
                const double xn = scal[S_XN];
                const double r = xn > 0 ? scal[S_STEP] / xn : INFINITY;
                rc[h[C_NRC]++] = r;
                if (r < c.tau) {
                    h[C_STOP] = KB_CGLS_CONVERGED;
                    h[C_RUN] = 0;
                }
            }
            if (h[C_ITERS] >= c.i_max) h[C_RUN] = 0;
        }
        if (h[C_RUN]) atomicOr(&any, 1);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        c.any[0] = any;
        if (c.use_cond) cudaGraphSetConditional(c.handle, any ? 1u : 0u);
    }
}

struct CglsPlanB {
    const kb_forward* aug;   // augmented operator (lam_x / lam_y unused: per-problem lam in w.lam)
    int B;
    const double* rhs;       // [B][T]
    const double* x0;        // [B][N] or null
    double* x;               // [B][N]
    SbBatchWs* w;
    CglsCtlB ctl;
};

static void cglsb_enqueue_init(CglsPlanB& P, cudaStream_t s) {
    const kb_forward* fw = P.aug;
    SbBatchWs& w = *P.w;
    const int64_t T = fwd_rows(fw), N = fw->n, Pn = (int64_t)fw->side * (fw->side - 1);
    const int n = fw->side;
    const int64_t big = std::max(T, N);
    if (P.x0 == nullptr) {
        KB_CUDA(cudaMemsetAsync(P.x, 0, sizeof(double) * (size_t)P.B * N, s));
        map_reduce_b<0>(T, BFCopy{w.r, P.rhs, T, T, T, w.active}, w.mr, nullptr, 0, s);
    } else {
        if (P.x0 != P.x) map_reduce_b<0>(N, BFCopy{P.x, P.x0, N, N, N, w.active}, w.mr, nullptr, 0, s);
        forward_top_b(fw, P.B, P.x, N, w.r, T, 0, w, w.active, 1, s);
        map_reduce_b<0>(2 * Pn, BFTail{P.x, w.r, fw->m, Pn, N, T, n, w.lam, w.active}, w.mr, nullptr, 0, s);
        map_reduce_b<0>(T, BFSub{w.r, P.rhs, T, w.active}, w.mr, nullptr, 0, s);
    }
    forward_top_b(fw, P.B, w.r, T, w.fv, N, 1, w, w.active, 1, s);
    map_reduce_b<0>(N, BFTailT{w.fv, w.r, fw->m, Pn, N, T, n, w.lam, w.active}, w.mr, nullptr, 0, s);
    map_reduce_b<2>(big, BFInit{w.w, w.fv, w.r, N, T, w.active}, w.mr, w.scal + S_RED, S_TOTAL, s,
                    BPost<FInitPost>{w.scal});
    k_cgls_init_ctl_b<<<1, 256, 0, s>>>(P.ctl);
    KB_LAUNCH_CHECK();
}

static void cglsb_enqueue_body(CglsPlanB& P, cudaStream_t s) {
    const kb_forward* fw = P.aug;
    SbBatchWs& w = *P.w;
    const int64_t T = fwd_rows(fw), N = fw->n, Pn = (int64_t)fw->side * (fw->side - 1);
    const int64_t big = std::max(T, N);
    double* x = P.x;
    forward_top_b(fw, P.B, w.w, N, w.z, T, 0, w, w.ctl + C_RUN, C_COUNT, s);
    map_reduce_b<3>(big, BF1{w.w, x, w.z, fw->m, N, Pn, T, fw->side, w.lam, w.scal, w.ctl}, w.mr, w.scal + S_RED,
                    S_TOTAL, s, BPost<F1Post>{w.scal});
    map_reduce_b<0>(big, BF2{x, w.w, w.r, w.z, N, T, w.scal, w.ctl}, w.mr, nullptr, 0, s);
    forward_top_b(fw, P.B, w.r, T, w.fv, N, 1, w, w.ctl + C_RUN, C_COUNT, s);
    map_reduce_b<2>(big, BF3{w.fv, w.r, fw->m, N, T, Pn, fw->side, w.lam, 1, w.scal, w.ctl}, w.mr,
                    w.scal + S_RED, S_TOTAL, s, BPost<F3Post>{w.scal});
    map_reduce_b<0>(N, BF4{w.w, w.fv, N, w.scal, w.ctl}, w.mr, nullptr, 0, s);
    k_cgls_control_b<<<1, 256, 0, s>>>(P.ctl);
    KB_LAUNCH_CHECK();
}

struct CglsKeyB {
    kb_forward fw;
    const void *rhs, *x0, *x;
    const void* ws[10];   // every workspace array the graph addresses (the layout depends on the mode)
    int B, i_max, exact;
    double tau;
    bool operator==(const CglsKeyB& o) const { return std::memcmp(this, &o, sizeof(CglsKeyB)) == 0; }
};
struct CglsGraphB {
    CglsKeyB key;
    cudaGraphExec_t exec;
};
static std::vector<CglsGraphB> g_cglsb_graphs;

static cudaGraphExec_t cglsb_build_graph(CglsPlanB& P) {
    if (!g_cgls_capture) KB_CUDA(cudaStreamCreateWithFlags(&g_cgls_capture, cudaStreamNonBlocking));
    cudaStream_t cs = g_cgls_capture;
    const bool prof = g_prof;
    g_prof = false;
    cudaGraph_t g = nullptr;
    try {
        KB_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaStreamCaptureStatus cst;
        cudaGraph_t capg;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphConditionalHandle h;
        KB_CUDA(cudaGraphConditionalHandleCreate(&h, capg, 1, cudaGraphCondAssignDefault));
        P.ctl.handle = h;
        P.ctl.use_cond = 1;
        cglsb_enqueue_init(P, cs);
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        KB_CUDA(cudaGraphAddNode(&cnode, capg, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        KB_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
        KB_CUDA(cudaStreamEndCapture(cs, &g));
        KB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        cglsb_enqueue_body(P, cs);
        cudaGraph_t body_out;
        KB_CUDA(cudaStreamEndCapture(cs, &body_out));
        cudaGraphExec_t exec;
        KB_CUDA(cudaGraphInstantiate(&exec, g, 0));
        KB_CUDA(cudaGraphDestroy(g));
        g_prof = prof;
        return exec;
    } catch (...) {
        g_prof = prof;
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
            cudaGraph_t junk = nullptr;
            cudaStreamEndCapture(cs, &junk);
            if (junk) cudaGraphDestroy(junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
    }
}

// Pinned host mailbox that grows on demand (per thread).
static double* pinned_doubles(size_t count) {
    static thread_local double* buf = nullptr;
    static thread_local size_t cap = 0;
    if (count > cap) {
        if (buf) cudaFreeHost(buf);
        buf = nullptr;
        const size_t want = std::max<size_t>(count, 4096);
        KB_CUDA(cudaMallocHost(&buf, sizeof(double) * want));
        cap = want;
    }
    return buf;
}

// One batched CGLS solve over the active problems (graph while-loop unless
// profiling / sharded).  Returns the per-problem control blocks in hh.
static void cglsb_core(CglsPlanB& P, int* hh, cudaStream_t s) {
    static const bool force_eager = std::getenv("KB_CGLS_EAGER") != nullptr;
    SbBatchWs& w = *P.w;
    if (!g_prof && !force_eager && P.aug->allreduce == nullptr) {
        CglsKeyB key;
        std::memset(&key, 0, sizeof(key));
        key.fw = *P.aug;
        key.rhs = P.rhs;
        key.x0 = P.x0;
        key.x = P.x;
        const void* wsp[10] = {w.scal, w.ctl, w.active, w.part, w.gather, w.mr.part, w.mr.counter, w.tmp, w.lam,
                               w.rc};
        std::memcpy(key.ws, wsp, sizeof(wsp));
        key.exact = g_sbb_exact;
        key.B = P.B;
        key.i_max = P.ctl.i_max;
        key.tau = P.ctl.tau;
        cudaGraphExec_t exec = nullptr;
        for (auto& e : g_cglsb_graphs)
            if (e.key == key) exec = e.exec;
        if (!exec) {
            exec = cglsb_build_graph(P);
            if (g_cglsb_graphs.size() >= 8) {
                cudaGraphExecDestroy(g_cglsb_graphs.front().exec);
                g_cglsb_graphs.erase(g_cglsb_graphs.begin());
            }
            g_cglsb_graphs.push_back({key, exec});
        }
        KB_CUDA(cudaGraphLaunch(exec, s));
    } else {
        P.ctl.use_cond = 0;
        cglsb_enqueue_init(P, s);
        int* any = reinterpret_cast<int*>(hh);
        for (;;) {
            KB_CUDA(cudaMemcpyAsync(any, w.any, sizeof(int), cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            if (!any[0]) break;
            cglsb_enqueue_body(P, s);
        }
    }
    KB_CUDA(cudaMemcpyAsync(hh, w.ctl, sizeof(int) * C_COUNT * P.B, cudaMemcpyDeviceToHost, s));
    KB_CUDA(cudaStreamSynchronize(s));
}

}  // namespace kb

extern "C" void kb_sb_batch_exact(int on) { g_sbb_exact = on != 0; }

extern "C" int kb_sb_batch_workspace_bytes(const kb_forward* fw, int nprob, size_t* bytes) {
    KB_GUARD({
        validate_fw(fw);
        KB_REQUIRE(bytes && nprob >= 1, "bad arguments");
        KB_REQUIRE(fw->kind == KB_FWD_KRON, "the batched sweep needs a Kronecker operator");
        kb_forward aug = make_aug(fw, 1.0);
        validate_fw(&aug);
        Sizer z;
        sbb_layout(&aug, nprob, z, nullptr);
        *bytes = z.off;
    })
}

extern "C" int kb_sb_run_batch(const kb_forward* fw, const double* b, const double* x_true, double* x,
                               kb_sb_batch* st, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        validate_fw(fw);
        KB_REQUIRE(st && b && x && st->lam_host && st->beta_host && st->outer_iters_host && st->stop_host,
                   "null argument");
        KB_REQUIRE(fw->kind == KB_FWD_KRON, "the batched sweep needs a Kronecker operator");
        KB_REQUIRE(fw->allreduce == nullptr, "the batched sweep runs on one device (no term sharding)");
        KB_REQUIRE(fw->m == fw->n, "operator must be square to start from the observed image");
        KB_REQUIRE(!fw->augmented, "pass the plain forward operator to kb_sb_run_batch");
        KB_REQUIRE(st->nprob >= 1 && st->nprob <= 65535, "nprob must be in [1, 65535]");
        KB_REQUIRE(st->l_max >= 1 && st->i_max >= 1, "l_max and i_max must be >= 1");
        KB_REQUIRE(st->i_max <= CGLS_ICAP, "i_max %d exceeds the CGLS history capacity %d", st->i_max, CGLS_ICAP);
        const int B = st->nprob;
        std::vector<double> lam(B), invg(B);
        for (int p = 0; p < B; ++p) {
            KB_REQUIRE(st->lam_host[p] > 0 && st->beta_host[p] > 0, "lam and beta must be positive");
            lam[p] = st->lam_host[p];
            invg[p] = 1.0 / (lam[p] * lam[p] / st->beta_host[p]);   // 1 / gamma, gamma = lam^2 / beta
        }
        kb_forward aug = make_aug(fw, 1.0);
        validate_fw(&aug);
        Arena a(ws, ws_bytes);
        SbBatchWs w;
        sbb_layout(&aug, B, a, &w);
        cudaStream_t s = as_stream(stream);
        const int64_t N = aug.n, P = (int64_t)aug.side * (aug.side - 1), T = fwd_rows(&aug);
        const int n = aug.side;
        // pinned mailbox: [4B + 8 doubles: reductions] [B * C_COUNT ints: CGLS control] [B ints: active flags]
        const size_t ctl_d = ((size_t)B * C_COUNT + 1) / 2 + 8, act_d = ((size_t)B + 1) / 2 + 8;
        double* hp = pinned_doubles(4 * (size_t)B + 8 + ctl_d + act_d);
        int* hc = reinterpret_cast<int*>(hp + 4 * B + 8);
        int* hact = reinterpret_cast<int*>(hp + 4 * B + 8 + ctl_d);
        KB_CUDA(cudaMemsetAsync(w.mr.counter, 0, sizeof(unsigned) * ((size_t)B + 64), s));
        KB_CUDA(cudaMemcpyAsync(w.lam, lam.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
        KB_CUDA(cudaMemcpyAsync(w.inv_gamma, invg.data(), sizeof(double) * B, cudaMemcpyHostToDevice, s));
        std::vector<int> active(B, 1);
        for (int p = 0; p < B; ++p) hact[p] = 1;
        KB_CUDA(cudaMemcpyAsync(w.active, hact, sizeof(int) * B, cudaMemcpyHostToDevice, s));
        // x_prev = b; d = g = 0  (splitbregman.py:158-162), per problem
        double* xprev = w.xa;
        double* xcur = w.xb;
        map_reduce_b<0>(N, BFCopy{xprev, b, N, N, 0, nullptr}, w.mr, nullptr, 0, s);
        KB_CUDA(cudaMemsetAsync(w.ddx, 0, sizeof(double) * 4 * (size_t)B * P, s));   // ddx..gy are contiguous
        double obs = 0.0, xt_norm = 1.0;
        if (x_true) {
            MR mr1{w.mr.part, w.mr.counter};
            map_reduce<2>(N, FNorm2{b, x_true, N}, mr1, w.red, s);
            KB_CUDA(cudaMemcpyAsync(hp, w.red, sizeof(double) * 2, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            obs = std::sqrt(hp[0]);
            xt_norm = std::sqrt(hp[1]);
            KB_REQUIRE(xt_norm != 0.0, "relative_error is undefined for a zero reference");
        }
        for (int p = 0; p < B; ++p) {
            st->outer_iters_host[p] = 0;
            st->stop_host[p] = KB_SB_MAX_ITER;
        }
        CglsPlanB cp{&aug, B, w.rhs, nullptr, nullptr, &w, {}};
        cp.ctl.h = w.ctl;
        cp.ctl.rc = w.rc;
        cp.ctl.res = w.res;
        cp.ctl.scal = w.scal;
        cp.ctl.active = w.active;
        cp.ctl.any = w.any;
        cp.ctl.nprob = B;
        cp.ctl.i_max = st->i_max;
        cp.ctl.tau = st->tau_cgls;
        std::vector<int> hctl((size_t)B * C_COUNT);
        int n_active = B;
        for (int l = 0; l < st->l_max && n_active > 0; ++l) {
            map_reduce_b<0>(T, BFRhs{w.rhs, b, w.ddx, w.ddy, w.gx, w.gy, N, P, T, w.lam, w.active}, w.mr, nullptr,
                            0, s);
            cp.x0 = st->warm_start ? xprev : nullptr;
            cp.x = xcur;
            cglsb_core(cp, hc, s);
            for (int p = 0; p < B; ++p)
                if (active[p] && hc[p * C_COUNT + C_ERR]) {
                    set_error("CGLS produced non-finite residual quantities (problem %d)", p);
                    throw Fail{KB_ENUMERICAL};
                }
            std::memcpy(hctl.data(), hc, sizeof(int) * (size_t)B * C_COUNT);
            map_reduce_b<3>(N, BFSbUpd{xcur, xprev, x_true, w.ddx, w.ddy, w.gx, w.gy, N, P, n, w.inv_gamma,
                                       st->variant == KB_SB_ISOTROPIC, w.active},
                            w.mr, w.red, 4, s);
            KB_CUDA(cudaMemcpyAsync(hp, w.red, sizeof(double) * 4 * B, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            bool changed = false;
            for (int p = 0; p < B; ++p) {
                if (!active[p]) continue;
                const double* r = hp + 4 * p;
                st->outer_iters_host[p]++;
                if (st->cgls_iters_host) st->cgls_iters_host[(int64_t)p * st->l_max + l] = hctl[p * C_COUNT + C_ITERS];
                if (r[1] == 0.0) {
                    set_error("relative_change is undefined for a zero previous iterate (problem %d)", p);
                    throw Fail{KB_EVALIDATION};
                }
                const double rc = std::sqrt(r[0]) / std::sqrt(r[1]);
                if (st->rc_host) st->rc_host[(int64_t)p * st->l_max + l] = rc;
                if (x_true) {
                    const double err = std::sqrt(r[2]);
                    if (st->re_host) st->re_host[(int64_t)p * st->l_max + l] = err / xt_norm;
                    double isnr;
                    if (err == 0.0 && obs == 0.0) isnr = 0.0;
                    else if (err == 0.0) isnr = INFINITY;
                    else if (obs == 0.0) isnr = -INFINITY;
                    else isnr = 20.0 * std::log10(obs / err);
                    if (st->isnr_host) st->isnr_host[(int64_t)p * st->l_max + l] = isnr;
                }
                if (rc < st->tau) {   // converged: its result is this outer iterate (x_prev after the swap)
                    st->stop_host[p] = KB_SB_CONVERGED;
                    KB_CUDA(cudaMemcpyAsync(x + (int64_t)p * N, xcur + (int64_t)p * N, sizeof(double) * N,
                                            cudaMemcpyDeviceToDevice, s));
                    active[p] = 0;
                    hact[p] = 0;
                    --n_active;
                    changed = true;
                }
            }
            std::swap(xprev, xcur);
            if (changed) KB_CUDA(cudaMemcpyAsync(w.active, hact, sizeof(int) * B, cudaMemcpyHostToDevice, s));
        }
        // problems that ran to l_max: result = x_prev
        for (int p = 0; p < B; ++p)
            if (active[p])
                KB_CUDA(cudaMemcpyAsync(x + (int64_t)p * N, xprev + (int64_t)p * N, sizeof(double) * N,
                                        cudaMemcpyDeviceToDevice, s));
        KB_CUDA(cudaStreamSynchronize(s));
    })
}
