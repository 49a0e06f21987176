// FP64 GEMM on the sm_100a FP64 tensor pipe (DMMA m8n8k4), for the
// Kronecker-sum apply of the split-Bregman inner loop (kronop.py:58-84).
//
// tcgen05 has no f64 kind, so FP64 tensor-core work on Blackwell goes through
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4).  The kernel computes
//     C_z = sum_{s < nseg} op(A_{z,s}) op(B_{z,s})  (+ beta C_z),  z < nbatch
// which covers both Kronecker stages: a batched stage (nbatch = k terms) and
// a segment-reduced stage (nseg = k terms summed into one output, i.e. one
// GEMM with inner dimension k*n1).  Row-major operands; trans flags select
// the smem staging layout so fragment reads are bank-conflict free.
//
// Tile configurations below (default: 128 x 64 x 16, 8 warps of 32 x 32,
// 3-stage cp.async ring, zero-filled edges for any M, N, K, ld).
#include <algorithm>
#include <cstdlib>

#include <cublas_v2.h>

#include "kb_common.cuh"

namespace kb {

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 8 : 0;
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, bool pred) {
    const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
    const int sz = pred ? 16 : 0;
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Tile configuration: CTA tile BM x BN x BK, STAGES-deep cp.async ring,
// WM x WN warps each owning a (BM/WM) x (BN/WN) accumulator tile of 8x8 DMMA
// blocks.  Padding keeps the 64-bit fragment reads bank-conflict free.
template <int BM_, int BN_, int BK_, int ST_, int WM_, int WN_, int MINB_>
struct GCfg {
    static constexpr int BM = BM_, BN = BN_, BK = BK_, STAGES = ST_, WM = WM_, WN = WN_, MINB = MINB_;
    static constexpr int THREADS = WM * WN * 32;
    static constexpr int WTM = BM / WM, WTN = BN / WN, MI = WTM / 8, NI = WTN / 8;
    static constexpr int PAD = 4;
    template <bool TA>
    struct A {
        static constexpr int rows = TA ? BK : BM;
        static constexpr int ld = TA ? (BM + PAD) : (BK + PAD);
        static constexpr int size = rows * ld;
    };
    template <bool TB>
    struct B {
        static constexpr int rows = TB ? BN : BK;
        static constexpr int ld = TB ? (BK + PAD) : (BN + PAD);
        static constexpr int size = rows * ld;
    };
    template <bool TA, bool TB>
    static constexpr size_t smem() { return sizeof(double) * STAGES * (A<TA>::size + B<TB>::size); }
};

// V16: operands 16-byte aligned with even leading dims and even M/N/K, so
// tiles move as 16-byte cp.async chunks (half the LSU ops of the 8-byte path).
// Split-K: blockIdx.z = batch * splits + split; split s handles k-tiles
// [s*T/splits, (s+1)*T/splits) and writes its own partial C (reduced later).
template <class CF, bool TA, bool TB, bool V16>
__global__ void __launch_bounds__(CF::THREADS, CF::MINB)
k_dgemm(int M, int N, int K, const double* __restrict__ A, int64_t lda, int64_t sa_batch,
        int64_t sa_seg, const double* __restrict__ B, int64_t ldb, int64_t sb_batch,
        int64_t sb_seg, double* __restrict__ C, int64_t ldc, int64_t sc_batch, int nseg,
        double beta, int splits, int64_t split_stride, GemmSkip skip) {
    constexpr int BM = CF::BM, BN = CF::BN, BK = CF::BK, STAGES = CF::STAGES, THREADS = CF::THREADS;
    constexpr int MI = CF::MI, NI = CF::NI;
    using AL = typename CF::template A<TA>;
    using BL = typename CF::template B<TB>;
    static_assert((BM * BK) % (2 * THREADS) == 0 && (BK * BN) % (2 * THREADS) == 0, "tile/threads mismatch");
    extern __shared__ __align__(16) double smem[];
    double* As = smem;                       // [STAGES][AL::size]
    double* Bs = smem + STAGES * AL::size;   // [STAGES][BL::size]

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int wm = warp % CF::WM, wn = warp / CF::WM;
    const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
    const int z = blockIdx.z / splits, split = blockIdx.z - z * splits;
    if (skip.flags) {   // batched solves: tiles of inactive problems do no work
        if (skip.rows > 0) {
            bool any = false;
            for (int p = m0 / skip.rows; p <= min(M - 1, m0 + BM - 1) / skip.rows; ++p) any |= skip.flags[p * skip.stride] != 0;
            if (!any) return;
        } else if (!skip.flags[z * skip.stride]) {
            return;
        }
    }
    const double* Ab = A + (int64_t)z * sa_batch;
    const double* Bb = B + (int64_t)z * sb_batch;
    double* Cb = C + (int64_t)z * sc_batch + (int64_t)split * split_stride;

    int kt_first = 0, ktiles = (K + BK - 1) / BK;
    if (skip.band || skip.band_a) {   // banded operand: only the k tiles that meet this CTA's columns (B) / rows (A)
        const int* bp = skip.band ? skip.band : skip.band_a;
        const int lo0 = __ldg(bp), hi0 = __ldg(bp + 1);
        if (lo0 > hi0) {   // all-zero blocks (band left at {INT_MAX, INT_MIN}): nothing to multiply
            kt_first = 0;
            ktiles = 0;
        } else {
            // offsets are within (-K, K): 64-bit bounds keep the arithmetic defined anyway
            int64_t lo = lo0, hi = hi0, klo, khi;
            if (skip.band) {
                if (TB) { const int64_t t = lo; lo = -hi; hi = -t; }   // logical B[k][c] = G[c][k]
                klo = max((int64_t)0, (int64_t)n0 - hi);
                khi = min((int64_t)K - 1, (int64_t)n0 + BN - 1 - lo);
            } else {
                if (TA) { const int64_t t = lo; lo = -hi; hi = -t; }   // stored A[k][m]: k - m in [-hi, -lo]
                klo = max((int64_t)0, (int64_t)m0 + lo);               // logical A[m][k]: k - m in [lo, hi]
                khi = min((int64_t)K - 1, (int64_t)m0 + BM - 1 + hi);
            }
            kt_first = khi >= klo ? (int)(klo / BK) : 0;
            ktiles = khi >= klo ? (int)(khi / BK) + 1 - kt_first : 0;
        }
    }
    const int Ttot = ktiles * nseg;
    const int t_begin = (int)((int64_t)Ttot * split / splits);
    const int T = (int)((int64_t)Ttot * (split + 1) / splits) - t_begin;

    auto load_tile = [&](int stage, int tt) {
        const int t = tt + t_begin;
        const int s = t / ktiles;
        const int k0 = (t - s * ktiles + kt_first) * BK;
        const double* Ap = Ab + (int64_t)s * sa_seg;
        const double* Bp = Bb + (int64_t)s * sb_seg;
        double* as = As + stage * AL::size;
        double* bs = Bs + stage * BL::size;
        if constexpr (V16) {
#pragma unroll
            for (int r = 0; r < (BM * BK) / (2 * THREADS); ++r) {
                const int idx = tid + r * THREADS;
                int i, j;
                if (!TA) { i = idx / (BK / 2); j = (idx % (BK / 2)) * 2; } else { j = idx / (BM / 2); i = (idx % (BM / 2)) * 2; }
                const int gm = m0 + i, gk = k0 + j;
                const bool ok = (gm < M) && (gk < K);
                const double* src = TA ? (Ap + (int64_t)(ok ? gk : 0) * lda + (ok ? gm : 0))
                                       : (Ap + (int64_t)(ok ? gm : 0) * lda + (ok ? gk : 0));
                double* dst = TA ? (as + j * AL::ld + i) : (as + i * AL::ld + j);
                cp_async16(dst, src, ok);
            }
#pragma unroll
            for (int r = 0; r < (BK * BN) / (2 * THREADS); ++r) {
                const int idx = tid + r * THREADS;
                int j, c;
                if (!TB) { j = idx / (BN / 2); c = (idx % (BN / 2)) * 2; } else { c = idx / (BK / 2); j = (idx % (BK / 2)) * 2; }
                const int gk = k0 + j, gn = n0 + c;
                const bool ok = (gk < K) && (gn < N);
                const double* src = TB ? (Bp + (int64_t)(ok ? gn : 0) * ldb + (ok ? gk : 0))
                                       : (Bp + (int64_t)(ok ? gk : 0) * ldb + (ok ? gn : 0));
                double* dst = TB ? (bs + c * BL::ld + j) : (bs + j * BL::ld + c);
                cp_async16(dst, src, ok);
            }
        } else {
#pragma unroll
            for (int r = 0; r < (BM * BK) / THREADS; ++r) {
                const int idx = tid + r * THREADS;
                int i, j;
                if (!TA) { i = idx / BK; j = idx % BK; } else { j = idx / BM; i = idx % BM; }
                const int gm = m0 + i, gk = k0 + j;
                const bool ok = (gm < M) && (gk < K);
                const double* src = TA ? (Ap + (int64_t)(ok ? gk : 0) * lda + (ok ? gm : 0))
                                       : (Ap + (int64_t)(ok ? gm : 0) * lda + (ok ? gk : 0));
                double* dst = TA ? (as + j * AL::ld + i) : (as + i * AL::ld + j);
                cp_async8(dst, src, ok);
            }
#pragma unroll
            for (int r = 0; r < (BK * BN) / THREADS; ++r) {
                const int idx = tid + r * THREADS;
                int j, c;
                if (!TB) { j = idx / BN; c = idx % BN; } else { c = idx / BK; j = idx % BK; }
                const int gk = k0 + j, gn = n0 + c;
                const bool ok = (gk < K) && (gn < N);
                const double* src = TB ? (Bp + (int64_t)(ok ? gn : 0) * ldb + (ok ? gk : 0))
                                       : (Bp + (int64_t)(ok ? gk : 0) * ldb + (ok ? gn : 0));
                double* dst = TB ? (bs + c * BL::ld + j) : (bs + j * BL::ld + c);
                cp_async8(dst, src, ok);
            }
        }
    };

    double acc[MI][NI][2];
#pragma unroll
    for (int a = 0; a < MI; ++a)
#pragma unroll
        for (int b = 0; b < NI; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

#pragma unroll
    for (int s = 0; s < STAGES - 1; ++s) {
        if (s < T) load_tile(s, s);
        cp_async_commit();
    }

    const int gid = lane >> 2, tig = lane & 3;
    for (int t = 0; t < T; ++t) {
        cp_async_wait<STAGES - 2>();
        __syncthreads();
        {
            const int nt = t + STAGES - 1;
            if (nt < T) load_tile(nt % STAGES, nt);
            cp_async_commit();
        }
        const double* as = As + (t % STAGES) * AL::size;
        const double* bs = Bs + (t % STAGES) * BL::size;
#pragma unroll
        for (int kk = 0; kk < BK; kk += 4) {
            double af[MI], bf[NI];
#pragma unroll
            for (int mi = 0; mi < MI; ++mi) {
                const int mm = wm * CF::WTM + mi * 8 + gid, k = kk + tig;
                af[mi] = TA ? as[k * AL::ld + mm] : as[mm * AL::ld + k];
            }
#pragma unroll
            for (int ni = 0; ni < NI; ++ni) {
                const int nn = wn * CF::WTN + ni * 8 + gid, k = kk + tig;
                bf[ni] = TB ? bs[nn * BL::ld + k] : bs[k * BL::ld + nn];
            }
#pragma unroll
            for (int mi = 0; mi < MI; ++mi)
#pragma unroll
                for (int ni = 0; ni < NI; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
    }
    cp_async_wait<0>();

#pragma unroll
    for (int mi = 0; mi < MI; ++mi) {
        const int gm = m0 + wm * CF::WTM + mi * 8 + gid;
        if (gm >= M) continue;
#pragma unroll
        for (int ni = 0; ni < NI; ++ni) {
            const int gn = n0 + wn * CF::WTN + ni * 8 + 2 * tig;
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                if (gn + q < N) {
                    double* cp = Cb + (int64_t)gm * ldc + gn + q;
                    *cp = (beta != 0.0) ? (acc[mi][ni][q] + beta * *cp) : acc[mi][ni][q];
                }
            }
        }
    }
}

__global__ void k_split_reduce(const double* __restrict__ part, int splits, int64_t split_stride, int M,
                               int N, double* __restrict__ C, int64_t ldc, int64_t sc_batch, int nbatch,
                               double beta, GemmSkip skip) {
    const int64_t per = (int64_t)M * N, total = per * nbatch;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total;
         e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t z = e / per, rem = e - z * per;
        if (skip.flags && skip.rows == 0 && !skip.flags[z * skip.stride]) continue;
        const int64_t i = rem / N, j = rem - i * N;
        const double* p = part + z * sc_batch + i * ldc + j;   // partials share C's layout
        double s = 0.0;
        for (int q = 0; q < splits; ++q) s += p[(int64_t)q * split_stride];
        double* c = C + z * sc_batch + i * ldc + j;
        *c = (beta != 0.0) ? (s + beta * *c) : s;
    }
}

// Tile configurations (selected by kb_dgemm_config / KB_DGEMM_CFG for tuning).
using Cfg0 = GCfg<128, 64, 16, 3, 4, 2, 2>;    // 8 warps of 32x32, 2 CTAs/SM
using Cfg1 = GCfg<128, 64, 32, 2, 4, 2, 2>;    // BK 32: half the barriers per flop
using Cfg2 = GCfg<128, 128, 16, 3, 2, 4, 1>;   // 8 warps of 64x32, 1 CTA/SM
using Cfg3 = GCfg<128, 128, 32, 2, 2, 4, 1>;
// narrow tiles along the banded dimension for the Toeplitz-split operator (bands of +-24 / +-31
// at n = 1024): the k window of a tile is band + tile extent wide, so a 32-row (A band) or
// 32-column (B band) tile executes well under half the k tiles of the default shape
using CfgNA = GCfg<32, 128, 16, 2, 1, 4, 5>;   // banded A: 4 warps of 32x32 (64-row tiles: 7 % slower; 3 stages: 5 % slower,
                                               // fewer CTAs per SM)
using CfgNB = GCfg<128, 32, 16, 2, 4, 1, 4>;   // banded B: 4 warps of 32x32 (16-column tiles: no better)
int g_dgemm_narrow = 0;   // set by kron_apply for operators with kb_kron.fband
static int g_dgemm_cfg = -1;
int g_dgemm_split_per_batch = 0;
GemmSkip g_dgemm_skip;   // set around the batched-solve GEMMs (kb_sb.cu), empty otherwise

template <class CF, bool TA, bool TB, bool V16>
static void launch_dgemm(int m, int n, int k, const double* A, int64_t lda, int64_t sa_b,
                         int64_t sa_s, const double* B, int64_t ldb, int64_t sb_b, int64_t sb_s,
                         double* C, int64_t ldc, int64_t sc_b, int nbatch, int nseg, double beta,
                         int splits, double* part, int64_t split_stride, cudaStream_t st) {
    const size_t smem = CF::template smem<TA, TB>();
    static bool configured = false;
    if (!configured) {
        KB_CUDA(cudaFuncSetAttribute(k_dgemm<CF, TA, TB, V16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem));
        configured = true;
    }
    dim3 grid((unsigned)cdiv(n, CF::BN), (unsigned)cdiv(m, CF::BM), (unsigned)(nbatch * splits));
    const double nb = (double)nbatch, ns = (double)nseg;
    ProfScope ps(st, PROF_DGEMM, 8.0 * nb * (ns * ((double)m * k + (double)k * n) + (double)m * n),
                 2.0 * m * n * (double)k * nb * ns);
    if (splits == 1) {
        k_dgemm<CF, TA, TB, V16><<<grid, CF::THREADS, smem, st>>>(m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s,
                                                                  C, ldc, sc_b, nseg, beta, 1, 0, g_dgemm_skip);
    } else {
        k_dgemm<CF, TA, TB, V16><<<grid, CF::THREADS, smem, st>>>(m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s,
                                                                  part, ldc, sc_b, nseg, 0.0, splits, split_stride,
                                                                  g_dgemm_skip);
        KB_LAUNCH_CHECK();
        const int64_t total = (int64_t)m * n * nbatch;
        k_split_reduce<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 8 * kSMs), 256, 0, st>>>(
            part, splits, split_stride, m, n, C, ldc, sc_b, nbatch, beta, g_dgemm_skip);
    }
    KB_LAUNCH_CHECK();
}

// Number of K splits so that the grid fills >= 2 waves.
template <class CF>
static int dgemm_splits(int m, int n, int k, int nbatch, int nseg) {
    const int64_t tiles = cdiv(n, CF::BN) * cdiv(m, CF::BM) * (int64_t)nbatch;
    const int64_t ktot = cdiv(k, CF::BK) * (int64_t)nseg;
    int s = 1;
    const int64_t min_tiles_per_split = tiles >= kSMs ? 8 : 1;   // small grids: split down to 1 k-tile
    while (tiles * s < 2 * CF::MINB * kSMs && ktot / (s * 2) >= min_tiles_per_split) s *= 2;
    return s;
}

template <class CF>
static void dgemm_cfg(int ta, int tb, int m, int n, int k, const double* A, int64_t lda, int64_t sa_b,
                      int64_t sa_s, const double* B, int64_t ldb, int64_t sb_b, int64_t sb_s, double* C,
                      int64_t ldc, int64_t sc_b, int nbatch, int nseg, double beta, cudaStream_t st,
                      double* part, int64_t part_doubles) {
    // g_dgemm_split_per_batch: split K exactly as a single batch entry would be
    // split, so each batch entry reproduces the unbatched GEMM bit for bit
    int splits = dgemm_splits<CF>(m, n, k, g_dgemm_split_per_batch ? 1 : nbatch, nseg);
    static const int split_env = std::getenv("KB_DGEMM_SPLITS") ? std::atoi(std::getenv("KB_DGEMM_SPLITS")) : 0;
    if (split_env > 0 && g_dgemm_narrow && g_dgemm_skip.band_a) splits = split_env;   // (tuning)
    const int64_t span = (nbatch - 1) * sc_b + (int64_t)(m - 1) * ldc + n;   // partials use C's layout
    if (part == nullptr) splits = 1;
    while (splits > 1 && (int64_t)splits * span > part_doubles) splits /= 2;
    KB_REQUIRE(nbatch * splits <= 65535, "dgemm: too many batches (%d)", nbatch);
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    const bool v16 = al16(A) && al16(B) && (lda % 2 == 0) && (ldb % 2 == 0) && (sa_b % 2 == 0) &&
                     (sa_s % 2 == 0) && (sb_b % 2 == 0) && (sb_s % 2 == 0) && (m % 2 == 0) &&
                     (n % 2 == 0) && (k % 2 == 0);
#define KB_DG(TA_, TB_)                                                                                    \
    do {                                                                                                   \
        if (v16)                                                                                           \
            launch_dgemm<CF, TA_, TB_, true>(m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, \
                                             nbatch, nseg, beta, splits, part, span, st);                  \
        else                                                                                               \
            launch_dgemm<CF, TA_, TB_, false>(m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc,     \
                                              sc_b, nbatch, nseg, beta, splits, part, span, st);          \
    } while (0)
    if (!ta && !tb) KB_DG(false, false);
    else if (!ta && tb) KB_DG(false, true);
    else if (ta && !tb) KB_DG(true, false);
    else KB_DG(true, true);
#undef KB_DG
}

void dgemm(int ta, int tb, int m, int n, int k, const double* A, int64_t lda, int64_t sa_b,
           int64_t sa_s, const double* B, int64_t ldb, int64_t sb_b, int64_t sb_s, double* C,
           int64_t ldc, int64_t sc_b, int nbatch, int nseg, double beta, cudaStream_t st,
           double* part, int64_t part_doubles) {
    KB_REQUIRE(m >= 0 && n >= 0 && k >= 0 && nbatch >= 1 && nseg >= 1, "dgemm: bad sizes");
    if (m == 0 || n == 0) return;
    if (g_dgemm_cfg < 0) {
        const char* e = std::getenv("KB_DGEMM_CFG");
        g_dgemm_cfg = e ? std::atoi(e) : 1;   // Cfg1 measured best on B200 (tools/gemm_bench.py)
    }
    static const int narrow_env = std::getenv("KB_DGEMM_NARROW") ? std::atoi(std::getenv("KB_DGEMM_NARROW")) : 3;
    if (g_dgemm_narrow && g_dgemm_skip.band_a && (narrow_env & 1)) {
        dgemm_cfg<CfgNA>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles);
        return;
    }
    if (g_dgemm_narrow && g_dgemm_skip.band && !g_dgemm_skip.flags && (narrow_env & 2)) {
        dgemm_cfg<CfgNB>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles);
        return;
    }
    switch (g_dgemm_cfg) {
        default: dgemm_cfg<Cfg1>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles); break;
        case 2: dgemm_cfg<Cfg2>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles); break;
        case 3: dgemm_cfg<Cfg3>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles); break;
        case 0: dgemm_cfg<Cfg0>(ta, tb, m, n, k, A, lda, sa_b, sa_s, B, ldb, sb_b, sb_s, C, ldc, sc_b, nbatch, nseg, beta, st, part, part_doubles); break;
    }
}

}  // namespace kb


namespace kb {
// ---- the dense reduced stage of the Kronecker apply on cuBLAS DGEMM --------------
// Y (r x c, row-major) = sum_{i < nblk} Bl_i^T P_i, Bl_i (kin x r) and P_i (kin x c)
// contiguous row-major blocks: ONE GEMM with inner dimension nblk * kin.  cuBLAS
// (35 TF/s on these shapes, profiles/gemm_cublas_r02.txt) beats our DMMA split-K
// kernel (25 TF/s) here; the banded G stage stays on k_dgemm, which skips the
// all-zero tiles cuBLAS would multiply.  Column-major view: Y^T = P^T Bl.
namespace {
struct Cublas {
    cublasHandle_t h = nullptr;
    void* ws = nullptr;
};
Cublas& cublas_state() {
    static thread_local Cublas c[16];
    int dev = 0;
    cudaGetDevice(&dev);
    return c[dev & 15];
}
}  // namespace

void cublas_prepare() {
    Cublas& c = cublas_state();
    if (c.h) return;
    if (cublasCreate(&c.h) != CUBLAS_STATUS_SUCCESS) {
        set_error("cublasCreate failed");
        throw Fail{KB_ERUNTIME};
    }
    constexpr size_t WS = 32u << 20;
    KB_CUDA(cudaMalloc(&c.ws, WS));
    cublasSetWorkspace(c.h, c.ws, WS);
    cublasSetMathMode(c.h, CUBLAS_DEFAULT_MATH);
}

void dgemm_sum_blocks(int r, int c, int kin, int nblk, const double* Bl, const double* P, double* Y,
                      cudaStream_t st) {
    cublas_prepare();
    Cublas& cb = cublas_state();
    cublasSetStream(cb.h, st);
    const double one = 1.0, zero = 0.0;
    const int64_t K = (int64_t)kin * nblk;
    KB_REQUIRE(K < (1ll << 31), "dgemm_sum_blocks: inner dimension too large");
    ProfScope ps(st, PROF_DGEMM, 8.0 * ((double)K * (r + c) + (double)r * c), 2.0 * r * (double)c * (double)K);
    const cublasStatus_t e = cublasDgemm(cb.h, CUBLAS_OP_N, CUBLAS_OP_T, c, r, (int)K, &one, P, c, Bl, r, &zero, Y, c);
    if (e != CUBLAS_STATUS_SUCCESS) {
        set_error("cublasDgemm failed (%d)", (int)e);
        throw Fail{KB_ERUNTIME};
    }
}
}  // namespace kb
