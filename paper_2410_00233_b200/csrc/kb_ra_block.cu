// One-launch R(A) product for a block of vectors (cooperative, sm_100a).
//
//   Y = R(A) X  (or R(A)^T X),  X, Y: nv vectors of length n^2
//
// R(A) = P_c K^T P_r^T: per vector, diagonal sums of the
// n x n image (w), a small GEMV with K (z = K^T w), and a Toeplitz broadcast
// y[a*n+b] = z[b - a + c]; the reflexive BC adds anti-diagonal sums and the
// two Hankel broadcast families (kb_ops.cuh ra_gather_rows / ra_bcast).  The three steps are phases of ONE cooperative
// kernel separated by grid barriers; K is read once for the whole block (the
// RSVD block products, lowrank.py:361-369, and the standalone product
// lowrank.py:211,238,250 with nv = 1).  Fixed-order reductions throughout.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "kb_ops.cuh"

namespace cg = cooperative_groups;

namespace kb {

constexpr int RB_THREADS = 256;
constexpr int RB_SEGS = 8;
constexpr int RB_MAXV = 16;

struct RaBlockParams {
    const void* X;
    void* Y;
    int64_t ldx, ldy;
    int nv;
    const void* M;     // Li x Lo row-major (K for the forward product, K^T for the transpose)
    int n, ci, Li, co, Lo, lmax;
    double* diag_part; // [RB_SEGS][nv][lmax]
    double* w;         // [nv][lmax]
    double* col_part;  // [RB_SEGS][nv][lmax]
    unsigned long long* dbg;   // optional phase timestamps (KB_PK_TRACE)
    int zlen;
    int refl;          // reflexive BC: Hankel index families too
};

__device__ __forceinline__ void rb_mark(const RaBlockParams& P, int slot) {
    if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        P.dbg[slot] = t;
    }
}

template <typename T>
__global__ void __launch_bounds__(RB_THREADS, 2) k_ra_block(RaBlockParams P) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    double* zs = sm;                       // [zlen]: z (phase 3) / staged w (phase 2)
    double* acc = sm + P.zlen;             // [8][33 * RB_MAXV]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n, nv = P.nv, L = P.lmax;
    const int nblk = gridDim.x;
    const T* X = static_cast<const T*>(P.X);
    T* Y = static_cast<T*>(P.Y);
    const T* M = static_cast<const T*>(P.M);
    rb_mark(P, 0);

    // ---- phase 1: diagonal-sum partials, items = (32-diagonal chunk, row segment)
    {
        // items = (vector, 32-diagonal chunk, row segment): the vectors of a block
        // are spread over the grid instead of being summed one after another
        const int chunks = (P.Li + 31) / 32;
        const int items = chunks * RB_SEGS;
        for (int itv = blockIdx.x; itv < items * nv; itv += nblk) {
            const int it = itv % items, v = itv / items;
            const int c = it % chunks, seg = it / chunks;
            const int u = c * 32 + lane;
            const int s0 = (int)((int64_t)n * seg / RB_SEGS), s1 = (int)((int64_t)n * (seg + 1) / RB_SEGS);
            {
                double a = 0.0;
                if (u < P.Li)
                    a = ra_gather_rows<T, false, 16>(X + (int64_t)v * P.ldx, n, u, P.ci, s0, s1, warp,
                                                     P.refl != 0);
                acc[warp * 33 + lane] = a;
                __syncthreads();
                if (warp == 0 && u < P.Li) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) t += acc[w * 33 + lane];
                    P.diag_part[((int64_t)seg * nv + v) * L + u] = t;
                }
                __syncthreads();
            }
        }
    }
    grid.sync();
    rb_mark(P, 1);
    // ---- phase 1b (nv > 1): w[v][u] = sum_seg diag_part[seg][v][u], fixed order
    if (nv > 1) {
        for (int64_t e = blockIdx.x * (int64_t)RB_THREADS + tid; e < (int64_t)nv * P.Li;
             e += (int64_t)nblk * RB_THREADS) {
            const int v = (int)(e / P.Li), u = (int)(e - (int64_t)v * P.Li);
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < RB_SEGS; ++q) t += __ldcg(P.diag_part + ((int64_t)q * nv + v) * L + u);
            P.w[(int64_t)v * L + u] = t;
        }
        grid.sync();
    }
    // ---- phase 2: K column-sum partials, items = (32-column chunk, row segment); K read once
    {
        const int chunks = (P.Lo + 31) / 32;
        const int items = chunks * RB_SEGS;
        for (int it = blockIdx.x; it < items; it += nblk) {
            const int cc = it % chunks, seg = it / chunks;
            const int c = cc * 32 + lane;
            const int r0 = (int)((int64_t)P.Li * seg / RB_SEGS), r1 = (int)((int64_t)P.Li * (seg + 1) / RB_SEGS);
            // stage w (fixed-order sum of the segment partials) for these rows in smem
            double* ws = zs;   // [(r1 - r0) * nv], reuses the z buffer (phase 3 runs after a barrier)
            for (int j = tid; j < (r1 - r0) * nv; j += RB_THREADS) {
                const int rr = j / nv, v = j - rr * nv;
                double t = 0.0;
                if (nv == 1) {
#pragma unroll
                    for (int q = 0; q < RB_SEGS; ++q) t += __ldcg(P.diag_part + (int64_t)q * L + r0 + rr);
                } else {
                    t = __ldcg(P.w + (int64_t)v * L + r0 + rr);
                }
                ws[j] = t;
            }
            __syncthreads();
            double a[RB_MAXV];
#pragma unroll
            for (int v = 0; v < RB_MAXV; ++v) a[v] = 0.0;
            int r = r0 + warp;
            for (; r + 120 < r1; r += 128) {          // 16 independent K loads in flight
                T mk[16];
#pragma unroll
                for (int k = 0; k < 16; ++k) mk[k] = (c < P.Lo) ? __ldg(M + (int64_t)(r + 8 * k) * P.Lo + c) : T(0);
#pragma unroll
                for (int k = 0; k < 16; ++k) {
                    const double* wr = ws + (r + 8 * k - r0) * nv;
#pragma unroll
                    for (int v = 0; v < RB_MAXV; ++v)
                        if (v < nv) a[v] += mk[k] * wr[v];
                }
            }
            for (; r < r1; r += 8) {
                const double mk = (c < P.Lo) ? (double)__ldg(M + (int64_t)r * P.Lo + c) : 0.0;
                const double* wr = ws + (r - r0) * nv;
#pragma unroll
                for (int v = 0; v < RB_MAXV; ++v)
                    if (v < nv) a[v] += mk * wr[v];
            }
#pragma unroll
            for (int v = 0; v < RB_MAXV; ++v)
                if (v < nv) acc[warp * (33 * RB_MAXV) + v * 33 + lane] = a[v];
            __syncthreads();
            for (int j = tid; j < nv * 32; j += RB_THREADS) {
                const int v = j >> 5, l = j & 31, col = cc * 32 + l;
                if (col < P.Lo) {
                    double t = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) t += acc[w * (33 * RB_MAXV) + v * 33 + l];
                    P.col_part[((int64_t)seg * nv + v) * L + col] = t;
                }
            }
            __syncthreads();
        }
    }
    grid.sync();
    rb_mark(P, 2);
    // ---- phase 3: z_v into shared memory, Toeplitz broadcast into y_v.  With
    // several vectors the grid is split into nv groups of blocks (block b writes
    // vector b % nv), so each block stages one z and the vectors are written
    // concurrently.
    const int64_t N = (int64_t)n * n;
    const int groups = nv <= nblk ? nv : 1;
    const int gsize = nblk / groups;                      // blocks per vector group
    const int gid = blockIdx.x % groups, grank = blockIdx.x / groups;
    const bool active = grank < gsize;                    // leftover blocks sit out
    for (int v = (groups > 1 ? gid : 0); v < nv; v += (groups > 1 ? nv : 1)) {
        for (int c = tid; c < P.Lo; c += RB_THREADS) {
            double t = 0.0;
#pragma unroll
            for (int q = 0; q < RB_SEGS; ++q) t += __ldcg(P.col_part + ((int64_t)q * nv + v) * L + c);
            zs[c] = t;
        }
        __syncthreads();
        T* y = Y + (int64_t)v * P.ldy;
        const int64_t nb = groups > 1 ? gsize : nblk;
        const int64_t bi = groups > 1 ? grank : blockIdx.x;
        for (int64_t e0 = (bi * RB_THREADS + tid) * 4; active && e0 < N; e0 += nb * RB_THREADS * 4) {
            T o[4];
            if (e0 + 4 <= N) {
                double yv[4];
                ra_bcast4(zs, (unsigned)e0, n, P.co, P.Lo, P.refl != 0, yv);
#pragma unroll
                for (int q = 0; q < 4; ++q) o[q] = (T)yv[q];
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int64_t e = e0 + q;
                    o[q] = e < N ? (T)ra_bcast(zs, (unsigned)e, n, P.co, P.Lo, P.refl != 0) : T(0);
                }
            }
            if (e0 + 4 <= N && ((P.ldy & 3) == 0)) {
                if constexpr (sizeof(T) == 4) {
                    *reinterpret_cast<float4*>(y + e0) = make_float4(o[0], o[1], o[2], o[3]);
                } else {
                    *reinterpret_cast<double2*>(y + e0) = make_double2(o[0], o[1]);
                    *reinterpret_cast<double2*>(y + e0 + 2) = make_double2(o[2], o[3]);
                }
            } else {
                for (int q = 0; q < 4; ++q)
                    if (e0 + q < N) y[e0 + q] = o[q];
            }
        }
        __syncthreads();
    }
    rb_mark(P, 3);
}

size_t ra_block_scratch_doubles(int lmax, int nv) {
    return (size_t)(2 * RB_SEGS + 1) * nv * lmax + 64;
}

// Returns false if the cooperative launch is not possible (caller falls back).
bool ra_block_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv,
                    int transpose, double* scratch, cudaStream_t st) {
    if (!ra_is_operator(op->kind) || nv < 1 || nv > RB_MAXV) return false;
    if (((uintptr_t)Y & 15) != 0) return false;
    RaBlockParams P{};
    const int cu = op->kh / 2, cv = op->kw / 2;
    P.X = X;
    P.Y = Y;
    P.ldx = ldx;
    P.ldy = ldy;
    P.nv = nv;
    P.n = op->side;
    P.refl = op->kind == KB_OP_RA_REFLEXIVE;
    if (!transpose) { P.ci = cu; P.Li = op->kh; P.co = cv; P.Lo = op->kw; P.M = op->k; }
    else { P.ci = cv; P.Li = op->kw; P.co = cu; P.Lo = op->kh; P.M = op->kt; }
    P.lmax = std::max(op->kh, op->kw);
    P.diag_part = scratch;
    P.w = scratch + (size_t)RB_SEGS * nv * P.lmax;
    P.col_part = P.w + (size_t)nv * P.lmax;
    P.zlen = std::max(P.lmax, (int)((P.Li + RB_SEGS - 1) / RB_SEGS + 1) * nv);
    const size_t smem = sizeof(double) * ((size_t)P.zlen + 8 * 33 * RB_MAXV);
    KB_REQUIRE(smem <= 100 * 1024, "R(A) block product: PSF support too large");
    static unsigned long long* dbg = nullptr;
    static const bool trace = std::getenv("KB_PK_TRACE") != nullptr;
    if (trace && !dbg) KB_CUDA(cudaMalloc(&dbg, 8 * sizeof(unsigned long long)));
    P.dbg = trace ? dbg : nullptr;
    struct Dump {
        unsigned long long* d; cudaStream_t s;
        ~Dump() {
            if (!d) return;
            unsigned long long t[4];
            cudaMemcpyAsync(t, d, sizeof(t), cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            fprintf(stderr, "[kb] ra_block phases (us): %.2f %.2f %.2f\n", (t[1] - t[0]) * 1e-3,
                    (t[2] - t[1]) * 1e-3, (t[3] - t[2]) * 1e-3);
        }
    } dump{trace ? dbg : nullptr, st};
    const int64_t N = (int64_t)P.n * P.n;
    const double bytes = (double)(op->dtype == KB_F32 ? 4 : 8) * (2.0 * nv * N + (double)op->kh * op->kw);
    ProfScope ps(st, PROF_RA_DIAG, bytes);
    cudaLaunchConfig_t lc = {};
    lc.blockDim = dim3(RB_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    int per_sm = 0;
    if (op->dtype == KB_F32) {
        static bool cfg = false;
        if (!cfg) {
            KB_CUDA(cudaFuncSetAttribute(k_ra_block<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
            cfg = true;
        }
        static size_t smem_q = 0;
        static int per_sm_q = 0;
        if (smem != smem_q) {   // occupancy depends only on the smem size: queried once per size
            KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_q, k_ra_block<float>, RB_THREADS, smem));
            smem_q = smem;
        }
        per_sm = per_sm_q;
        if (per_sm < 1) return false;
        lc.gridDim = dim3(kSMs * std::min(per_sm, 2));
        KB_CUDA(cudaLaunchKernelEx(&lc, k_ra_block<float>, P));
    } else {
        static bool cfg = false;
        if (!cfg) {
            KB_CUDA(cudaFuncSetAttribute(k_ra_block<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
            cfg = true;
        }
        static size_t smem_q = 0;
        static int per_sm_q = 0;
        if (smem != smem_q) {   // occupancy depends only on the smem size: queried once per size
            KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_q, k_ra_block<double>, RB_THREADS, smem));
            smem_q = smem;
        }
        per_sm = per_sm_q;
        if (per_sm < 1) return false;
        lc.gridDim = dim3(kSMs * std::min(per_sm, 2));
        KB_CUDA(cudaLaunchKernelEx(&lc, k_ra_block<double>, P));
    }
    return true;
}

}  // namespace kb
