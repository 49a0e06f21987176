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
#include <cuda.h>
#include <cudaTypedefs.h>

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

size_t ra_tiled_scratch_doubles(int n, int lmax, int nv);
bool ra_tiled_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv, int transpose,
                    double* scratch, cudaStream_t st);

size_t ra_block_scratch_doubles(int n, int lmax, int nv) {
    return std::max((size_t)(2 * RB_SEGS + 1) * nv * lmax + 64, ra_tiled_scratch_doubles(n, lmax, nv));
}

// Returns false if the cooperative launch is not possible (caller falls back).
bool ra_block_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv,
                    int transpose, double* scratch, cudaStream_t st) {
    if (!ra_is_operator(op->kind) || nv < 1 || nv > RB_MAXV) return false;
    static const bool no_tiled = std::getenv("KB_RA_NO_TILED") != nullptr;
    if (!no_tiled && ra_tiled_apply(op, X, ldx, Y, ldy, nv, transpose, scratch, st)) return true;
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

// ------------------------------------------------------------------ tiled block product
// Y = R(A) X (or R(A)^T X) for zero BC and n a multiple of 128, as four
// stream-ordered kernels instead of one cooperative kernel with grid
// barriers (every phase runs at full occupancy, no barrier latency):
//
//   k_rat_diag   tile (32 image rows x 128 columns of one vector) through
//                shared memory -> its 159 diagonal sums (fp64, fixed order)
//   k_rat_w      w[v][u] = sum of the tile sums on diagonal u - c_in, tiles
//                in fixed (row block, column block) order -- deterministic
//   k_rat_z      z[v][c] = sum_r Mt[c, r] w[v][r]: contiguous rows of K^T
//                (forward) or K (transpose), w staged in shared memory,
//                16 rows x <= 16 vectors per CTA
//   k_rat_bcast  y[v][a*n + b] = z[v][b - a + c_out], float4 / double2 stores
//
// The only HBM streams are the n^2 inputs (read once), the n^2 outputs
// (written once) and K (read once per block of vectors): the product's
// algorithmic bytes.
namespace kb {

constexpr int RT_ROWS = 32, RT_COLS = 128, RT_DIAG = RT_ROWS + RT_COLS - 1, RT_DP = 160;

// Programmatic dependent launch: the next kernel of the chain is launched
// while this one drains (launch latency hidden); it waits in pdl_wait()
// until this grid has completed and its writes are visible.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename T>
__global__ void __launch_bounds__(256) k_rat_diag(const T* __restrict__ X, int64_t ldx, int n, double* __restrict__ part) {
    __shared__ T tile[RT_ROWS][RT_COLS + (sizeof(T) == 4 ? 4 : 2)];
    const int cbn = n / RT_COLS, tiles = (n / RT_ROWS) * cbn;
    const int t = blockIdx.x, v = blockIdx.y;
    const int rb = t / cbn, cb = t - rb * cbn;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const T* x = X + (int64_t)v * ldx + (int64_t)(rb * RT_ROWS) * n + cb * RT_COLS;
    if constexpr (sizeof(T) == 4) {
        float4 q[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) q[j] = __ldcs(reinterpret_cast<const float4*>(x + (int64_t)(warp + 8 * j) * n) + lane);
#pragma unroll
        for (int j = 0; j < 4; ++j) *reinterpret_cast<float4*>(&tile[warp + 8 * j][4 * lane]) = q[j];
    } else {
        double2 q[8];
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h)
                q[2 * j + h] = __ldcs(reinterpret_cast<const double2*>(x + (int64_t)(warp + 8 * j) * n + 64 * h) + lane);
#pragma unroll
        for (int j = 0; j < 4; ++j)
#pragma unroll
            for (int h = 0; h < 2; ++h) *reinterpret_cast<double2*>(&tile[warp + 8 * j][64 * h + 2 * lane]) = q[2 * j + h];
    }
    __syncthreads();
    pdl_trigger();
    if (tid < RT_DIAG) {
        const int off = tid - (RT_ROWS - 1);   // column - row inside the tile
        const int r0 = max(0, -off), r1 = min(RT_ROWS, RT_COLS - off);
        double s = 0.0;
        for (int r = r0; r < r1; ++r) s += (double)tile[r][r + off];
        part[((int64_t)v * tiles + t) * RT_DP + tid] = s;
    }
}

// (opt-in, KB_RAT_TMA=1) fp32 inputs: persistent CTAs stream their tiles through a 2-stage shared-memory
// ring, each tile ONE TMA tensor copy (cp.async.bulk.tensor.3d over the [nv][n][n]
// view of X, box 128 x 32 x 1, evict-first, completion on the stage's mbarrier), the
// next tile in flight while this one's diagonal sums are formed.
constexpr int RT_TMA_STAGES = 2;
__global__ void __launch_bounds__(256) k_rat_diag_tma(const __grid_constant__ CUtensorMap map, int n, int nv,
                                                      double* __restrict__ part) {
    __shared__ alignas(128) float tile[RT_TMA_STAGES][RT_ROWS][RT_COLS];
    __shared__ alignas(8) unsigned long long mbar[RT_TMA_STAGES];
    const int cbn = n / RT_COLS, tiles = (n / RT_ROWS) * cbn, total = tiles * nv;
    const int tid = threadIdx.x;
    unsigned long long pol = 0;
    auto issue = [&](int k, int st) {   // thread 0: tile k of this CTA into stage st
        const int id = blockIdx.x + k * gridDim.x;
        if (id >= total) return;
        const int v = id / tiles, t = id - v * tiles, rb = t / cbn, cb = t - rb * cbn;
        const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[st]));
        const unsigned ts = static_cast<unsigned>(__cvta_generic_to_shared(&tile[st][0][0]));
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the stage
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(RT_ROWS * RT_COLS * 4)
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3, %4}], [%5], %6;"
            ::"r"(ts), "l"(reinterpret_cast<unsigned long long>(&map)), "r"(cb * RT_COLS), "r"(rb * RT_ROWS), "r"(v),
            "r"(mb), "l"(pol)
            : "memory");
    };
    if (tid == 0) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int st = 0; st < RT_TMA_STAGES; ++st) {
            const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[st]));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(mb) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        for (int st = 0; st < RT_TMA_STAGES; ++st) issue(st, st);
    }
    __syncthreads();
    for (int k = 0; blockIdx.x + k * gridDim.x < total; ++k) {
        const int st = k % RT_TMA_STAGES;
        const unsigned par = (unsigned)(k / RT_TMA_STAGES) & 1u;
        if (tid == 0) {
            const unsigned mb = static_cast<unsigned>(__cvta_generic_to_shared(&mbar[st]));
            asm volatile(
                "{\n\t.reg .pred P1;\n\t"
                "WAIT_TILE:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
                "@!P1 bra WAIT_TILE;\n\t}" ::"r"(mb), "r"(par)
                : "memory");
        }
        __syncthreads();
        if (k == 0) pdl_trigger();
        const int id = blockIdx.x + k * gridDim.x;
        if (tid < RT_DIAG) {
            const int off = tid - (RT_ROWS - 1);   // column - row inside the tile
            const int r0 = max(0, -off), r1 = min(RT_ROWS, RT_COLS - off);
            double s = 0.0;
            for (int r = r0; r < r1; ++r) s += (double)tile[st][r][r + off];
            part[(int64_t)id * RT_DP + tid] = s;
        }
        __syncthreads();   // every thread is done with the stage before it is refilled
        if (tid == 0) issue(k + RT_TMA_STAGES, st);
    }
}

// w[v][u] (u < Li) = sum over tiles of the sums on diagonal d = u - ci (column
// - row): one warp per (u, v), lane = row block (strided), all loads in
// flight, then a fixed-order warp tree.
__global__ void __launch_bounds__(256) k_rat_w(const double* __restrict__ part, int n, int ci, int Li,
                                               double* __restrict__ w, int ldw) {
    const int lane = threadIdx.x & 31;
    const int u = blockIdx.x * 8 + (threadIdx.x >> 5), v = blockIdx.y;
    pdl_wait();
    pdl_trigger();
    if (u >= Li) return;
    const int cbn = n / RT_COLS, rbn = n / RT_ROWS, tiles = rbn * cbn;
    const int d = u - ci;
    const double* pv = part + (int64_t)v * tiles * RT_DP;
    double s = 0.0;
    for (int rb0 = 0; rb0 < rbn; rb0 += 64) {
        double q[4];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int rb = rb0 + lane + 32 * h;
            q[2 * h] = q[2 * h + 1] = 0.0;
            if (rb < rbn) {
                // tile (rb, cb) holds diagonals [128 cb - 32 rb - 31, 128 cb - 32 rb + 127]: <= 2 column blocks
                const int lo = d + RT_ROWS * rb - (RT_COLS - 1), hi = d + RT_ROWS * rb + (RT_ROWS - 1);
                const int cb0 = lo <= 0 ? 0 : (lo + RT_COLS - 1) / RT_COLS;
                const int cb1 = hi < 0 ? -1 : min(cbn - 1, hi / RT_COLS);
#pragma unroll
                for (int j = 0; j < 2; ++j) {
                    const int cb = cb0 + j;
                    if (cb <= cb1) {
                        const int i = d - (RT_COLS * cb - RT_ROWS * rb - (RT_ROWS - 1));
                        q[2 * h + j] = __ldg(pv + (int64_t)(rb * cbn + cb) * RT_DP + i);
                    }
                }
            }
        }
        s += (q[0] + q[1]) + (q[2] + q[3]);
    }
    s = warp_sum(s);
    if (lane == 0) w[(int64_t)v * ldw + u] = s;
}

// z[v][c] = sum_r Mt[c, r] w[v][r] (v < NV, a compile-time bound >= nv):
// one warp per row c (8 rows per CTA).  The whole row is loaded first
// (<= RZ_ML per lane, one round trip), overlapping the staging of w (all
// vectors, shared memory, zero-padded to NV), then one FMA chain per vector.
constexpr int RZ_ML = 64;   // Li <= 2048
template <typename T, int NV>
__global__ void __launch_bounds__(256) k_rat_z(const T* __restrict__ Mt, int Li, int Lo, const double* __restrict__ w,
                                               int ldw, int nv, double* __restrict__ z, int ldz) {
    extern __shared__ double wsm[];   // [NV][Li]
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x * 8 + warp;
    T m[RZ_ML];
#pragma unroll
    for (int k = 0; k < RZ_ML; ++k) {
        const int r = lane + 32 * k;
        m[k] = (c < Lo && r < Li) ? __ldg(Mt + (int64_t)c * Li + r) : T(0);
    }
    pdl_wait();      // w is written by the previous kernel; the K rows above are not
    pdl_trigger();
    // staging: 16-byte cp.async copies (no registers, all in flight at once);
    // rows of wsm padded to an even length, the padding entry never used
    const int LiP = (Li + 1) & ~1, half = LiP / 2;
    for (int idx = tid; idx < nv * half; idx += 256) {
        const int v = idx / half, pr = idx - v * half;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(wsm + v * LiP + 2 * pr));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(w + (int64_t)v * ldw + 2 * pr)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
#pragma unroll
    for (int k = 0; k < RZ_ML; ++k) {
        const int r = lane + 32 * k;
        if (r < Li) {
            const double mk = (double)m[k];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = fma(mk, wsm[v * LiP + r], acc[v]);
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double s = warp_sum(acc[v]);
        if (lane == 0 && c < Lo && v < nv) z[(int64_t)v * ldz + c] = s;
    }
}

// Programmatic dependent launch for the chain's later kernels (the first kernel of a
// product is launched normally: its input may be the previous product's output).
// For a 16-vector block it hides ~2 us of launch/drain gaps (37.0 -> 35.3 us).
static thread_local bool g_rat_pdl = true;

// z for 8 or 16 vectors on the FP64 tensor cores (mma.sync m8n8k4, SASS
// DMMA): CTA = 8 rows c of Mt, warp w = the w-th eighth of the r range; per
// 4-wide r step each lane holds Mt[c0 + gid][r + tig] (fp32 widened) as the
// A fragment and w[v][r + tig] (v = n*8 + gid, staged by cp.async) as the B
// fragments; the 8 warp partials are added in warp order.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <typename T, int NT>   // NT = 8-vector tiles (1 or 2)
__global__ void __launch_bounds__(256) k_rat_z_mma(const T* __restrict__ Mt, int Li, int Lo,
                                                   const double* __restrict__ w, int ldw, int nv,
                                                   double* __restrict__ z, int ldz) {
    extern __shared__ double wsm[];   // [NT*8][LiP]
    __shared__ double red[8][8][NT * 8 + 1];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int c0 = blockIdx.x * 8;
    const int LiP = (Li + 3) & ~3, half = LiP / 2;
    for (int idx = tid; idx < (NT * 8 - nv) * LiP; idx += 256) wsm[nv * LiP + idx] = 0.0;   // unused vectors
    // r range of this warp (multiples of 4)
    const int steps = LiP / 4, per = (steps + 7) / 8;
    const int s0 = warp * per, s1 = min(steps, s0 + per);
    const int c = c0 + gid;
    // this warp's A fragments (one Mt entry per lane per r step): K does not depend on
    // the previous kernel, so these loads are in flight before the dependency wait
    constexpr int AB = 40;
    T a[AB];
#pragma unroll
    for (int j = 0; j < AB; ++j) {
        const int r = 4 * (s0 + j) + tig;
        a[j] = (c < Lo && r < Li && s0 + j < s1) ? __ldg(Mt + (int64_t)c * Li + r) : T(0);
    }
    pdl_wait();      // w is written by the previous kernel (k_rat_w)
    pdl_trigger();
    for (int idx = tid; idx < nv * half; idx += 256) {
        const int v = idx / half, pr = idx - v * half;
        const unsigned dst = static_cast<unsigned>(__cvta_generic_to_shared(wsm + v * LiP + 2 * pr));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst), "l"(w + (int64_t)v * ldw + 2 * pr)
                     : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
    // the copies' tail past Li is scratch: zero it (0 * NaN would poison the MMA)
    for (int idx = tid; idx < nv * (LiP - Li); idx += 256) {
        const int v = idx / (LiP - Li), r = Li + idx - v * (LiP - Li);
        wsm[v * LiP + r] = 0.0;
    }
    __syncthreads();
    double acc[NT][2];
#pragma unroll
    for (int q = 0; q < NT; ++q) acc[q][0] = acc[q][1] = 0.0;
#pragma unroll
    for (int j = 0; j < AB; ++j) {
        const int r = 4 * (s0 + j) + tig;
        if (s0 + j < s1) {
#pragma unroll
            for (int q = 0; q < NT; ++q) dmma884(acc[q][0], acc[q][1], (double)a[j], wsm[(q * 8 + gid) * LiP + r]);
        }
    }
    for (int sb = s0 + AB; sb < s1; ++sb) {   // long rows (Li > 1280)
        const int r = 4 * sb + tig;
        const double av = (c < Lo && r < Li) ? (double)__ldg(Mt + (int64_t)c * Li + r) : 0.0;
#pragma unroll
        for (int q = 0; q < NT; ++q) dmma884(acc[q][0], acc[q][1], av, wsm[(q * 8 + gid) * LiP + r]);
    }
    // lane holds Z^T tile rows c0 + gid, vectors q*8 + 2*tig + {0,1}
#pragma unroll
    for (int q = 0; q < NT; ++q) {
        red[warp][gid][q * 8 + 2 * tig] = acc[q][0];
        red[warp][gid][q * 8 + 2 * tig + 1] = acc[q][1];
    }
    __syncthreads();
    for (int e = tid; e < 8 * NT * 8; e += 256) {
        const int row = e / (NT * 8), v = e - row * (NT * 8);
        double s = 0.0;
#pragma unroll
        for (int ww = 0; ww < 8; ++ww) s += red[ww][row][v];
        if (c0 + row < Lo && v < nv) z[(int64_t)v * ldz + c0 + row] = s;
    }
}

template <typename K, typename... A>
static void pdl_launch(K kern, dim3 grid, size_t smem, cudaStream_t st, A... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(256);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = attr;
    lc.numAttrs = g_rat_pdl ? 1 : 0;
    KB_CUDA(cudaLaunchKernelEx(&lc, kern, args...));
}

template <typename T>
static void rat_z_launch(const T* Mt, int Li, int Lo, const double* w, int ldw, int nv, double* z, cudaStream_t st) {
    const size_t smem = sizeof(double) * (size_t)((Li + 1) & ~1);
    auto go = [&](auto kern, int NVc) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(smem * NVc)));
        pdl_launch(kern, dim3((Lo + 7) / 8), smem * NVc, st, Mt, Li, Lo, w, ldw, nv, z, ldw);
    };
    if (nv <= 1) go(k_rat_z<T, 1>, 1);
    else if (nv <= 2) go(k_rat_z<T, 2>, 2);
    else if (nv <= 4) go(k_rat_z<T, 4>, 4);
    else {   // 5..16 vectors: FP64 tensor cores
        const int NT = nv <= 8 ? 1 : 2;
        const size_t sm2 = sizeof(double) * (size_t)NT * 8 * ((Li + 3) & ~3);
        if (NT == 1) {
            KB_CUDA(cudaFuncSetAttribute(k_rat_z_mma<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
            pdl_launch(k_rat_z_mma<T, 1>, dim3((Lo + 7) / 8), sm2, st, Mt, Li, Lo, w, ldw, nv, z, ldw);
        } else {
            KB_CUDA(cudaFuncSetAttribute(k_rat_z_mma<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
            pdl_launch(k_rat_z_mma<T, 2>, dim3((Lo + 7) / 8), sm2, st, Mt, Li, Lo, w, ldw, nv, z, ldw);
        }
    }
}

// y[v][a*n + b] = (T) z[v][b - a + co] (0 outside [0, Lo))
template <typename T>
__global__ void __launch_bounds__(256) k_rat_bcast(const double* __restrict__ z, int ldz, int n, int co, int Lo,
                                                   T* __restrict__ Y, int64_t ldy) {
    extern __shared__ double zraw[];
    T* zsm = reinterpret_cast<T*>(zraw);   // z already rounded to T: one conversion per entry of z
    const int v = blockIdx.y;
    pdl_wait();
    for (int c0 = threadIdx.x; c0 < Lo; c0 += 8 * 256) {   // all loads in flight, then the stores
        double q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = c0 + 256 * k < Lo ? __ldg(z + (int64_t)v * ldz + c0 + 256 * k) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (c0 + 256 * k < Lo) zsm[c0 + 256 * k] = (T)q[k];
    }
    __syncthreads();
    const int64_t N = (int64_t)n * n;
    T* y = Y + (int64_t)v * ldy;
    // the cell (a, b) of e0 advances by a fixed stride: updated without a division
    const int64_t stride = (int64_t)gridDim.x * 256 * 4;
    const int da = (int)(stride / n), db = (int)(stride - (int64_t)da * n);
    int64_t e0 = ((int64_t)blockIdx.x * 256 + threadIdx.x) * 4;
    int a = (int)(e0 / n), b = (int)(e0 - (int64_t)a * n);
    for (; e0 < N; e0 += stride) {
        T o[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {   // n % 4 == 0: the 4 cells share the row a
            const int u = b + q - a + co;
            o[q] = (u >= 0 && u < Lo) ? zsm[u] : T(0);
        }
        if constexpr (sizeof(T) == 4) {
            __stcs(reinterpret_cast<float4*>(y + e0), make_float4(o[0], o[1], o[2], o[3]));
        } else {
            __stcs(reinterpret_cast<double2*>(y + e0), make_double2(o[0], o[1]));
            __stcs(reinterpret_cast<double2*>(y + e0 + 2), make_double2(o[2], o[3]));
        }
        a += da;
        b += db;
        if (b >= n) { b -= n; ++a; }
    }
}

// Tensor map of X as [nv][n][n] fp32 (row stride n, vector stride ldx), box 128 x 32 x 1;
// false when the driver entry point is unavailable (the per-thread-load kernel is used).
static bool tma_map_f32(CUtensorMap* map, const void* X, int n, int nv, int64_t ldx) {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    static bool tried = false;
    if (!tried) {
        tried = true;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q) !=
                cudaSuccess ||
            q != cudaDriverEntryPointSuccess)
            encode = nullptr;
        cudaGetLastError();
    }
    // opt-in (KB_RAT_TMA=1): measured 38.8 us per 16-vector block against 35.4 us for the
    // per-thread 16-byte loads of k_rat_diag (same run), so the loads stay the default
    static const bool on = std::getenv("KB_RAT_TMA") != nullptr;
    if (!encode || !on) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)nv};
    const cuuint64_t strides[2] = {(cuuint64_t)n * 4, (cuuint64_t)ldx * 4};
    const cuuint32_t box[3] = {RT_COLS, RT_ROWS, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<void*>(X), dims, strides, box, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t ra_tiled_scratch_doubles(int n, int lmax, int nv) {
    if (n < RT_COLS || n % RT_COLS) return 0;
    const size_t tiles = (size_t)(n / RT_ROWS) * (n / RT_COLS);
    return (size_t)nv * tiles * RT_DP + 2 * (size_t)nv * (lmax + 8) + 64;
}

// false when outside the tiled path's envelope (the caller falls back)
bool ra_tiled_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv, int transpose,
                    double* scratch, cudaStream_t st) {
    if (op->kind != KB_OP_RA_ZERO || nv < 1 || nv > 16) return false;
    const int n = op->side;
    if (n < RT_COLS || n % RT_COLS) return false;
    const int vec = op->dtype == KB_F32 ? 4 : 2;
    if ((ldx % 4) || (ldy % 4) || ((uintptr_t)X % 16) || ((uintptr_t)Y % 16)) return false;
    (void)vec;
    const int cu = op->kh / 2, cv = op->kw / 2;
    int ci, Li, co, Lo;
    const void* Mt;
    if (!transpose) { ci = cu; Li = op->kh; co = cv; Lo = op->kw; Mt = op->kt; }   // z = K^T w: rows of K^T
    else { ci = cv; Li = op->kw; co = cu; Lo = op->kh; Mt = op->k; }               // z = K w: rows of K
    const int lmax = std::max(op->kh, op->kw);
    const int tiles = (n / RT_ROWS) * (n / RT_COLS);
    double* part = scratch;
    double* w = part + (size_t)nv * tiles * RT_DP;
    double* z = w + (size_t)nv * ((lmax + 9) & ~1);
    const int ldw = (lmax + 9) & ~1;   // even: 16-byte aligned rows for the cp.async staging
    const int64_t N = (int64_t)n * n;
    const double bytes = (double)(op->dtype == KB_F32 ? 4 : 8) * (2.0 * nv * N + (double)op->kh * op->kw);
    ProfScope ps(st, PROF_RA_DIAG, bytes);
    // broadcast: ~4 CTAs per SM in total, so each CTA's staging of z (Lo doubles) is small
    // next to the part of the output it writes
    const int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 256 * 4), (4 * kSMs + nv - 1) / nv));
    if (Li > 32 * RZ_ML || (size_t)Li * 8 * 16 > 200 * 1024) return false;
    static const int pdl_env = std::getenv("KB_RAT_PDL") ? std::atoi(std::getenv("KB_RAT_PDL")) : -1;
    g_rat_pdl = pdl_env >= 0 ? pdl_env != 0 : true;   // measured: nv=16 37.0 -> 35.3 us with PDL
    if (op->dtype == KB_F32) {
        CUtensorMap map;
        if (tma_map_f32(&map, X, n, nv, ldx))
            k_rat_diag_tma<<<std::min(tiles * nv, 6 * kSMs), 256, 0, st>>>(map, n, nv, part);
        else
            k_rat_diag<float><<<dim3(tiles, nv), 256, 0, st>>>(static_cast<const float*>(X), ldx, n, part);
        pdl_launch(k_rat_w, dim3((Li + 7) / 8, nv), 0, st, (const double*)part, n, ci, Li, w, ldw);
        rat_z_launch<float>(static_cast<const float*>(Mt), Li, Lo, w, ldw, nv, z, st);
        pdl_launch(k_rat_bcast<float>, dim3(bgrid, nv), sizeof(double) * Lo, st, (const double*)z, ldw, n, co, Lo,
                   static_cast<float*>(Y), (int64_t)ldy);
    } else {
        k_rat_diag<double><<<dim3(tiles, nv), 256, 0, st>>>(static_cast<const double*>(X), ldx, n, part);
        pdl_launch(k_rat_w, dim3((Li + 7) / 8, nv), 0, st, (const double*)part, n, ci, Li, w, ldw);
        rat_z_launch<double>(static_cast<const double*>(Mt), Li, Lo, w, ldw, nv, z, st);
        pdl_launch(k_rat_bcast<double>, dim3(bgrid, nv), sizeof(double) * Lo, st, (const double*)z, ldw, n, co, Lo,
                   static_cast<double*>(Y), (int64_t)ldy);
    }
    KB_LAUNCH_CHECK();
    return true;
}

}  // namespace kb
