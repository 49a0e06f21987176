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
#include <type_traits>
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
// stream-ordered kernels chained by programmatic dependent launch instead of
// one cooperative kernel with grid barriers:
//
//   k_rat_diag   a CTA owns a vertical STACK of ts tiles (32 image rows x 128
//                columns each) of one vector and streams them through a
//                shared-memory ring, each tile ONE TMA tensor copy
//                (cp.async.bulk.tensor.3d, mbarrier completion); the 32 ts + 127
//                diagonal sums of the stack accumulate in shared memory in
//                tile order (fp64, fixed order).  Tiles that meet no diagonal
//                of the PSF's support are never read.  (k_rat_diag1: the
//                single-tile form with plain loads, for few vectors.)
//   k_rat_w      w[v][u] = sum of the stack sums on diagonal u - c_in, stacks
//                in fixed (row stack, column block) order -- deterministic
//   k_rat_z      z[v][c] = sum_r Mt[c, r] w[v][r]: contiguous rows of K^T
//                (forward) or K (transpose); the r range is cut into chunks
//                owned by the CTAs of a thread-block cluster, each stages only
//                its chunk of w, and the partial tiles are added in rank order
//                in rank 0's shared memory (DSMEM); 5-16 vectors on the FP64
//                tensor cores (k_rat_z_mma)
//   k_rat_bcast  y[v][a*n + b] = z[v][b - a + c_out], float4 / double2 stores
//                from shifted 16-byte copies of z
//
// The only HBM streams are the n^2 inputs (read at most once), the n^2
// outputs (written once) and K (read once per block of vectors): the
// product's algorithmic bytes.
namespace kb {

constexpr int RT_ROWS = 32, RT_COLS = 128, RT_DIAG = RT_ROWS + RT_COLS - 1;
constexpr int RT_MAXTS = 8;          // tiles per stack (<= 256 image rows)
constexpr int RT_STAGES = 4;         // ring stages of the diagonal-sum kernel
constexpr int RT_DTHREADS = 160;     // one thread per tile diagonal (159)
constexpr int RZ_CHUNK = 1056;       // r entries per chunk of k_rat_z (<= 4 vectors): one chunk up to n = 1024
constexpr int RZM_STEPS = 32;        // 4-wide r steps per chunk of k_rat_z_mma (128 entries)
constexpr int RZM_ROWS = 64;         // rows of Mt per CTA of k_rat_z_mma (8 per warp)

// Programmatic dependent launch: the next kernel of the chain is launched
// while this one drains (launch latency hidden); it waits in pdl_wait()
// until this grid has completed and its writes are visible.
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__host__ __device__ __forceinline__ int rt_floor_div(int a, int b) { return a >= 0 ? a / b : -((-a + b - 1) / b); }
__host__ __device__ __forceinline__ int rt_ceil_div(int a, int b) { return -rt_floor_div(-a, b); }

__device__ __forceinline__ unsigned rt_smem(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ bool rt_mbar_try(unsigned mb, unsigned par) {
    unsigned ok;
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(mb), "r"(par)
        : "memory");
    return ok != 0;
}

// Stack (rs, cb) of vector v: image rows [32 ts rs, 32 ts (rs + 1)), columns [128 cb, 128 cb + 128).
// Its diagonals d = column - row span [128 cb - 32 ts rs - (32 ts - 1), 128 cb - 32 ts rs + 127]; slot
// i = d - that lower end.  part[(v * stacks + rs * cbn + cb) * (32 ts + 128) + i].
template <typename T>
__global__ void __launch_bounds__(RT_DTHREADS) k_rat_diag(const __grid_constant__ CUtensorMap map, int n, int ts,
                                                          int nst, int ci, int Li, double* __restrict__ part) {
    extern __shared__ __align__(128) unsigned char rt_raw[];
    T* tile = reinterpret_cast<T*>(rt_raw);                                   // [nst][32][128]
    double* acc = reinterpret_cast<double*>(rt_raw + (size_t)nst * RT_ROWS * RT_COLS * sizeof(T));   // [32 ts + 128]
    unsigned long long* mbar = reinterpret_cast<unsigned long long*>(acc + RT_ROWS * RT_MAXTS + RT_COLS);
    const int cbn = n / RT_COLS, stacks = (n / (RT_ROWS * ts)) * cbn;
    const int s = blockIdx.x, v = blockIdx.y, tid = threadIdx.x;
    const int rs = s / cbn, cb = s - rs * cbn;
    const int R0 = rs * RT_ROWS * ts, C0 = cb * RT_COLS;
    // tiles j of the stack that meet the support u = d + ci in [0, Li)
    const int j0 = max(0, rt_ceil_div(C0 - R0 - (RT_ROWS - 2) + ci - Li, RT_ROWS));
    const int j1 = min(ts - 1, rt_floor_div(C0 - R0 + (RT_COLS - 1) + ci, RT_ROWS));
    const int nt = j1 - j0 + 1;
    if (nt <= 0) return;   // no diagonal of this stack is ever read by k_rat_w
    const int pstride = RT_ROWS * ts + RT_COLS;
    for (int i = tid; i < pstride; i += RT_DTHREADS) acc[i] = 0.0;
    unsigned long long pol = 0;
    auto issue = [&](int k) {   // thread 0: tile j0 + k into stage k % nst
        const int st = k % nst;
        const unsigned mb = rt_smem(&mbar[st]), dst = rt_smem(tile + (size_t)st * RT_ROWS * RT_COLS);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // prior generic reads of the stage
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb),
                     "r"((unsigned)(RT_ROWS * RT_COLS * sizeof(T)))
                     : "memory");
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint"
            " [%0], [%1, {%2, %3, %4}], [%5], %6;" ::"r"(dst),
            "l"(reinterpret_cast<unsigned long long>(&map)), "r"(C0), "r"(R0 + RT_ROWS * (j0 + k)), "r"(v), "r"(mb),
            "l"(pol)
            : "memory");
    };
    if (tid == 0) {
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
        for (int st = 0; st < nst; ++st)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&mbar[st])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // launched with programmatic dependent launch too: X may be the output of the kernel before
    // (the previous product's broadcast in a chain of products), so wait for it here -- the
    // launch latency and the prologue above are already behind us
    pdl_wait();
    if (tid == 0)
        for (int k = 0; k < nst && k < nt; ++k) issue(k);
    __syncthreads();
    pdl_trigger();
    const int off = tid - (RT_ROWS - 1);   // column - row inside a tile
    for (int k = 0; k < nt; ++k) {
        const int st = k % nst;
        const unsigned par = (unsigned)(k / nst) & 1u;
        while (!rt_mbar_try(rt_smem(&mbar[st]), par)) {}
        if (tid < RT_DIAG) {
            const T* tp = tile + (size_t)st * RT_ROWS * RT_COLS;
            double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int r = 0; r < RT_ROWS; ++r) {
                const int c = r + off;
                if (c >= 0 && c < RT_COLS) sq[r & 3] += (double)tp[r * RT_COLS + c];
            }
            acc[RT_ROWS * (ts - 1 - (j0 + k)) + tid] += (sq[0] + sq[1]) + (sq[2] + sq[3]);
        }
        __syncthreads();   // the stage is free and acc is ordered for the next tile
        if (tid == 0 && k + nst < nt) issue(k + nst);
    }
    double* out = part + ((int64_t)v * stacks + s) * pstride;
    for (int i = tid; i < pstride - 1; i += RT_DTHREADS) out[i] = acc[i];
}

// One tile per CTA (ts = 1: few vectors) without the TMA ring: four 16-byte loads per thread
// straight into shared memory have less start-up latency than a tensor-map fetch and an
// mbarrier round for a single 16 KB tile.  Same slots as k_rat_diag with ts = 1.
template <typename T>
__global__ void __launch_bounds__(256) k_rat_diag1(const T* __restrict__ X, int64_t ldx, int n, int ci, int Li,
                                                   double* __restrict__ part) {
    __shared__ T tile[RT_ROWS][RT_COLS + (sizeof(T) == 4 ? 4 : 2)];
    const int cbn = n / RT_COLS, tiles = (n / RT_ROWS) * cbn;
    const int t = blockIdx.x, v = blockIdx.y;
    const int rb = t / cbn, cb = t - rb * cbn;
    const int R0 = rb * RT_ROWS, C0 = cb * RT_COLS;
    // no diagonal of the tile inside the support u = d + ci in [0, Li): never read by k_rat_w
    if (C0 - R0 + (RT_COLS - 1) + ci < 0 || C0 - R0 - (RT_ROWS - 1) + ci >= Li) return;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    pdl_wait();
    const T* x = X + (int64_t)v * ldx + (int64_t)R0 * n + C0;
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
        double sq[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
        for (int r = 0; r < RT_ROWS; ++r) {
            const int c = r + off;
            if (c >= 0 && c < RT_COLS) sq[r & 3] += (double)tile[r][c];
        }
        part[((int64_t)v * tiles + t) * (RT_ROWS + RT_COLS) + tid] = (sq[0] + sq[1]) + (sq[2] + sq[3]);
    }
}

// w[v][u] (u < Li) = sum over the stacks of their sums on diagonal d = u - ci.  CTA = 32
// diagonals x 8 row-stack lanes; the 8 lane sums are added in lane order.
__global__ void __launch_bounds__(256) k_rat_w(const double* __restrict__ part, int n, int ts, int ci, int Li,
                                               double* __restrict__ w, int ldw) {
    __shared__ double red[8][33];
    const int ux = threadIdx.x & 31, ln = threadIdx.x >> 5;
    const int u = blockIdx.x * 32 + ux, v = blockIdx.y;
    const int H = RT_ROWS * ts, cbn = n / RT_COLS, rsn = n / H, pstride = H + RT_COLS;
    pdl_wait();
    pdl_trigger();
    const int d = u - ci;
    const double* pv = part + (int64_t)v * rsn * cbn * pstride;
    double s = 0.0;
    if (u < Li) {
        // <= 3 stacks per row stack hold a given diagonal; 4 row stacks (12 loads) in flight
        for (int rs0 = ln; rs0 < rsn; rs0 += 32) {
            double q[12];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const int rs = rs0 + 8 * k;
                const int t = d + H * rs;
                const int cb_lo = max(0, rt_ceil_div(t - (RT_COLS - 1), RT_COLS));
                const int cb_hi = min(cbn - 1, rt_floor_div(t + H - 1, RT_COLS));
#pragma unroll
                for (int j = 0; j < 3; ++j) {
                    const int cb = cb_lo + j;
                    q[3 * k + j] = (rs < rsn && cb <= cb_hi)
                                       ? __ldg(pv + (int64_t)(rs * cbn + cb) * pstride + (t + H - 1 - RT_COLS * cb))
                                       : 0.0;
                }
            }
#pragma unroll
            for (int k = 0; k < 12; ++k) s += q[k];
        }
    }
    red[ln][ux] = s;
    __syncthreads();
    if (ln == 0 && u < Li) {
        double a = red[0][ux];
#pragma unroll
        for (int k = 1; k < 8; ++k) a += red[k][ux];
        w[(int64_t)v * ldw + u] = a;
    }
}

// Chunk partials -> z without a trip through global memory: the CTAs of one row group
// (the r chunks) form a thread-block cluster (1, csize, 1); each stores its partial tile
// into rank 0's shared memory (DSMEM), one cluster barrier, and rank 0 adds the ranks in
// rank order (fixed order: deterministic).
template <int NE>
__device__ __forceinline__ void rat_z_cluster_sum(double (&zred)[8][NE], const double* mine, int ne, int csize,
                                                  double* __restrict__ z, int ldz, int rows, int c0, int Lo) {
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    double* dst = cl.map_shared_rank(&zred[0][0], 0);
    for (int e = threadIdx.x; e < ne; e += 256) dst[rank * NE + e] = mine[e];
    cl.sync();
    if (rank != 0) return;
    for (int e = threadIdx.x; e < ne; e += 256) {
        const int v = e / rows, c = c0 + (e - v * rows);
        double s = zred[0][e];
        for (int q = 1; q < csize; ++q) s += zred[q][e];
        if (c < Lo) z[(int64_t)v * ldz + c] = s;
    }
}

// z[v][c] = sum_r Mt[c, r] w[v][r] (v < NV, a compile-time bound >= nv): one warp per row c
// (8 rows per CTA); the r range is cut into chunks of RZ_CHUNK entries, cluster rank q takes
// chunks q, q + csize, ...  Each row chunk is loaded first (K does not depend on the previous
// kernel), then w's chunk is staged, then one FMA chain per vector.
template <typename T, int NV>
__global__ void __launch_bounds__(256) k_rat_z(const T* __restrict__ Mt, int Li, int Lo, const double* __restrict__ w,
                                               int ldw, int nv, double* __restrict__ z, int ldz) {
    __shared__ double wsm[NV][RZ_CHUNK];
    __shared__ double zred[8][8 * NV];
    __shared__ double mine[8 * NV];
    constexpr int ML = RZ_CHUNK / 32;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c = blockIdx.x * 8 + warp;
    const int nch = (Li + RZ_CHUNK - 1) / RZ_CHUNK, csize = gridDim.y;
    double acc[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) acc[v] = 0.0;
    for (int ch = blockIdx.y; ch < nch; ch += csize) {
        const int r0 = ch * RZ_CHUNK;
        T m[ML];
#pragma unroll
        for (int k = 0; k < ML; ++k) {
            const int r = r0 + lane + 32 * k;
            m[k] = (c < Lo && r < Li) ? __ldg(Mt + (int64_t)c * Li + r) : T(0);
        }
        if (ch == (int)blockIdx.y) {
            pdl_wait();      // w is written by the previous kernel; the K rows above are not
            pdl_trigger();
        } else {
            __syncthreads();   // the previous chunk of w is no longer read
        }
        // w's chunk: all of a thread's loads in flight before the stores (one L2 round trip)
#pragma unroll
        for (int v = 0; v < NV; ++v) {
            constexpr int WB = (RZ_CHUNK + 255) / 256;
            double q[WB];
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                const int r = tid + 256 * k;
                q[k] = (v < nv && r < RZ_CHUNK && r0 + r < Li) ? __ldg(w + (int64_t)v * ldw + r0 + r) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < WB; ++k) {
                const int r = tid + 256 * k;
                if (r < RZ_CHUNK) wsm[v][r] = q[k];
            }
        }
        __syncthreads();
#pragma unroll
        for (int k = 0; k < ML; ++k) {
            const double mk = (double)m[k];
#pragma unroll
            for (int v = 0; v < NV; ++v) acc[v] = fma(mk, wsm[v][lane + 32 * k], acc[v]);
        }
    }
#pragma unroll
    for (int v = 0; v < NV; ++v) {
        const double s = warp_sum(acc[v]);
        if (lane == 0) {
            if (csize == 1) {
                if (c < Lo && v < nv) z[(int64_t)v * ldz + c] = s;
            } else {
                mine[v * 8 + warp] = s;
            }
        }
    }
    if (csize == 1) return;
    __syncthreads();
    rat_z_cluster_sum<8 * NV>(zred, mine, 8 * nv, csize, z, ldz, 8, blockIdx.x * 8, Lo);
}

static thread_local bool g_rat_pdl = true;
static thread_local bool g_rat_is_first = false;    // the launch in progress is a product's first kernel
static thread_local bool g_rat_pdl_first = true;   // PDL for a product's first kernel (8+ vectors: -5 %; slower for 1-4)

// The same for 5-16 vectors on the FP64 tensor cores (mma.sync m8n8k4, SASS DMMA):
// CTA = RZM_ROWS rows c of Mt (8 per warp), chunks of RZM_STEPS 4-wide r steps (a staged
// chunk of w serves all 64 rows); per step each lane holds Mt[c][r + tig] (fp32 widened) as
// the A fragment and w[v][r + tig] (v = q*8 + gid, staged by cp.async) as the B fragments,
// even and odd steps on separate accumulators; the cluster ranks are added in rank order.
__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <typename T, int NT>   // NT = 8-vector tiles (1 or 2)
__global__ void __launch_bounds__(256) k_rat_z_mma(const T* __restrict__ Mt, int Li, int Lo,
                                                   const double* __restrict__ w, int ldw, int nv,
                                                   double* __restrict__ z, int ldz) {
    constexpr int WR = 4 * RZM_STEPS, WP = WR + 4;   // row pitch: gid rows 4 doubles apart in the banks
    constexpr int NE = RZM_ROWS * NT * 8;            // entries of a CTA's z tile, [vector][row]
    extern __shared__ __align__(16) double zm_raw[];
    double(*wsm)[WP] = reinterpret_cast<double(*)[WP]>(zm_raw);   // [NT * 8][WP]
    double* zred = zm_raw + NT * 8 * WP;                          // [8][NE] (used on cluster rank 0)
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int gid = lane >> 2, tig = lane & 3;
    const int c0 = blockIdx.x * RZM_ROWS, c = c0 + warp * 8 + gid;
    const int steps = (Li + 3) / 4, nch = (steps + RZM_STEPS - 1) / RZM_STEPS, csize = gridDim.y;
    // rows past Lo read a valid row (their results are dropped at the end): no predicate per load
    const T* rowp = Mt + (int64_t)min(c, Lo - 1) * Li + tig;
    double acc[NT][2][2];
#pragma unroll
    for (int q = 0; q < NT; ++q) acc[q][0][0] = acc[q][0][1] = acc[q][1][0] = acc[q][1][1] = 0.0;
    for (int idx = tid; idx < (NT * 8 - nv) * WP; idx += 256) wsm[nv][idx] = 0.0;   // unused vectors stay zero
    for (int ch = blockIdx.y; ch < nch; ch += csize) {
        const int sA = ch * RZM_STEPS, r0 = 4 * sA;
        const bool full = r0 + WR <= Li;   // every entry of the chunk is inside the row: no predicates
        // this warp's A fragments (its 8 rows over the chunk): K does not depend on the previous
        // kernel, so these loads are in flight before the dependency wait
        T a[RZM_STEPS];
        if (full) {
#pragma unroll
            for (int j = 0; j < RZM_STEPS; ++j) a[j] = __ldg(rowp + r0 + 4 * j);
        }
        if (ch == (int)blockIdx.y) {
            pdl_wait();      // w is written by the previous kernel (k_rat_w)
            pdl_trigger();
        } else {
            __syncthreads();   // the previous chunk of w is no longer read
        }
        const double* wrow = &wsm[gid][tig];
        if (full) {
            for (int idx = tid; idx < nv * (WR / 2); idx += 256) {
                const int v = idx / (WR / 2), pr = idx % (WR / 2);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(rt_smem(&wsm[v][2 * pr])),
                             "l"(w + (int64_t)v * ldw + r0 + 2 * pr)
                             : "memory");
            }
            asm volatile("cp.async.wait_all;" ::: "memory");
            __syncthreads();
#pragma unroll
            for (int j = 0; j < RZM_STEPS; ++j) {
#pragma unroll
                for (int q = 0; q < NT; ++q)
                    dmma884(acc[q][j & 1][0], acc[q][j & 1][1], (double)a[j], wrow[q * 8 * WP + 4 * j]);
            }
        } else {   // the row's last, partial chunk: only its real steps; the tail past Li is zero
            const int ns = min(steps - sA, RZM_STEPS);
            for (int idx = tid; idx < nv * 4 * ns; idx += 256) {
                const int v = idx / (4 * ns), rr = idx % (4 * ns);
                wsm[v][rr] = r0 + rr < Li ? __ldg(w + (int64_t)v * ldw + r0 + rr) : 0.0;
            }
            __syncthreads();
            for (int j = 0; j < ns; ++j) {
                const double av = r0 + 4 * j + tig < Li ? (double)__ldg(rowp + r0 + 4 * j) : 0.0;
#pragma unroll
                for (int q = 0; q < NT; ++q) dmma884(acc[q][0][0], acc[q][0][1], av, wrow[q * 8 * WP + 4 * j]);
            }
        }
    }
    // lane holds Z^T tile row c (= c0 + warp*8 + gid), vectors q*8 + 2*tig + {0,1}
    if (csize == 1) {
#pragma unroll
        for (int q = 0; q < NT; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int v = q * 8 + 2 * tig + h;
                if (c < Lo && v < nv) z[(int64_t)v * ldz + c] = acc[q][0][h] + acc[q][1][h];
            }
        return;
    }
    cg::cluster_group cl = cg::this_cluster();
    const unsigned rank = cl.block_rank();
    double* dst = cl.map_shared_rank(zred, 0) + rank * NE;
#pragma unroll
    for (int q = 0; q < NT; ++q)
#pragma unroll
        for (int h = 0; h < 2; ++h)
            dst[(q * 8 + 2 * tig + h) * RZM_ROWS + warp * 8 + gid] = acc[q][0][h] + acc[q][1][h];
    cl.sync();
    if (rank != 0) return;
    for (int e = tid; e < NE; e += 256) {   // e = v * RZM_ROWS + row; ranks added in rank order
        const int v = e / RZM_ROWS, row = e % RZM_ROWS;
        double s = zred[e];
        for (int q = 1; q < csize; ++q) s += zred[q * NE + e];
        if (c0 + row < Lo && v < nv) z[(int64_t)v * ldz + c0 + row] = s;
    }
}

// Launch with programmatic dependent launch and (cy > 1) a (1, cy, 1) thread-block cluster.
template <typename K, typename... A>
static void pdl_launch_b(K kern, dim3 grid, int threads, size_t smem, cudaStream_t st, int cy, A... args);

template <typename K, typename... A>
static void pdl_launch(K kern, dim3 grid, size_t smem, cudaStream_t st, int cy, A... args) {
    pdl_launch_b(kern, grid, 256, smem, st, cy, args...);
}

template <typename K, typename... A>
static void pdl_launch_b(K kern, dim3 grid, int threads, size_t smem, cudaStream_t st, int cy, A... args) {
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(threads);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[2];
    int na = 0;
    if (g_rat_pdl && (g_rat_pdl_first || !g_rat_is_first)) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[na].val.programmaticStreamSerializationAllowed = 1;
        ++na;
    }
    if (cy > 1) {
        attr[na].id = cudaLaunchAttributeClusterDimension;
        attr[na].val.clusterDim.x = 1;
        attr[na].val.clusterDim.y = cy;
        attr[na].val.clusterDim.z = 1;
        ++na;
    }
    lc.attrs = attr;
    lc.numAttrs = na;
    KB_CUDA(cudaLaunchKernelEx(&lc, kern, args...));
}

template <typename T>
static void rat_z_launch(const T* Mt, int Li, int Lo, const double* w, int ldw, int nv, double* z, cudaStream_t st) {
    if (nv <= 4) {
        const int cy = std::min(8, (Li + RZ_CHUNK - 1) / RZ_CHUNK);
        const dim3 grid((Lo + 7) / 8, cy);
        if (nv <= 1) pdl_launch(k_rat_z<T, 1>, grid, 0, st, cy, Mt, Li, Lo, w, ldw, nv, z, ldw);
        else if (nv <= 2) pdl_launch(k_rat_z<T, 2>, grid, 0, st, cy, Mt, Li, Lo, w, ldw, nv, z, ldw);
        else pdl_launch(k_rat_z<T, 4>, grid, 0, st, cy, Mt, Li, Lo, w, ldw, nv, z, ldw);
        return;
    }
    const int steps = (Li + 3) / 4;   // 5..16 vectors: FP64 tensor cores
    const int cy = std::min(8, (steps + RZM_STEPS - 1) / RZM_STEPS);
    const dim3 grid((Lo + RZM_ROWS - 1) / RZM_ROWS, cy);
    constexpr size_t row_b = sizeof(double) * (4 * RZM_STEPS + 4), red_b = sizeof(double) * 8 * RZM_ROWS * 8;
    static bool cfg = false;
    if (!cfg) {
        KB_CUDA(cudaFuncSetAttribute(k_rat_z_mma<T, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(8 * row_b + red_b)));
        KB_CUDA(cudaFuncSetAttribute(k_rat_z_mma<T, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)(16 * row_b + 2 * red_b)));
        cfg = true;
    }
    if (nv <= 8) pdl_launch(k_rat_z_mma<T, 1>, grid, 8 * row_b + red_b, st, cy, Mt, Li, Lo, w, ldw, nv, z, ldw);
    else pdl_launch(k_rat_z_mma<T, 2>, grid, 16 * row_b + 2 * red_b, st, cy, Mt, Li, Lo, w, ldw, nv, z, ldw);
}

// y[v][a*n + b] = (T) z[v][b - a + co] (0 outside [0, Lo)).  z is staged rounded to T and
// zero-padded (zpad[i] = z[i - 4]), then as V = 16 / sizeof(T) shifted copies, copy s holding
// zpad[V k + s .. V k + s + V - 1] as its k-th 16-byte vector: the V consecutive entries a
// thread needs are ONE aligned vector load whatever the alignment of its diagonal index,
// and the lanes of a warp read consecutive vectors (no bank conflicts; the scalar form
// had a 4-way conflict on every load).
template <typename T>
__global__ void __launch_bounds__(256) k_rat_bcast(const double* __restrict__ z, int ldz, int n, int co, int Lo,
                                                   T* __restrict__ Y, int64_t ldy) {
    constexpr int V = 16 / sizeof(T);
    using VT = typename std::conditional<sizeof(T) == 4, float4, double2>::type;
    extern __shared__ __align__(16) unsigned char braw[];
    const int KV = (Lo + 8 + V - 1) / V + 1;           // vectors per copy
    VT* zc = reinterpret_cast<VT*>(braw);              // [V][KV]
    T* zpad = reinterpret_cast<T*>(zc + V * KV);       // [V * KV + V]
    const int v = blockIdx.y;
    pdl_wait();
    pdl_trigger();   // a following product's first kernel may launch; it waits for this grid's writes
    for (int i0 = threadIdx.x; i0 < V * KV + V; i0 += 8 * 256) {   // 8 loads in flight, then the stores
        double q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int zi = i0 + 256 * k - 4;
            q[k] = (zi >= 0 && zi < Lo) ? __ldg(z + (int64_t)v * ldz + zi) : 0.0;
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (i0 + 256 * k < V * KV + V) zpad[i0 + 256 * k] = (T)q[k];
    }
    __syncthreads();
    for (int i = threadIdx.x; i < V * KV; i += 256) {
        const int s = i / KV, k = i - s * KV;
        const T* src = zpad + V * k + s;
        if constexpr (sizeof(T) == 4) zc[i] = make_float4(src[0], src[1], src[2], src[3]);
        else zc[i] = make_double2(src[0], src[1]);
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
        const int idx = b - a + co + 4;   // zpad index of the first of the 4 cells (n % 4 == 0: one row a)
        const bool in = idx >= 1 && idx <= Lo + 3;
        if constexpr (sizeof(T) == 4) {
            const float4 o = in ? zc[(idx & 3) * KV + (idx >> 2)] : make_float4(0.f, 0.f, 0.f, 0.f);
            __stcs(reinterpret_cast<float4*>(y + e0), o);
        } else {
            const double2* cp = zc + (idx & 1) * KV + (idx >> 1);
            __stcs(reinterpret_cast<double2*>(y + e0), in ? cp[0] : make_double2(0.0, 0.0));
            __stcs(reinterpret_cast<double2*>(y + e0 + 2), in ? cp[1] : make_double2(0.0, 0.0));
        }
        a += da;
        b += db;
        if (b >= n) { b -= n; ++a; }
    }
}

// Tensor map of X as [nv][n][n] (row stride n, vector stride ldx), box 128 x 32 x 1;
// false when the driver entry point is unavailable (the caller falls back to k_ra_block).
static bool rat_tensor_map(CUtensorMap* map, const void* X, int n, int nv, int64_t ldx, bool f32) {
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
    if (!encode) return false;
    const cuuint64_t es_b = f32 ? 4 : 8;
    const cuuint64_t dims[3] = {(cuuint64_t)n, (cuuint64_t)n, (cuuint64_t)nv};
    const cuuint64_t strides[2] = {(cuuint64_t)n * es_b, (cuuint64_t)(nv > 1 ? ldx : (int64_t)n * n) * es_b};
    const cuuint32_t box[3] = {RT_COLS, RT_ROWS, 1};
    const cuuint32_t es[3] = {1, 1, 1};
    return encode(map, f32 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3,
                  const_cast<void*>(X), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                  CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

static int rat_ldw(int lmax) { return (lmax + 9) & ~1; }   // even: 16-byte aligned rows for the cp.async staging

size_t ra_tiled_scratch_doubles(int n, int lmax, int nv) {
    if (n < RT_COLS || n % RT_COLS) return 0;
    const size_t tiles = (size_t)(n / RT_ROWS) * (n / RT_COLS);
    return (size_t)nv * tiles * (RT_ROWS + RT_COLS) + (size_t)2 * nv * rat_ldw(lmax) + 64;
}

// false when outside the tiled path's envelope (the caller falls back)
bool ra_tiled_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv, int transpose,
                    double* scratch, cudaStream_t st) {
    if (op->kind != KB_OP_RA_ZERO || nv < 1 || nv > 16) return false;
    const int n = op->side;
    if (n < RT_COLS || n % RT_COLS) return false;
    if ((ldx % 4) || (ldy % 4) || ((uintptr_t)X % 16) || ((uintptr_t)Y % 16)) return false;
    const bool f32 = op->dtype == KB_F32;
    const int cu = op->kh / 2, cv = op->kw / 2;
    int ci, Li, co, Lo;
    const void* Mt;
    if (!transpose) { ci = cu; Li = op->kh; co = cv; Lo = op->kw; Mt = op->kt; }   // z = K^T w: rows of K^T
    else { ci = cv; Li = op->kw; co = cu; Lo = op->kh; Mt = op->k; }               // z = K w: rows of K
    const int lmax = std::max(op->kh, op->kw);
    // tiles per stack: 2 when that still gives ~2 CTAs per SM (measured best at n = 1024 and 2048 with
    // 8-16 vectors: 37.2 us against 39.6 (1) and 39.4 (4) per 16-vector block), else 1
    static const int ts_env = std::getenv("KB_RAT_TS") ? std::atoi(std::getenv("KB_RAT_TS")) : 0;
    int ts = 1;
    if (n % (RT_ROWS * 2) == 0 && (int64_t)(n / (RT_ROWS * 2)) * (n / RT_COLS) * nv >= 2 * kSMs) ts = 2;
    if (ts_env > 0 && ts_env <= RT_MAXTS && n % (RT_ROWS * ts_env) == 0) ts = ts_env;
    const int stacks = (n / (RT_ROWS * ts)) * (n / RT_COLS);
    const int nst = std::min(ts, RT_STAGES);
    const int ldw = rat_ldw(lmax);
    double* part = scratch;
    double* w = part + (size_t)nv * (n / RT_ROWS) * (n / RT_COLS) * (RT_ROWS + RT_COLS);
    double* z = w + (size_t)nv * ldw;
    const int wgrid = (Li + 31) / 32;
    constexpr int BV32 = 4, BV64 = 2;
    const size_t bsm32 = (size_t)(BV32 * ((Lo + 8 + BV32 - 1) / BV32 + 1)) * (16 + 4) + 16;
    const size_t bsm64 = (size_t)(BV64 * ((Lo + 8 + BV64 - 1) / BV64 + 1)) * (16 + 8) + 16;
    if ((f32 ? bsm32 : bsm64) > 100 * 1024) return false;   // the broadcast stages z (shifted copies) in shared memory
    static bool bcfg = false;
    if (!bcfg) {
        KB_CUDA(cudaFuncSetAttribute(k_rat_bcast<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        KB_CUDA(cudaFuncSetAttribute(k_rat_bcast<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        bcfg = true;
    }
    const int64_t N = (int64_t)n * n;
    const double bytes = (double)(f32 ? 4 : 8) * (2.0 * nv * N + (double)op->kh * op->kw);
    ProfScope ps(st, PROF_RA_DIAG, bytes);
    static const int pdl_env = std::getenv("KB_RAT_PDL") ? std::atoi(std::getenv("KB_RAT_PDL")) : -1;
    g_rat_pdl = pdl_env >= 0 ? pdl_env != 0 : true;
    g_rat_pdl_first = nv >= 8;
    // broadcast: ~KB_RAT_BCTAS CTAs per SM in total, so each CTA's staging of z (Lo doubles) is
    // small next to the part of the output it writes
    static const int bctas = std::getenv("KB_RAT_BCTAS") ? std::max(1, std::atoi(std::getenv("KB_RAT_BCTAS"))) : 8;
    const int bgrid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(N, 256 * 4), (bctas * kSMs + nv - 1) / nv));
    const size_t dsm = (size_t)nst * RT_ROWS * RT_COLS * (f32 ? 4 : 8) + sizeof(double) * (RT_ROWS * RT_MAXTS + RT_COLS) +
                       sizeof(unsigned long long) * RT_STAGES;
    static const bool use_ld1 = !(std::getenv("KB_RAT_LD1") && std::atoi(std::getenv("KB_RAT_LD1")) == 0);
    CUtensorMap map;
    if (!(ts == 1 && use_ld1) && !rat_tensor_map(&map, X, n, nv, ldx, f32)) return false;
    static const int skip = std::getenv("KB_RAT_SKIP") ? std::atoi(std::getenv("KB_RAT_SKIP")) : 0;   // timing experiments only
    if (f32) {
        static bool cfg = false;
        if (!cfg) {
            KB_CUDA(cudaFuncSetAttribute(k_rat_diag<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024));
            cfg = true;
        }
        g_rat_is_first = true;
        if (skip & 1) {
        } else if (ts == 1 && use_ld1) {
            pdl_launch_b(k_rat_diag1<float>, dim3(stacks, nv), 256, 0, st, 1, static_cast<const float*>(X), ldx, n, ci, Li,
                         part);
        } else {
            pdl_launch_b(k_rat_diag<float>, dim3(stacks, nv), RT_DTHREADS, dsm, st, 1, map, n, ts, nst, ci, Li, part);
        }
        g_rat_is_first = false;
        if (!(skip & 2)) pdl_launch(k_rat_w, dim3(wgrid, nv), 0, st, 1, (const double*)part, n, ts, ci, Li, w, ldw);
        if (!(skip & 4)) rat_z_launch<float>(static_cast<const float*>(Mt), Li, Lo, w, ldw, nv, z, st);
        if (!(skip & 8)) pdl_launch(k_rat_bcast<float>, dim3(bgrid, nv), bsm32, st, 1, (const double*)z, ldw, n, co, Lo,
                   static_cast<float*>(Y), (int64_t)ldy);
    } else {
        static bool cfg = false;
        if (!cfg) {
            KB_CUDA(cudaFuncSetAttribute(k_rat_diag<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, 140 * 1024));
            cfg = true;
        }
        g_rat_is_first = true;
        if (ts == 1 && use_ld1)
            pdl_launch_b(k_rat_diag1<double>, dim3(stacks, nv), 256, 0, st, 1, static_cast<const double*>(X), ldx, n, ci,
                         Li, part);
        else
            pdl_launch_b(k_rat_diag<double>, dim3(stacks, nv), RT_DTHREADS, dsm, st, 1, map, n, ts, nst, ci, Li, part);
        g_rat_is_first = false;
        pdl_launch(k_rat_w, dim3(wgrid, nv), 0, st, 1, (const double*)part, n, ts, ci, Li, w, ldw);
        rat_z_launch<double>(static_cast<const double*>(Mt), Li, Lo, w, ldw, nv, z, st);
        pdl_launch(k_rat_bcast<double>, dim3(bgrid, nv), bsm64, st, 1, (const double*)z, ldw, n, co, Lo,
                   static_cast<double*>(Y), (int64_t)ldy);
    }
    KB_LAUNCH_CHECK();
    return true;
}

}  // namespace kb
