// Persistent cooperative eGKB for the matrix-free R(A) (fp32 / fp64), sm_100a.
//
// The whole bidiagonalisation (lowrank.py:207-303) runs in ONE kernel launch:
// 2 CTAs per SM, grid-wide barriers (cooperative groups) between the phases
// of each half step, and the reference's breakdown tests and nu rank rule
// evaluated redundantly (and identically) by every CTA, so the loop needs no
// host round trip and no per-phase kernel launch.  One half step is
//
//   diag   : partial diagonal sums of the input basis vector  (R(A) product, part 1)
//   colsum : partial K (or K^T) column sums                     (part 2)
//   dots   : z -> Toeplitz y ; v = y - beta*prev ; h = S^T v ; |v|^2 ; |y|^2
//   apply  : v1 = v - S h (one classical GS pass), |v1|^2      (v kept in registers)
//   write  : out = v1 / t                                      (t = |v1|)
//
// with 5 grid barriers; the vector v never leaves registers between dots,
// apply and write (each thread owns up to MAXG*VEC elements), so one pass
// writes the new basis vector and the reorthogonalisation reads the basis
// twice (coefficients, update).  All cross-CTA sums are fixed-order
// (per-CTA partials reduced in index order), so results are deterministic.
#include <cooperative_groups.h>

#include <type_traits>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "kb_ops.cuh"

namespace cg = cooperative_groups;

namespace kb {

constexpr int PK_THREADS = 256;
constexpr int PK_SEGS = 8;
constexpr int PK_NSTRIDE = 16;   // norm partials one 128-B line apart (no hot lines in the reduction)

struct PkParams {
    const void* K;    // kh x kw
    const void* Kt;   // kw x kh
    int kh, kw, n;
    int refl;         // reflexive BC (Hankel index families, kb_ops.cuh)
    void* S;
    void* Q;
    int64_t ld_s, ld_q;
    int cap;
    const void* y0;
    int* hdr;
    double *alphas, *ts, *zetas, *nus;
    double tol, tau;
    int k_max, p, k_min, full_reorth;
    double* diag_part;   // [PK_SEGS][Lmax]
    double* col_part;    // [PK_SEGS][Lmax]
    double* blk_part;    // [grid][cap + 4]
    double* norm_part;   // [grid][PK_NSTRIDE]
    double* zbuf;        // [Lmax]: z = K^T w (or K w), summed by each column chunk's last finisher
    double* bres;        // [cap + 4]: results published by a reduce-barrier's last arriver
    unsigned* bar;       // [0]: arrivals, [32]: generation, [64..): per-column-chunk finish counters
    int nbar;            // words in bar + wfix (zeroed before the launch)
    unsigned long long* wfix;   // [2][Lmax] fixed-point diagonal sums (tiled kernel)
    long long* xacc;            // [2][cap + 4][3] exact limb accumulators of the grid sums (tiled kernel)
    void* raw_s;         // pending unnormalised s vector (N elements)
    void* raw_q;         // pending unnormalised q vector
    int ng;              // element groups per thread
    int lmax;
    unsigned long long* dbg;   // optional phase timestamps (block 0), KB_PK_TRACE
    int* dbg_n;
    int cg_sync;               // 1: cooperative-groups grid.sync (KB_PK_CGSYNC=1) instead of pk_grid_sync
};

__device__ __forceinline__ void pk_mark(const PkParams& P, int tag = 0) {
    if (P.dbg && blockIdx.x == 0 && threadIdx.x == 0) {
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        t = (t & ~15ull) | (unsigned)tag;   // phase tag in the low bits (ns resolution is not needed)
        const int k = *P.dbg_n;
        if (k < 4096) P.dbg[k] = t;
        *P.dbg_n = k + 1;
    }
}

enum { PH_DONE = 0, PH_FIRED, PH_REASON, PH_STOP, PH_BREAK, PH_TBREAK, PH_OVERFLOW, PH_ERR, PH_NA, PH_NT,
       PH_NN };

template <typename T, int VEC>
struct PkIO;
template <>
struct PkIO<float, 4> {
    static __device__ __forceinline__ void load(const float* p, float* v) {
        const float4 q = __ldcg(reinterpret_cast<const float4*>(p));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
    static __device__ __forceinline__ void store(float* p, const float* v) {
        *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
    }
};
template <>
struct PkIO<double, 2> {
    static __device__ __forceinline__ void load(const double* p, double* v) {
        const double2 q = __ldcg(reinterpret_cast<const double2*>(p));
        v[0] = q.x; v[1] = q.y;
    }
    static __device__ __forceinline__ void store(double* p, const double* v) {
        *reinterpret_cast<double2*>(p) = make_double2(v[0], v[1]);
    }
};

// fl32(a / b) computed as fl32(fl64(a / b)): double rounding is innocuous for
// a quotient of two floats (53 >= 2 * 24 + 2), so this equals the correctly
// rounded fp32 division bit for bit -- without the subnormal slow path of the
// fp32 division routine, which the Gaussian-tail entries of the Krylov vectors
// (subnormal in fp32) hit on every element (10x slower stores).
// (inline PTX: the compiler would otherwise fold the widened division back
// into the fp32 one, slow path included).
// A zero dividend (the exact zeros of the Gaussian-tail entries) would
// still take the division's special-case path, so it is answered directly.
__device__ __forceinline__ float pk_fdiv_exact(float a, float b) {
    const float fa = fabsf(a);
    if (fa >= 0x1p-100f && fa <= 0x1p100f)   // comfortably normal: the fp32 division's fast path
        return __fdiv_rn(a, b);
    if (a == 0.f) return __int_as_float((__float_as_int(a) ^ __float_as_int(b)) & 0x80000000);
    double q;
    asm("div.rn.f64 %0, %1, %2;" : "=d"(q) : "d"((double)a), "d"((double)b));
    return (float)q;
}
// The same correctly rounded fl32(a / b) with rb = RN64(1 / b) precomputed:
// for fp32 a and b the exact quotient is never closer than 2^-48 (relative)
// to an fp32 rounding boundary unless it is representable, and (double)a * rb
// is within 2^-52 of it, so rounding it to fp32 gives the correctly rounded
// quotient -- subnormal results and signed zeros included -- for two
// conversions and a multiply instead of a double division.
__device__ __forceinline__ float pk_fdiv_exact(float a, float b, double rb) {
    const float fa = fabsf(a);
    if (fa >= 0x1p-100f && fa <= 0x1p100f) return __fdiv_rn(a, b);
    return (float)((double)a * rb);
}

__device__ __forceinline__ float pk_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double pk_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float pk_sub(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double pk_sub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float pk_div(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double pk_div(double a, double b) { return __ddiv_rn(a, b); }

// Fixed-order sum over the grid's per-CTA partials part[b * stride + j],
// slots j < nslots.  A warp covers Wp = pow2ceil(min(nslots, 32)) slots with
// 32 / Wp lanes per slot (lane = sub * Wp + slot): every request reads one
// CTA's partial row (coalesced, one 128-B line when stride is padded), the
// 8 warps x (32 / Wp) subs split the CTAs, all loads of a lane are issued
// before they are summed (one L2 round trip), then subs are combined by a
// fixed shuffle tree and warps in warp order.  Result -> out[];  `tmp` is
// >= 8 * 32 doubles of shared memory.  Ends with __syncthreads().
constexpr int PK_RED_BATCH = 20;   // loads in flight per lane
__device__ __forceinline__ void pk_reduce_slots(const double* part, int stride, int nblk, int nslots,
                                                double* out, double* tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int wp = 1;
    while (wp < nslots && wp < 32) wp <<= 1;
    const int subs = 32 / wp, sub = lane / wp, sl = lane % wp;
    for (int j0 = 0; j0 < nslots; j0 += wp) {
        const int j = j0 + sl;
        double s = 0.0;
        if (j < nslots) {
            for (int b0 = warp + 8 * sub; b0 < nblk; b0 += 8 * subs * PK_RED_BATCH) {
                double q[PK_RED_BATCH];
#pragma unroll
                for (int k = 0; k < PK_RED_BATCH; ++k) {
                    const int b = b0 + 8 * subs * k;
                    q[k] = b < nblk ? __ldcg(part + (int64_t)b * stride + j) : 0.0;
                }
#pragma unroll
                for (int k = 0; k < PK_RED_BATCH; ++k) s += q[k];
            }
        }
        for (int o = 16; o >= wp; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        tmp[warp * 32 + lane] = s;
        __syncthreads();
        if (warp == 0 && lane < wp && j < nslots) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t += tmp[w * 32 + lane];
            out[j] = t;
        }
        __syncthreads();
    }
}


// Grid barrier followed by the fixed-order reduction of the per-CTA partials
// part[b * stride + j] (j < nslots) in every CTA (pk_reduce_slots: coalesced,
// one L2 round trip).  A "last arriver reduces and publishes" variant was
// measured slower (tools/red_probe.cu: 3.5 vs 2.7 us for 15 slots); the tiled
// kernel avoids the partial array altogether (xacc_add / xacc_get).  On
// return out[j] (shared memory) holds the sums in every CTA.
__device__ __forceinline__ void pk_reduce_barrier(const double* part, int stride, int nslots, double* out,
                                                  double* tmp) {
    cg::this_grid().sync();
    pk_reduce_slots(part, stride, gridDim.x, nslots, out, tmp);
}

template <typename T>
struct PkHalf {
    const T* x;       // input basis vector of the R(A) product (normalised)
    const T* prev;    // previous basis vector (normalised), v = y - beta * prev
    T beta;
    const T* S;       // basis to project against
    int64_t ld;
    int m;            // basis vectors in S
    T* out;           // new basis slot (receives fl(v1 / t), as lowrank.py:247, 260)
    int transpose;    // 0: y = R x (s step), 1: y = R^T x (q step)
};

// One half step.  Returns t = |v1| (identical in every CTA).
template <typename T, int VEC, int MAXG>
__device__ double pk_half(const PkParams& P, const PkHalf<T>& H, double* sm, double& ysq_out, cg::grid_group& grid) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    const int nblk = gridDim.x;
    const int cu = P.kh / 2, cv = P.kw / 2;
    const int ci = H.transpose ? cv : cu, Li = H.transpose ? P.kw : P.kh;
    const int co = H.transpose ? cu : cv, Lo = H.transpose ? P.kh : P.kw;
    const T* M = static_cast<const T*>(H.transpose ? P.Kt : P.K);   // Li x Lo row-major
    double* zs = sm;                              // [lmax]
    double* red = zs + P.lmax;                    // [cap + 4]
    double* acc = red + P.cap + 4;                // [8][max(cap + 2, 33)]
    const int64_t G = (int64_t)nblk * PK_THREADS;
    const int64_t gt = (int64_t)blockIdx.x * PK_THREADS + tid;

    // ---- diag: part[s][u] = sum_{rows a in segment s} x[a, a + u - ci]
    {
        const int chunks = (Li + 31) / 32;
        const int items = chunks * PK_SEGS;
        for (int it = blockIdx.x; it < items; it += nblk) {
            const int c = it % chunks, seg = it / chunks;
            const int u = c * 32 + lane;
            const int s0 = (int)((int64_t)n * seg / PK_SEGS), s1 = (int)((int64_t)n * (seg + 1) / PK_SEGS);
            double a = 0.0;
            if (u < Li) a = ra_gather_rows<T, true>(H.x, n, u, ci, s0, s1, warp, P.refl != 0);
            acc[warp * 33 + lane] = a;
            __syncthreads();
            if (warp == 0 && u < Li) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) t += acc[w * 33 + lane];
                P.diag_part[(int64_t)seg * P.lmax + u] = t;
            }
            __syncthreads();
        }
    }
    grid.sync();
    pk_mark(P);
    // ---- colsum: part[s][c] = sum_{rows r in segment s} M[r, c] * w[r],  w[r] = sum_s diag_part[s][r]
    {
        const int chunks = (Lo + 31) / 32;
        const int items = chunks * PK_SEGS;
        for (int it = blockIdx.x; it < items; it += nblk) {
            const int cc = it % chunks, seg = it / chunks;
            const int c = cc * 32 + lane;
            const int r0 = (int)((int64_t)Li * seg / PK_SEGS), r1 = (int)((int64_t)Li * (seg + 1) / PK_SEGS);
            // stage w[r] = sum_s diag_part[s][r] for this segment's rows in smem (zs is free here)
            for (int j = tid; j < r1 - r0; j += PK_THREADS) {
                double t = 0.0;
#pragma unroll
                for (int q = 0; q < PK_SEGS; ++q) t += __ldcg(P.diag_part + (int64_t)q * P.lmax + r0 + j);
                zs[j] = t;
            }
            __syncthreads();
            double a = 0.0;
            int r = r0 + warp;
            for (; r + 56 < r1; r += 64) {            // 8 independent K loads in flight
                double mk[8];
#pragma unroll
                for (int k = 0; k < 8; ++k) mk[k] = (c < Lo) ? (double)__ldg(M + (int64_t)(r + 8 * k) * Lo + c) : 0.0;
#pragma unroll
                for (int k = 0; k < 8; ++k) a += mk[k] * zs[r + 8 * k - r0];
            }
            for (; r < r1; r += 8)
                if (c < Lo) a += (double)__ldg(M + (int64_t)r * Lo + c) * zs[r - r0];
            acc[warp * 33 + lane] = a;
            __syncthreads();
            if (warp == 0 && c < Lo) {
                double t = 0.0;
#pragma unroll
                for (int w = 0; w < 8; ++w) t += acc[w * 33 + lane];
                P.col_part[(int64_t)seg * P.lmax + c] = t;
            }
            // the last of the chunk's PK_SEGS items sums the segments (fixed
            // order) into z, so the dots phase reads z instead of every CTA
            // re-reducing all the partials
            __shared__ int s_fin;
            __syncthreads();
            if (tid == 0) {
                unsigned old;
                asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(P.bar + 64 + cc), "r"(1u) : "memory");
                s_fin = (old == PK_SEGS - 1);
                if (s_fin) P.bar[64 + cc] = 0u;   // next use is several grid barriers later
            }
            __syncthreads();
            if (s_fin && warp == 0 && c < Lo) {
                double q[PK_SEGS];
#pragma unroll
                for (int sg = 0; sg < PK_SEGS; ++sg) q[sg] = __ldcg(P.col_part + (int64_t)sg * P.lmax + c);
                double t = 0.0;
#pragma unroll
                for (int sg = 0; sg < PK_SEGS; ++sg) t += q[sg];
                __stcg(P.zbuf + c, t);
            }
        }
    }
    grid.sync();
    pk_mark(P);
    // ---- z (Toeplitz coefficients) into shared memory
    for (int c0 = tid; c0 < Lo; c0 += 8 * PK_THREADS) {   // all loads in flight, then the stores
        double q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = c0 + k * PK_THREADS < Lo ? __ldcg(P.zbuf + c0 + k * PK_THREADS) : 0.0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (c0 + k * PK_THREADS < Lo) zs[c0 + k * PK_THREADS] = q[k];
    }
    const int W = H.m + 2;
    for (int i = tid; i < 8 * W; i += PK_THREADS) acc[i] = 0.0;
    __syncthreads();
    pk_mark(P);
    // ---- dots: v = y - beta*prev (fp32 ops as the reference) ; h = S^T v
    // The dot products and the projection run in the working precision T
    // like the reference's BLAS sdot/saxpy (per-thread FMA chains over the
    // thread's <= MAXG*VEC entries; the per-thread partials are widened once
    // and reduced across the grid in fp64, fixed order): no per-element
    // fp32 -> fp64 conversions, whose 16/clk/SM pipe bounded these phases.
    T v[MAXG][VEC];
    double ysq = 0.0, vsq = 0.0;
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
        const int64_t e0 = (g * G + gt) * VEC;
        if (g < P.ng && e0 < N) {
            T pv[VEC];
            if (H.prev) {
                PkIO<T, VEC>::load(H.prev + e0, pv);
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q) pv[q] = T(0);
            }
            double yd[VEC];
            if constexpr (VEC == 4) {
                ra_bcast4(zs, (unsigned)e0, n, co, Lo, P.refl != 0, yd);   // one division per group
            } else {
#pragma unroll
                for (int q = 0; q < VEC; ++q) yd[q] = ra_bcast(zs, (unsigned)(e0 + q), n, co, Lo, P.refl != 0);
            }
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const T yv = (T)yd[q];
                ysq += (double)yv * (double)yv;
                v[g][q] = pk_sub(yv, pk_mul(H.beta, pv[q]));
            }
        } else {
#pragma unroll
            for (int q = 0; q < VEC; ++q) v[g][q] = T(0);
        }
    }
    pk_mark(P);
#pragma unroll 4
    for (int i = 0; i < H.m; ++i) {
        const T* Si = H.S + (int64_t)i * H.ld;
        T dt = T(0);
#pragma unroll
        for (int g = 0; g < MAXG; ++g) {
            const int64_t e0 = (g * G + gt) * VEC;
            if (g < P.ng && e0 < N) {
                T sv[VEC];
                PkIO<T, VEC>::load(Si + e0, sv);
#pragma unroll
                for (int q = 0; q < VEC; ++q) dt = fma(sv[q], v[g][q], dt);
            }
        }
        const double d = warp_sum((double)dt);
        if (lane == 0) acc[warp * W + i] += d;
    }
#pragma unroll
    for (int g = 0; g < MAXG; ++g)
#pragma unroll
        for (int q = 0; q < VEC; ++q) vsq += (double)v[g][q] * (double)v[g][q];
    vsq = warp_sum(vsq);
    ysq = warp_sum(ysq);
    if (lane == 0) {
        acc[warp * W + H.m] += vsq;
        acc[warp * W + H.m + 1] += ysq;
    }
    __syncthreads();
    pk_mark(P);
    for (int j = tid; j < W; j += PK_THREADS) {
        double t = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) t += acc[w * W + j];
        P.blk_part[(int64_t)blockIdx.x * (P.cap + 4) + j] = t;
    }
    pk_reduce_barrier(P.blk_part, P.cap + 4, W, red, acc);
    pk_mark(P);
    ysq_out = red[H.m + 1];
    double t;
    if (H.m == 0) {
        t = sqrt(red[0]);
    } else {
    // ---- apply: v1 = v - S h in T (one FMA per basis entry, as saxpy), kept in registers
    constexpr int GA = MAXG <= 4 ? MAXG : 4;   // element groups per pass over the basis
    T* cf = reinterpret_cast<T*>(acc);          // coefficients in T (acc is free after the barrier)
    for (int i = tid; i < H.m; i += PK_THREADS) cf[i] = (T)red[i];
    __syncthreads();
    double v1sq = 0.0;
#pragma unroll
    for (int g0 = 0; g0 < MAXG; g0 += GA) {
        if (g0 >= P.ng) break;
#pragma unroll 4
        for (int i = 0; i < H.m; ++i) {
            const T* Si = H.S + (int64_t)i * H.ld;
            const T c = cf[i];
#pragma unroll
            for (int g = 0; g < GA; ++g) {
                const int64_t e0 = ((g0 + g) * G + gt) * VEC;
                if (g0 + g < P.ng && e0 < N) {
                    T sv[VEC];
                    PkIO<T, VEC>::load(Si + e0, sv);
#pragma unroll
                    for (int q = 0; q < VEC; ++q) v[g0 + g][q] = fma(-c, sv[q], v[g0 + g][q]);
                }
            }
        }
#pragma unroll
        for (int g = 0; g < GA; ++g)
#pragma unroll
            for (int q = 0; q < VEC; ++q) v1sq += (double)v[g0 + g][q] * (double)v[g0 + g][q];
    }
    v1sq = warp_sum(v1sq);
    __syncthreads();   // cf (in acc) is read until every warp has finished the projection
    if (lane == 0) acc[warp] = v1sq;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += acc[w];
        P.norm_part[(int64_t)blockIdx.x * PK_NSTRIDE] = s;
    }
    pk_reduce_barrier(P.norm_part, PK_NSTRIDE, 1, red + P.cap + 2, acc);
    pk_mark(P);
    t = sqrt(red[P.cap + 2]);
    }
    // ---- write: out = fl(v1 / t)
    const T td = (T)t;
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
        const int64_t e0 = (g * G + gt) * VEC;
        if (g < P.ng && e0 < N) {
            T o[VEC];
#pragma unroll
            for (int q = 0; q < VEC; ++q) o[q] = pk_div((T)v[g][q], td);
            PkIO<T, VEC>::store(H.out + e0, o);
        }
    }
    grid.sync();
    pk_mark(P);
    return t;
}

template <typename T, int VEC, int MAXG>
__global__ void __launch_bounds__(PK_THREADS, 2) k_egkb_persistent(PkParams P) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    const int64_t N = (int64_t)n * n;
    const int nblk = gridDim.x;
    T* S = static_cast<T*>(P.S);
    T* Q = static_cast<T*>(P.Q);
    const T* y0 = static_cast<const T*>(P.y0);
    double* red = sm + P.lmax;
    double* acc = red + P.cap + 4;
    const int64_t G = (int64_t)nblk * PK_THREADS;
    const int64_t gt = (int64_t)blockIdx.x * PK_THREADS + tid;
    const bool rec = (blockIdx.x == 0 && tid == 0);

    // ---- s1 = y0 / |y0|   (lowrank.py:207-210)
    T v0[MAXG][VEC];
    double vsq = 0.0;
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
        const int64_t e0 = (g * G + gt) * VEC;
        if (g < P.ng && e0 < N) {
            PkIO<T, VEC>::load(y0 + e0, v0[g]);
#pragma unroll
            for (int q = 0; q < VEC; ++q) vsq += (double)v0[g][q] * (double)v0[g][q];
        }
    }
    vsq = warp_sum(vsq);
    if (lane == 0) acc[warp] = vsq;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; ++w) s += acc[w];
        P.norm_part[(int64_t)blockIdx.x * PK_NSTRIDE] = s;
    }
    pk_reduce_barrier(P.norm_part, PK_NSTRIDE, 1, red, acc);
    pk_mark(P);
    const double t1 = sqrt(red[0]);
    {
        const T td = (T)t1;
#pragma unroll
        for (int g = 0; g < MAXG; ++g) {
            const int64_t e0 = (g * G + gt) * VEC;
            if (g < P.ng && e0 < N) {
                T o[VEC];
#pragma unroll
                for (int q = 0; q < VEC; ++q) o[q] = pk_div(v0[g][q], td);
                PkIO<T, VEC>::store(S + e0, o);
            }
        }
    }
    grid.sync();
    pk_mark(P);
    // ---- the half steps, ONE call site of pk_half (one inlined copy: the
    // kernel's instruction footprint is a third of three separate calls):
    //   step 0      : q1 = B^T s1 / alpha1                    (lowrank.py:211-215)
    //   odd steps   : s step, s_{j+1} = B q_j - alpha_j s_j   (lowrank.py:237-247)
    //   even steps  : q step, q_{j+1} = B^T s_{j+1} - t q_j   (lowrank.py:249-260) + control
    int done = 1, fired = -1, reason = 0, stop = 0, breakdown = 0, tbreak = 0, overflow = 0, err = 0;
    int na = 1, nt = 1, nn = 1;
    double zeta_last = 0.0, nu_last = 1e308, alpha_cur = 0.0, t_new = 0.0, u2 = 0.0;
    for (int step = 0;; ++step) {
        PkHalf<T> h;
        if (step == 0) {
            h = PkHalf<T>{S, nullptr, T(0), Q, P.ld_q, 0, Q, 1};
        } else if (step & 1) {
            h = PkHalf<T>{Q + (int64_t)(done - 1) * P.ld_q, S + (int64_t)(done - 1) * P.ld_s, (T)alpha_cur, S, P.ld_s,
                          P.full_reorth ? done : 0, S + (int64_t)done * P.ld_s, 0};
        } else {
            h = PkHalf<T>{S + (int64_t)done * P.ld_s, Q + (int64_t)(done - 1) * P.ld_q, (T)t_new, Q, P.ld_q, done,
                          Q + (int64_t)done * P.ld_q, 1};
        }
        double aux = 0.0;
        const double val = pk_half<T, VEC, MAXG>(P, h, sm, aux, grid);
        if (step == 0) {
            const double a1 = val;
            zeta_last = a1 * t1;
            alpha_cur = a1;
            if (rec) {
                P.ts[0] = t1;
                P.alphas[0] = a1;
                P.zetas[0] = zeta_last;
                P.nus[0] = nu_last;
            }
            if (t1 == 0.0) err = 1;
            else if (a1 == 0.0) err = 2;
            if (err) {
                stop = 1;
                break;
            }
            continue;
        }
        if (step & 1) {
            t_new = val;
            u2 = aux;
            continue;
        }
        const double a_new = val, p2 = aux;
        // control (identical in every CTA; CTA 0 records the trace)
        if (t_new <= P.tol * sqrt(u2)) {
            breakdown = tbreak = 1;
            stop = 1;
        } else if (a_new <= P.tol * sqrt(p2)) {
            breakdown = 1;
            if (rec) P.ts[nt] = t_new;
            ++nt;
            stop = 1;
        } else {
            if (rec) {
                P.ts[nt] = t_new;
                P.alphas[na] = a_new;
            }
            ++nt;
            ++na;
            const double zeta = a_new * t_new;
            const double nu = sqrt(zeta * zeta_last);
            if (rec) {
                P.zetas[nn] = zeta;
                P.nus[nn] = nu;
            }
            ++nn;
            zeta_last = zeta;
            const double nu_prev = nu_last;
            nu_last = nu;
            alpha_cur = a_new;
            ++done;
            if (fired < 0) {
                if (nu > nu_prev) {
                    fired = max(done - 1, P.k_min);
                    reason = KB_STOP_NU_ROSE;
                } else if (nu < P.tau) {
                    fired = max(done, P.k_min);
                    reason = KB_STOP_NU_BELOW_TOL;
                }
            }
            const int limit = fired >= 0 ? fired + P.p + 1 : P.k_max + 1;
            if (done >= limit) stop = 1;
            if (done + 1 > P.cap) {
                stop = 1;
                overflow = 1;
            }
        }
        if (stop) break;
    }
    if (rec) {
        int* h = P.hdr;
        h[PH_DONE] = done;
        h[PH_FIRED] = fired;
        h[PH_REASON] = reason;
        h[PH_STOP] = stop;
        h[PH_BREAK] = breakdown;
        h[PH_TBREAK] = tbreak;
        h[PH_OVERFLOW] = overflow;
        h[PH_ERR] = err;
        h[PH_NA] = na;
        h[PH_NT] = nt;
        h[PH_NN] = nn;
    }
}

// ------------------------------------------------------------------ tiled variant
// Zero BC, fp32, n a multiple of 128 (or a divisor of 128).  Same recurrence
// with four grid synchronisations per half step (three when there is nothing
// to project against) instead of five, and no pass that re-reads the input
// vector for its diagonal sums:
//
//   A  z        : z = K^T w (or K w), one contiguous row dot product per entry
//      -- grid.sync
//   B  dots     : y = P z ; v = y - beta*prev ; h = S^T v ; |v|^2 ; |y|^2
//      -- grid.sync + reduction
//   C  apply    : v1 = v - S h ; |v1|^2                (v kept in registers)
//      -- grid.sync + reduction (t = |v1|)
//   D  store    : x = fl(v1 / t) (lowrank.py:247, 260) stored, and the
//                 diagonal sums w of x for the NEXT product, from registers
//      -- grid.sync
//
// Each CTA owns whole 1024-element tiles of the n x n image (8*RW rows x TW
// columns, one float4 per thread, column-block-major tile order, balanced
// contiguous tile ranges), so its diagonal sums are compact: the tile values
// go through shared memory, each thread sums one diagonal of the CTA's tile
// stack, and the sums are added to the global w with 64-bit integer atomics
// in fixed point (entries of a unit vector are <= 1: scale 2^(61 - log2 n),
// so no sum can overflow).  Integer addition is exact, so w does not depend
// on the order of the atomics: the run stays deterministic without per-CTA
// partial arrays, and every fp32 entry above 2^-(61 - log2 n) enters the
// sum exactly (w is at least as accurate as an fp64 summation).

// ---- per-thread copy ring: each thread streams its own float4 of every owned
// tile of the next basis vectors into shared memory with cp.async (16 B,
// L2 only), PK_NS vectors ahead, so the dots / projection loops keep many
// vectors in flight without holding them in registers.  A thread reads back
// only what it copied itself: no cross-thread synchronisation is needed.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}

__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// ring stages (basis vectors in flight per thread): 4 with <= 4 owned tiles
// per thread; with more tiles one stage already keeps 8-16 float4 per thread
// in flight, and the ring shares the tile buffer (used only in phase D)
template <int MAXG>
__host__ __device__ constexpr int pk_ns() { return MAXG <= 4 ? 4 : (MAXG <= 8 ? 2 : 1); }

// Item G of the thread's stream (stage G % NS) <- its float4 of each owned tile of `vec`
// (vec == nullptr: an empty group, keeps the group accounting uniform).
template <int MAXG, int NS>
__device__ __forceinline__ void ring_fill(float* ring, int stage_floats, int tbo, unsigned G, const float* vec,
                                          const int (&eo)[MAXG], int ng) {
    if (vec) {
        float* dst = ring + (int)(G % NS) * stage_floats + tbo;
#pragma unroll
        for (int g = 0; g < MAXG; ++g)
            if (g < ng) cp_async16(dst + g * 1024, vec + eo[g]);
    }
    cp_async_commit();
}

// ---- exact grid sums without a partial array: every CTA adds its fp64 partial,
// scaled by 2^79, as three 40-bit integer limbs (trunc toward zero, so each
// limb carries the value's sign) with 64-bit integer REDs; integer addition is
// exact and order-free, <= 2^9 CTAs leave 24 bits of headroom per limb, and
// |partial| < 2^39 is far above anything a half step produces.  After the
// grid sync each CTA reads the 3 limb sums (one line) and recombines them in
// a fixed order: deterministic, and at least as accurate as an fp64 tree.
constexpr int XACC_S = 79;
__device__ __forceinline__ void xacc_add(long long* acc3, double x) {
    const double y = ldexp(x, XACC_S);
    const double hi = trunc(ldexp(y, -80));
    const double r1 = y - ldexp(hi, 80);          // exact: multiples of ulp(y), |r1| < 2^80
    const double mid = trunc(ldexp(r1, -40));
    const double r2 = r1 - ldexp(mid, 40);        // exact, |r2| < 2^40
    const long long lo = __double2ll_rn(r2);
    if (hi != 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(acc3 + 0), (unsigned long long)(long long)hi);
    if (mid != 0.0) atomicAdd(reinterpret_cast<unsigned long long*>(acc3 + 1), (unsigned long long)(long long)mid);
    if (lo != 0) atomicAdd(reinterpret_cast<unsigned long long*>(acc3 + 2), (unsigned long long)lo);
}
__device__ __forceinline__ double xacc_get(const long long* acc3) {
    const long long h = (long long)__ldcg(reinterpret_cast<const unsigned long long*>(acc3 + 0));
    const long long m = (long long)__ldcg(reinterpret_cast<const unsigned long long*>(acc3 + 1));
    const long long l = (long long)__ldcg(reinterpret_cast<const unsigned long long*>(acc3 + 2));
    return ldexp(ldexp((double)h, 80) + ldexp((double)m, 40) + (double)l, -XACC_S);
}

// Grid barrier of the tiled kernel: each CTA's thread 0 posts ONE release-add on a
// monotonically increasing arrival counter (bar[0], zeroed before the launch) and polls
// it with acquire loads until every CTA of this barrier generation has arrived.  No
// returning atomic and no generation flip by a master CTA: one L2 round trip fewer on
// the critical path than grid.sync().  The CTA barriers on both sides carry the other
// threads' writes (before) and the acquired view (after), as in grid.sync().
__device__ __forceinline__ void pk_grid_sync(const PkParams& P, unsigned& gen) {
    gen += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* ctr = P.bar;
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(ctr) : "memory");
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
        } while ((int)(v - gen) < 0);
    }
    __syncthreads();
}

// The same barrier in two halves, so that work which does not depend on the other CTAs can
// run between the arrival and the wait (it hides behind the slowest CTA).
__device__ __forceinline__ void pk_grid_arrive(const PkParams& P, unsigned& gen) {
    gen += gridDim.x;
    __syncthreads();
    if (threadIdx.x == 0) asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(P.bar) : "memory");
}
__device__ __forceinline__ void pk_grid_wait(const PkParams& P, unsigned gen) {
    if (threadIdx.x == 0) {
        unsigned v;
        do {
            asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(P.bar) : "memory");
        } while ((int)(v - gen) < 0);
    }
    __syncthreads();
}

struct TileGeo {
    int TW, LR, RW, RB, T;   // tile width, lanes per row, rows per warp, row blocks, tiles
};

__device__ __forceinline__ void tile_range(int T, int b, int nblk, int& t0, int& ng) {
    t0 = (int)((int64_t)T * b / nblk);
    ng = (int)((int64_t)T * (b + 1) / nblk) - t0;
}

// fixed-point exponent for entries bounded by 2|v|: sums of <= n of them stay < 2^62
__device__ __forceinline__ int pk_fix_exp(double vnorm, int n) {
    int e = 0;
    if (!(vnorm > 0.0) || !isfinite(vnorm)) return 0;
    frexp(2.0 * vnorm, &e);   // 2|v| < 2^e
    int ln = 0;
    while ((1 << ln) < n) ++ln;
    return 62 - ln - e;
}


// Diagonal sums of the CTA's register-held tile values (staged in tb) for a
// product with diagonal offset ci and Li diagonals, added in fixed point to wf.
template <int MAXG>
__device__ __forceinline__ void tile_diag_atomics(const PkParams& P, const TileGeo& Gm, const float* tb, int t0,
                                                  int ng, int ci, int Li, double scale, unsigned long long* wf) {
    const int n = P.n, R = 8 * Gm.RW;
    int g = 0;
    while (g < ng) {
        const int cb = (t0 + g) / Gm.RB, rb0 = (t0 + g) - cb * Gm.RB;
        int h = 1;
        while (g + h < ng && (t0 + g + h) / Gm.RB == cb) ++h;     // stack of h tiles in column block cb
        const int A0 = rb0 * R, A1 = A0 + h * R, C0 = cb * Gm.TW;
        const float* sb = tb + g * 1024;                           // stack rows, row-major, TW wide
        const int dlo = C0 - (A1 - 1), nd = Gm.TW + h * R - 1;
        for (int i = threadIdx.x; i < nd; i += PK_THREADS) {
            const int d = dlo + i, u = d + ci;
            if (u < 0 || u >= Li) continue;
            const int a_lo = max(A0, C0 - d), a_hi = min(A1, C0 + Gm.TW - d);
            // x * 2^F is exact in fp32 (a power of two, |x| <= 1, F <= 60), and its
            // round-to-nearest integer equals __double2ll_rn((double)x * 2^F): one
            // conversion per entry; 8 entries in flight along the diagonal
            const float fs = (float)scale;
            const float* pd = sb + (a_lo - A0) * Gm.TW + (a_lo + d - C0);
            const int len = a_hi - a_lo, step = Gm.TW + 1;
            long long s = 0;
            int k = 0;
            for (; k + 8 <= len; k += 8) {
                float q[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) q[j] = pd[(k + j) * step];
#pragma unroll
                for (int j = 0; j < 8; ++j) s += __float2ll_rn(q[j] * fs);
            }
            for (; k < len; ++k) s += __float2ll_rn(pd[k * step] * fs);
            if (s != 0) atomicAdd(wf + u, (unsigned long long)s);
        }
        g += h;
    }
    (void)n;
}

// z[c] = sum_r Mt[c, r] w(r) for this CTA's rows c in [b Lo / grid, (b+1) Lo / grid):
// Mt is K^T for the forward product (z = K^T w) and K for the transpose, so
// every z entry is ONE contiguous row dot product (warp per row, lanes over
// r, fixed order): no column partials, no second pass.  w is staged in
// shared memory; its loads and the first batch of row loads are issued
// together (one L2 round trip).
__device__ __forceinline__ void pk_zrows(const PkParams& P, const float* Mt, int Li, int Lo, double* ws,
                                         const unsigned long long* wsrc, double s2) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int c0 = (int)((int64_t)Lo * blockIdx.x / gridDim.x), c1 = (int)((int64_t)Lo * (blockIdx.x + 1) / gridDim.x);
    constexpr int RB = 32;   // row loads in flight per lane
    float mk[RB];
    const int c_first = c0 + warp;
    if (c_first < c1) {
        const float* row = Mt + (int64_t)c_first * Li;
#pragma unroll
        for (int k = 0; k < RB; ++k) mk[k] = (lane + 32 * k < Li) ? __ldg(row + lane + 32 * k) : 0.f;
    }
    // w(r) = wfix[r] * 2^-F, all loads in flight before the stores
    for (int r0 = tid; r0 < Li; r0 += 8 * PK_THREADS) {
        long long q[8];
#pragma unroll
        for (int k = 0; k < 8; ++k) q[k] = r0 + k * PK_THREADS < Li ? (long long)__ldcg(wsrc + r0 + k * PK_THREADS) : 0;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            if (r0 + k * PK_THREADS < Li) ws[r0 + k * PK_THREADS] = (double)q[k] * s2;
    }
    pk_mark(P, 9);
    __syncthreads();
    pk_mark(P, 10);
    for (int c = c_first; c < c1; c += PK_THREADS / 32) {
        const float* row = Mt + (int64_t)c * Li;
        if (c != c_first) {
#pragma unroll
            for (int k = 0; k < RB; ++k) mk[k] = (lane + 32 * k < Li) ? __ldg(row + lane + 32 * k) : 0.f;
        }
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < RB; ++k)
            if (lane + 32 * k < Li) a += (double)mk[k] * ws[lane + 32 * k];
        for (int r0 = 32 * RB; r0 < Li; r0 += 32 * RB) {        // long rows (Li > 1024)
#pragma unroll
            for (int k = 0; k < RB; ++k) mk[k] = (r0 + lane + 32 * k < Li) ? __ldg(row + r0 + lane + 32 * k) : 0.f;
#pragma unroll
            for (int k = 0; k < RB; ++k)
                if (r0 + lane + 32 * k < Li) a += (double)mk[k] * ws[r0 + lane + 32 * k];
        }
        a = warp_sum(a);
        if (lane == 0) __stcg(P.zbuf + c, a);
    }
}

// x = fl(v / t) for the register-held tile values: stored to `out`, staged
// in shared memory, and its fixed-point diagonal sums added to wf.
template <int MAXG>
__device__ __forceinline__ void pk_store_diag(const PkParams& P, const TileGeo& Gm, float (&v)[MAXG][4], float td,
                                              float* out, const int (&eo)[MAXG], int ng, float* tb, int tbo, int t0,
                                              int ci, int Li, double fxs, unsigned long long* wf) {
    const double rtd = 1.0 / (double)td;
#pragma unroll
    for (int g = 0; g < MAXG; ++g)
        if (g < ng) {
            float o[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) o[q] = pk_fdiv_exact(v[g][q], td, rtd);
            PkIO<float, 4>::store(out + eo[g], o);
            *reinterpret_cast<float4*>(tb + g * 1024 + tbo) = make_float4(o[0], o[1], o[2], o[3]);
        }
    __syncthreads();
    pk_mark(P, 12);
    tile_diag_atomics<MAXG>(P, Gm, tb, t0, ng, ci, Li, fxs, wf);
    pk_mark(P, 13);
}

// DEFER: the normalisation of a projected vector is deferred by one phase, so phases C and D
// share one grid synchronisation (3 per half step instead of 4): the diagonal sums for the
// next product are taken from the UNNORMALISED v1 (fixed point scaled by a power of two
// >= 2 |v|) in the same phase that accumulates |v1|^2, the next phase A reads them as
// w / t, and x = fl(v1 / t) is stored from registers at the start of that phase A.
template <int MAXG, bool DEFER>
__global__ void __launch_bounds__(PK_THREADS, 2) k_egkb_tiled(PkParams P, TileGeo Gm) {
    cg::grid_group grid = cg::this_grid();
    unsigned gen = 0;
    auto gsync = [&]() {
        if (P.cg_sync & 1) grid.sync();
        else pk_grid_sync(P, gen);
    };
    extern __shared__ double sm[];
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = P.n;
    const int nblk = gridDim.x;
    float* S = static_cast<float*>(P.S);
    float* Q = static_cast<float*>(P.Q);
    const float* y0 = static_cast<const float*>(P.y0);
    double* zs = sm;                               // [lmax]
    double* red = zs + P.lmax;                     // [cap + 4]
    double* acc = red + P.cap + 4;                 // [8][max(cap + 2, 33)]
    float* tb = reinterpret_cast<float*>(acc + 8 * max(P.cap + 2, 33));   // [MAXG * 1024]
    // basis streaming ring: NS stages after the tile buffer (MAXG <= 4) or over it
    constexpr int PK_NS = pk_ns<MAXG>();
    float* ringb = MAXG <= 4 ? tb + MAXG * 1024 : tb;
    constexpr int SF = MAXG * 1024;                // floats per stage
    const bool rec = (blockIdx.x == 0 && tid == 0);
    const int cu = P.kh / 2, cv = P.kw / 2;

    // element offsets of this thread (one float4 per tile)
    int t0, ng;
    tile_range(Gm.T, blockIdx.x, nblk, t0, ng);
    int eo[MAXG];
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
        const int t = min(t0 + g, Gm.T - 1);
        const int cb = t / Gm.RB, rb = t - cb * Gm.RB;
        const int a = rb * 8 * Gm.RW + warp * Gm.RW + lane / Gm.LR;
        eo[g] = a * n + cb * Gm.TW + (lane % Gm.LR) * 4;
    }
    const int tbo = warp * 128 + lane * 4;         // this thread's float4 inside a staged tile
    unsigned rbase = 0;                            // items streamed so far (uniform)
    // ---- prologue: v <- y0, t1 = |y0|, diagonal sums of y0 for step 0 (R^T, q side)
    float v[MAXG][4];
    double vsq = 0.0;
#pragma unroll
    for (int g = 0; g < MAXG; ++g) {
        if (g < ng) {
            PkIO<float, 4>::load(y0 + eo[g], v[g]);
#pragma unroll
            for (int q = 0; q < 4; ++q) vsq += (double)v[g][q] * (double)v[g][q];
        } else {
#pragma unroll
            for (int q = 0; q < 4; ++q) v[g][q] = 0.f;
        }
    }
    vsq = warp_sum(vsq);
    if (lane == 0) acc[warp] = vsq;
    __syncthreads();
    long long* xdot = P.xacc;                       // [cap + 4][3]: dots / |v|^2 / |y|^2
    long long* xnrm = P.xacc + 3 * (P.cap + 4);     // [3]: |v1|^2 (and |y0|^2)
    if (tid == 0) {
        double s = 0.0;
#pragma unroll
        for (int w = 0; w < 8; ++w) s += acc[w];
        xacc_add(xnrm, s);
    }
    gsync();
    if (tid == 0) red[0] = xacc_get(xnrm);
    __syncthreads();
    pk_mark(P, 1);
    const double t1 = sqrt(red[0]);
    // entries of a normalised vector are <= 1: one fixed-point scale for the run
    const int Fx = pk_fix_exp(0.5, n);
    const double fxs = ldexp(1.0, Fx), fxs_inv = ldexp(1.0, -Fx);
    // s1 = fl(y0 / t1) (lowrank.py:207-210), stored, and its diagonal sums for step 0 (R^T)
    pk_store_diag<MAXG>(P, Gm, v, (float)t1, S, eo, ng, tb, tbo, t0, cv, P.kw, fxs, P.wfix);
    gsync();
    pk_mark(P, 2);

    int done = 1, fired = -1, reason = 0, stop = 0, breakdown = 0, tbreak = 0, overflow = 0, err = 0;
    int na = 1, nt = 1, nn = 1;
    double zeta_last = 0.0, nu_last = 1e308, alpha_cur = 0.0, t_new = 0.0, u2 = 0.0;
    if (t1 == 0.0) {
        err = 1;
        stop = 1;
    }
    // DEFER: the vector held in v is still unnormalised (norm pend_t, destination pend_out);
    // wscale turns the fixed-point diagonal sums of the current product's input into w
    bool pend = false;
    float pend_t = 1.f;
    float* pend_out = nullptr;
    double wscale = fxs_inv;
    auto store_pending = [&]() {
        const double rtd = 1.0 / (double)pend_t;
#pragma unroll
        for (int g = 0; g < MAXG; ++g)
            if (g < ng) {
                // v1 is read back from the tile buffer (staged there for the diagonal sums), so
                // no register holds it across phase A
                const float4 u = *reinterpret_cast<const float4*>(tb + g * 1024 + tbo);
                float o[4];
                o[0] = pk_fdiv_exact(u.x, pend_t, rtd);
                o[1] = pk_fdiv_exact(u.y, pend_t, rtd);
                o[2] = pk_fdiv_exact(u.z, pend_t, rtd);
                o[3] = pk_fdiv_exact(u.w, pend_t, rtd);
                PkIO<float, 4>::store(pend_out + eo[g], o);
            }
        pend = false;
    };
    for (int step = 0; !stop; ++step) {
        const int tr = (step & 1) ? 0 : 1;           // step 0 and even steps: q side (R^T)
        const float* prev;
        float beta;
        const float* B;
        int m;
        float* out;
        if (step == 0) {
            prev = nullptr; beta = 0.f; B = Q; m = 0; out = Q;
        } else if (tr == 0) {
            prev = S + (int64_t)(done - 1) * P.ld_s; beta = (float)alpha_cur; B = S;
            m = P.full_reorth ? done : 0; out = S + (int64_t)done * P.ld_s;
        } else {
            prev = Q + (int64_t)(done - 1) * P.ld_q; beta = (float)t_new; B = Q; m = done;
            out = Q + (int64_t)done * P.ld_q;
        }
        const int64_t ldb = tr ? P.ld_q : P.ld_s;
        const int Li = tr ? P.kw : P.kh;
        const int co = tr ? cu : cv, Lo = tr ? P.kh : P.kw;
        const float* Mt = static_cast<const float*>(tr ? P.K : P.Kt);   // rows of M^T (M = K or K^T)
        unsigned long long* wcur = P.wfix + (int64_t)(step & 1) * P.lmax;

        // the accumulators were last read before the previous phase's sync: reset them
        // (DEFER: |v1|^2 alternates between two accumulators, each reset two phases after its read)
        if (blockIdx.x == 0)
            for (int j = tid; j < 3 * (P.cap + (DEFER ? 4 : 5)); j += PK_THREADS) P.xacc[j] = 0;

        // ---- A: z rows from the diagonal sums of the input vector.  The ring
        // starts fetching the first basis vectors of the dots (phase B) now.
        if constexpr (MAXG > 4 && !DEFER) {   // (MAXG <= 4: issued during the previous step's phase D)
            if (m > 0)
#pragma unroll
                for (int k = 0; k < PK_NS; ++k)
                    ring_fill<MAXG, PK_NS>(ringb, SF, tbo, rbase + k, k < 2 * m ? B + (int64_t)(k % m) * ldb : nullptr, eo, ng);
        }
        pk_mark(P, 7);
        pk_zrows(P, Mt, Li, Lo, zs, wcur, wscale);
        pk_mark(P, 8);
        // prefetch prev (used right after the barrier) while the grid synchronises
        float pv[MAXG][4];
#pragma unroll
        for (int g = 0; g < MAXG; ++g) {
#pragma unroll
            for (int q = 0; q < 4; ++q) pv[g][q] = 0.f;
            if (g < ng && prev) PkIO<float, 4>::load(prev + eo[g], pv[g]);
        }
        auto prefill = [&]() {   // the first basis vectors of the dots (phase B)
            if (m > 0)
#pragma unroll
                for (int k = 0; k < PK_NS; ++k)
                    ring_fill<MAXG, PK_NS>(ringb, SF, tbo, rbase + k, k < 2 * m ? B + (int64_t)(k % m) * ldb : nullptr, eo, ng);
        };
        if constexpr (DEFER) {
            if constexpr (MAXG <= 4) prefill();   // (the ring does not share the tile buffer)
            if constexpr (MAXG > 4) {
                if (pend) store_pending();
                prefill();
            }
        }
        gsync();
        pk_mark(P, 3);

        // ---- B: zero the consumed w; z; y; v = y - beta*prev; dots
        for (int i = blockIdx.x * PK_THREADS + tid; i < P.lmax; i += nblk * PK_THREADS) wcur[i] = 0ull;
        if constexpr (DEFER) {
            if (blockIdx.x == 0 && tid < 3) xnrm[3 * ((step + 1) & 1) + tid] = 0;
        }
        // z staged already rounded to fp32: y = fl32(z[u]) for every cell of a diagonal,
        // so one conversion per diagonal instead of one per cell
        float* zsf = reinterpret_cast<float*>(zs);
        for (int c0 = tid; c0 < Lo; c0 += 8 * PK_THREADS) {
            double q[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) q[k] = c0 + k * PK_THREADS < Lo ? __ldcg(P.zbuf + c0 + k * PK_THREADS) : 0.0;
#pragma unroll
            for (int k = 0; k < 8; ++k)
                if (c0 + k * PK_THREADS < Lo) zsf[c0 + k * PK_THREADS] = (float)q[k];
        }
        const int W = m + 2;
        for (int i = tid; i < 8 * W; i += PK_THREADS) acc[i] = 0.0;
        __syncthreads();
        pk_mark(P, 11);
        float ysqf = 0.f;   // |y|^2 only feeds the breakdown threshold: fp32 per thread
        vsq = 0.0;
#pragma unroll
        for (int g = 0; g < MAXG; ++g) {
            if (g < ng) {
                const int a = eo[g] / n, b0 = eo[g] - a * n;   // 4 cells of one image row
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const int u = b0 + q - a + co;
                    const float yv = (u >= 0 && u < Lo) ? zsf[u] : 0.f;
                    ysqf = fmaf(yv, yv, ysqf);
                    v[g][q] = __fsub_rn(yv, __fmul_rn(beta, pv[g][q]));
                }
            } else {
#pragma unroll
                for (int q = 0; q < 4; ++q) v[g][q] = 0.f;
            }
        }
        {
            // items rbase .. rbase + m - 1 of the stream: the basis vectors in order, two per
            // iteration (independent FMA chains and warp sums; per vector the same order of
            // operations as one at a time, so the sums are bit-identical)
            int i = 0;
            if constexpr (PK_NS >= 4) {
                for (; i + 2 <= m; i += 2) {
                    const unsigned G = rbase + i;
                    cp_async_wait<PK_NS - 2>();
                    const float* sb0 = ringb + (int)(G % PK_NS) * SF + tbo;
                    const float* sb1 = ringb + (int)((G + 1) % PK_NS) * SF + tbo;
                    float dt0 = 0.f, dt1 = 0.f;
#pragma unroll
                    for (int g = 0; g < MAXG; ++g)
                        if (g < ng) {
                            const float4 s0 = *reinterpret_cast<const float4*>(sb0 + g * 1024);
                            const float4 s1 = *reinterpret_cast<const float4*>(sb1 + g * 1024);
                            dt0 = fmaf(s0.x, v[g][0], dt0);
                            dt1 = fmaf(s1.x, v[g][0], dt1);
                            dt0 = fmaf(s0.y, v[g][1], dt0);
                            dt1 = fmaf(s1.y, v[g][1], dt1);
                            dt0 = fmaf(s0.z, v[g][2], dt0);
                            dt1 = fmaf(s1.z, v[g][2], dt1);
                            dt0 = fmaf(s0.w, v[g][3], dt0);
                            dt1 = fmaf(s1.w, v[g][3], dt1);
                        }
                    ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + PK_NS,
                                           i + PK_NS < 2 * m ? B + (int64_t)((i + PK_NS) % m) * ldb : nullptr, eo, ng);
                    ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + 1 + PK_NS,
                                           i + 1 + PK_NS < 2 * m ? B + (int64_t)((i + 1 + PK_NS) % m) * ldb : nullptr, eo, ng);
                    const double d0 = warp_sum((double)dt0), d1 = warp_sum((double)dt1);
                    if (lane == 0) {
                        acc[warp * W + i] += d0;
                        acc[warp * W + i + 1] += d1;
                    }
                }
            }
            for (; i < m; ++i) {
                const unsigned G = rbase + i;
                cp_async_wait<PK_NS - 1>();
                const float* sb = ringb + (int)(G % PK_NS) * SF + tbo;
                float dt = 0.f;
#pragma unroll
                for (int g = 0; g < MAXG; ++g)
                    if (g < ng) {
                        const float4 sv = *reinterpret_cast<const float4*>(sb + g * 1024);
                        dt = fmaf(sv.x, v[g][0], dt);
                        dt = fmaf(sv.y, v[g][1], dt);
                        dt = fmaf(sv.z, v[g][2], dt);
                        dt = fmaf(sv.w, v[g][3], dt);
                    }
                ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + PK_NS, i + PK_NS < 2 * m ? B + (int64_t)((i + PK_NS) % m) * ldb : nullptr,
                                eo, ng);
                const double d = warp_sum((double)dt);
                if (lane == 0) acc[warp * W + i] += d;
            }
        }
#pragma unroll
        for (int g = 0; g < MAXG; ++g)
#pragma unroll
            for (int q = 0; q < 4; ++q) vsq += (double)v[g][q] * (double)v[g][q];
        vsq = warp_sum(vsq);
        const double ysq = warp_sum((double)ysqf);
        if (lane == 0) {
            acc[warp * W + m] += vsq;
            acc[warp * W + m + 1] += ysq;
        }
        __syncthreads();
        pk_mark(P, 15);
        for (int j = tid; j < W; j += PK_THREADS) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t += acc[w * W + j];
            xacc_add(xdot + 3 * j, t);
        }
        if (DEFER && MAXG <= 4 && pend && !(P.cg_sync & 1)) {
            // x = fl(v1 / t) of the previous half step, stored between the arrival and the
            // wait (nothing reads it before the next half step's barriers)
            pk_grid_arrive(P, gen);
            store_pending();
            pk_grid_wait(P, gen);
        } else {
            if (DEFER && pend) store_pending();
            gsync();
        }
        for (int j = tid; j < W; j += PK_THREADS) red[j] = xacc_get(xdot + 3 * j);
        __syncthreads();
        pk_mark(P, 4);
        const double aux = red[m + 1];
        const double vnorm = sqrt(red[m]);

        // ---- C: v1 = v - S h ; t = |v1|
        double val;
        const int ci_n = tr ? cu : cv, Li_n = tr ? P.kh : P.kw;   // next product: the other side
        unsigned long long* wnext = P.wfix + (int64_t)((step + 1) & 1) * P.lmax;
        if (m == 0) {
            val = vnorm;
        } else {
            float* cf = reinterpret_cast<float*>(acc);
            for (int i = tid; i < m; i += PK_THREADS) cf[i] = (float)red[i];
            __syncthreads();
            double v1sq = 0.0;
            {
                // items rbase + m .. rbase + 2m - 1: the same basis vectors again, two per
                // iteration (one wait and eight loads in flight; per element the same order)
                int i = 0;
                if constexpr (PK_NS >= 4) {
                    for (; i + 2 <= m; i += 2) {
                        const unsigned G = rbase + m + i;
                        cp_async_wait<PK_NS - 2>();
                        const float* sb0 = ringb + (int)(G % PK_NS) * SF + tbo;
                        const float* sb1 = ringb + (int)((G + 1) % PK_NS) * SF + tbo;
                        const float c0 = cf[i], c1 = cf[i + 1];
#pragma unroll
                        for (int g = 0; g < MAXG; ++g)
                            if (g < ng) {
                                const float4 s0 = *reinterpret_cast<const float4*>(sb0 + g * 1024);
                                const float4 s1 = *reinterpret_cast<const float4*>(sb1 + g * 1024);
                                v[g][0] = fmaf(-c1, s1.x, fmaf(-c0, s0.x, v[g][0]));
                                v[g][1] = fmaf(-c1, s1.y, fmaf(-c0, s0.y, v[g][1]));
                                v[g][2] = fmaf(-c1, s1.z, fmaf(-c0, s0.z, v[g][2]));
                                v[g][3] = fmaf(-c1, s1.w, fmaf(-c0, s0.w, v[g][3]));
                            }
                        ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + PK_NS,
                                               i + PK_NS < m ? B + (int64_t)(i + PK_NS) * ldb : nullptr, eo, ng);
                        ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + 1 + PK_NS,
                                               i + 1 + PK_NS < m ? B + (int64_t)(i + 1 + PK_NS) * ldb : nullptr, eo, ng);
                    }
                }
                for (; i < m; ++i) {
                    const unsigned G = rbase + m + i;
                    cp_async_wait<PK_NS - 1>();
                    const float* sb = ringb + (int)(G % PK_NS) * SF + tbo;
                    const float c = cf[i];
#pragma unroll
                    for (int g = 0; g < MAXG; ++g)
                        if (g < ng) {
                            const float4 sv = *reinterpret_cast<const float4*>(sb + g * 1024);
                            v[g][0] = fmaf(-c, sv.x, v[g][0]);
                            v[g][1] = fmaf(-c, sv.y, v[g][1]);
                            v[g][2] = fmaf(-c, sv.z, v[g][2]);
                            v[g][3] = fmaf(-c, sv.w, v[g][3]);
                        }
                    ring_fill<MAXG, PK_NS>(ringb, SF, tbo, G + PK_NS, i + PK_NS < m ? B + (int64_t)(i + PK_NS) * ldb : nullptr,
                                    eo, ng);
                }
#pragma unroll
                for (int g = 0; g < MAXG; ++g)
#pragma unroll
                    for (int q = 0; q < 4; ++q) v1sq += (double)v[g][q] * (double)v[g][q];
            }
            rbase += 2 * m;
            v1sq = warp_sum(v1sq);
            long long* xn = DEFER ? xnrm + 3 * (step & 1) : xnrm;
            if constexpr (DEFER) {
                // the diagonal sums of the unnormalised v1 for the next product, in fixed point
                // scaled for entries below 2 |v| (|v1| <= |v| up to rounding)
                const int Fp = max(-100, min(100, pk_fix_exp(vnorm, n)));
#pragma unroll
                for (int g = 0; g < MAXG; ++g)
                    if (g < ng)
                        *reinterpret_cast<float4*>(tb + g * 1024 + tbo) = make_float4(v[g][0], v[g][1], v[g][2], v[g][3]);
                wscale = ldexp(1.0, -Fp);
                __syncthreads();   // cf (in acc) is read until every warp has finished the projection
                if (lane == 0) acc[warp] = v1sq;
                __syncthreads();
                if (tid == 0) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) s += acc[w];
                    xacc_add(xn, s);
                }
                if (!(P.cg_sync & 2)) tile_diag_atomics<MAXG>(P, Gm, tb, t0, ng, ci_n, Li_n, ldexp(1.0, Fp), wnext);
            } else {
                __syncthreads();   // cf (in acc) is read until every warp has finished the projection
                if (lane == 0) acc[warp] = v1sq;
                __syncthreads();
                if (tid == 0) {
                    double s = 0.0;
#pragma unroll
                    for (int w = 0; w < 8; ++w) s += acc[w];
                    xacc_add(xn, s);
                }
            }
            gsync();
            if (tid == 0) red[P.cap + 2] = xacc_get(xn);
            __syncthreads();
            pk_mark(P, 5);
            val = sqrt(red[P.cap + 2]);
            if constexpr (DEFER) {
                pend = true;
                pend_t = (float)val;
                pend_out = out;
                wscale /= (double)pend_t;
            }
        }
        // ---- control (identical in every CTA; CTA 0 records the trace), before D so
        // the next step's basis vectors stream in while D runs
        if (step == 0) {
            const double a1 = val;
            zeta_last = a1 * t1;
            alpha_cur = a1;
            if (rec) {
                P.ts[0] = t1;
                P.alphas[0] = a1;
                P.zetas[0] = zeta_last;
                P.nus[0] = nu_last;
            }
            if (a1 == 0.0) {
                err = 2;
                stop = 1;
            }
        } else if (tr == 0) {
            t_new = val;
            u2 = aux;
        } else {
        const double a_new = val, p2 = aux;
        if (t_new <= P.tol * sqrt(u2)) {
            breakdown = tbreak = 1;
            stop = 1;
        } else if (a_new <= P.tol * sqrt(p2)) {
            breakdown = 1;
            if (rec) P.ts[nt] = t_new;
            ++nt;
            stop = 1;
        } else {
            if (rec) {
                P.ts[nt] = t_new;
                P.alphas[na] = a_new;
            }
            ++nt;
            ++na;
            const double zeta = a_new * t_new;
            const double nu = sqrt(zeta * zeta_last);
            if (rec) {
                P.zetas[nn] = zeta;
                P.nus[nn] = nu;
            }
            ++nn;
            zeta_last = zeta;
            const double nu_prev = nu_last;
            nu_last = nu;
            alpha_cur = a_new;
            ++done;
            if (fired < 0) {
                if (nu > nu_prev) {
                    fired = max(done - 1, P.k_min);
                    reason = KB_STOP_NU_ROSE;
                } else if (nu < P.tau) {
                    fired = max(done, P.k_min);
                    reason = KB_STOP_NU_BELOW_TOL;
                }
            }
            const int limit = fired >= 0 ? fired + P.p + 1 : P.k_max + 1;
            if (done >= limit) stop = 1;
            if (done + 1 > P.cap) {
                stop = 1;
                overflow = 1;
            }
        }
        }
        if constexpr (MAXG <= 4 && !DEFER) {   // the ring does not share the tile buffer used by D
            if (!stop) {
                const int trn = ((step + 1) & 1) ? 0 : 1;
                const float* Bn = trn ? Q : S;
                const int mn = trn ? done : (P.full_reorth ? done : 0);
                const int64_t ldn = trn ? P.ld_q : P.ld_s;
                if (mn > 0)
#pragma unroll
                    for (int k = 0; k < PK_NS; ++k)
                        ring_fill<MAXG, PK_NS>(ringb, SF, tbo, rbase + k, k < 2 * mn ? Bn + (int64_t)(k % mn) * ldn : nullptr,
                                               eo, ng);
            }
        }
        // ---- D: out = fl(v1 / t) (lowrank.py:247, 260), stored, and its diagonal
        // sums for the next product
        pk_mark(P, 14);
        if (!pend) {
            pk_store_diag<MAXG>(P, Gm, v, (float)val, out, eo, ng, tb, tbo, t0, ci_n, Li_n, fxs, wnext);
            wscale = fxs_inv;
            gsync();
        } else if (stop) {
            store_pending();
        }
        pk_mark(P, 6);

        if (stop) break;
    }
    if (rec) {
        int* h = P.hdr;
        h[PH_DONE] = done;
        h[PH_FIRED] = fired;
        h[PH_REASON] = reason;
        h[PH_STOP] = stop;
        h[PH_BREAK] = breakdown;
        h[PH_TBREAK] = tbreak;
        h[PH_OVERFLOW] = overflow;
        h[PH_ERR] = err;
        h[PH_NA] = na;
        h[PH_NT] = nt;
        h[PH_NN] = nn;
    }
}

// ------------------------------------------------------------------ host side
constexpr int PK_MAXG_F32 = 16, PK_MAXG_F64 = 16;

template <typename T, int VEC, int MAXG>
static bool pk_launch(PkParams& P, cudaStream_t st, int& grid_out) {
    auto kern = k_egkb_persistent<T, VEC, MAXG>;
    const size_t smem =
        sizeof(double) * ((size_t)P.lmax + (P.cap + 4) + 8 * (size_t)std::max(P.cap + 2, 33) + 64);
    static bool configured = false;
    if (!configured) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
        configured = true;
    }
    // occupancy and SM count depend only on the device and the smem size: queried once
    static int dev = -1, sms = 0;
    static size_t smem_cached = 0;
    static int per_sm = 0;
    int cur = 0;
    KB_CUDA(cudaGetDevice(&cur));
    if (cur != dev || smem != smem_cached) {
        KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PK_THREADS, smem));
        KB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur));
        dev = cur;
        smem_cached = smem;
        if (std::getenv("KB_DEBUG")) fprintf(stderr, "[kb] persistent eGKB: %d CTAs/SM, smem %zu\n", per_sm, smem);
    }
    if (per_sm < 1) return false;
    const int grid = sms * std::min(per_sm, 2);
    const int64_t N = (int64_t)P.n * P.n;
    const int64_t per = (int64_t)grid * PK_THREADS * VEC;
    P.ng = (int)((N + per - 1) / per);
    if (P.ng > MAXG) return false;
    void* args[] = {&P};
    ProfScope ps(st, PROF_REORTH, 0.0);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(PK_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    (void)args;
    KB_CUDA(cudaMemsetAsync(P.bar, 0, sizeof(unsigned) * P.nbar, st));
    KB_CUDA(cudaLaunchKernelEx(&lc, kern, P));
    grid_out = grid;
    return true;
}

template <int MAXG, bool DEFER>
static bool tiled_launch_g(PkParams& P, const TileGeo& Gm, int per_sm_cap, cudaStream_t st) {
    auto kern = k_egkb_tiled<MAXG, DEFER>;
    const size_t smem = sizeof(double) * ((size_t)P.lmax + (P.cap + 4) + 8 * (size_t)std::max(P.cap + 2, 33)) +
                        sizeof(float) * 1024 * MAXG * (MAXG <= 4 ? 1 + pk_ns<MAXG>() : pk_ns<MAXG>());
    static bool configured = false;
    if (!configured) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 110 * 1024));
        configured = true;
    }
    if (smem > 110 * 1024) return false;
    static int dev = -1, sms = 0;
    static size_t smem_cached = 0;
    static int per_sm = 0;
    int cur = 0;
    KB_CUDA(cudaGetDevice(&cur));
    if (cur != dev || smem != smem_cached) {
        KB_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, PK_THREADS, smem));
        KB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, cur));
        dev = cur;
        smem_cached = smem;
        if (std::getenv("KB_DEBUG")) fprintf(stderr, "[kb] tiled eGKB<%d>: %d CTAs/SM, smem %zu\n", MAXG, per_sm, smem);
    }
    if (per_sm < 1) return false;
    static const int grid_env = std::getenv("KB_PK_GRID") ? std::atoi(std::getenv("KB_PK_GRID")) : 0;
    static const int cg_env = std::getenv("KB_PK_CGSYNC") ? std::atoi(std::getenv("KB_PK_CGSYNC")) : 0;
    P.cg_sync = cg_env;   // bit 0: cooperative-groups grid.sync; bit 1 (timing experiment): DEFER without its atomics
    int grid = std::min(sms * std::min(per_sm, per_sm_cap), Gm.T);
    if (grid_env > 0) grid = std::min(grid, grid_env);
    if ((Gm.T + grid - 1) / grid > MAXG) return false;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(grid);
    lc.blockDim = dim3(PK_THREADS);
    lc.dynamicSmemBytes = smem;
    lc.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    lc.attrs = attr;
    lc.numAttrs = 1;
    KB_CUDA(cudaMemsetAsync(P.bar, 0, sizeof(unsigned) * P.nbar, st));
    ProfScope ps(st, PROF_REORTH, 0.0);   // the kernel alone (the memset of the barrier words is not its time)
    KB_CUDA(cudaLaunchKernelEx(&lc, kern, P, Gm));
    return true;
}

// Tiled kernel envelope: fp32 zero BC, n a multiple of 128 or a divisor of 128 with n^2 >= 1024.
static bool tiled_launch(PkParams& P, cudaStream_t st) {
    const int n = P.n;
    TileGeo Gm{};
    if (n >= 128 && n % 128 == 0) Gm.TW = 128;
    else if (n >= 32 && 128 % n == 0) Gm.TW = n;
    else return false;
    if (P.ld_s % 4 || P.ld_q % 4) return false;
    Gm.LR = Gm.TW / 4;
    Gm.RW = 32 / Gm.LR;
    Gm.RB = n / (8 * Gm.RW);
    Gm.T = (int)((int64_t)n * n / 1024);
    static const int cps = std::getenv("KB_PK_CTAS_PER_SM") ? std::atoi(std::getenv("KB_PK_CTAS_PER_SM")) : 2;
    const int per = cps * kSMs;
    const int need = (Gm.T + std::min(per, Gm.T) - 1) / std::min(per, Gm.T);
    // deferred normalisation (3 grid syncs per half step) is opt-in: measured slower on B200
    // (n=1024 0.90 vs 0.84 ms, n=2048 2.56 vs 2.34 ms: the saved barrier is outweighed by
    // slower z rows and basis streams right after the merged phase)
    static const int defer = std::getenv("KB_PK_DEFER") ? std::atoi(std::getenv("KB_PK_DEFER")) : 0;
    if (defer) {
        if (need <= 4) return tiled_launch_g<4, true>(P, Gm, cps, st);
        if (need <= 8) return tiled_launch_g<8, true>(P, Gm, cps, st);
        if (need <= 16) return tiled_launch_g<16, true>(P, Gm, cps, st);
        return false;
    }
    if (need <= 4) return tiled_launch_g<4, false>(P, Gm, cps, st);
    if (need <= 8) return tiled_launch_g<8, false>(P, Gm, cps, st);
    if (need <= 16) return tiled_launch_g<16, false>(P, Gm, cps, st);
    return false;
}

// Sizes of the scratch the persistent kernel needs (doubles).
// barrier words (unsigned): arrivals, generation, per-column-chunk counters
static size_t pk_bar_only_words(int lmax) { return (64 + (size_t)(lmax + 31) / 32 + 32 + 1) & ~(size_t)1; }
static size_t pk_xacc_words(int cap) { return 2 * 2 * 3 * (size_t)(cap + 4); }
static size_t pk_bar_words(int lmax, int cap) {
    return pk_bar_only_words(lmax) + 4 * (size_t)lmax + pk_xacc_words(cap);
}
static size_t pk_bar_doubles(int lmax, int cap) { return (pk_bar_words(lmax, cap) + 1) / 2; }

size_t pk_scratch_doubles(int lmax, int cap) {
    return 2 * (size_t)PK_SEGS * lmax + (size_t)(8 * kSMs) * (cap + 4) + 8 * kSMs * PK_NSTRIDE + 2 * (size_t)cap + 256 +
           (size_t)lmax + (size_t)cap + 8 + pk_bar_doubles(lmax, cap);
}

// Returns false when the configuration is outside the persistent kernel's
// envelope (the caller then uses the graph path).
bool egkb_persistent(const kb_operator* op, const kb_egkb_config* cfg, kb_egkb_state* st, const void* y0,
                     int* hdr, double* trace, double* scratch, void* raw, double tol, double** scales_out,
                     cudaStream_t s) {
    if (!ra_is_operator(op->kind)) return false;
    if (cfg->reorth_passes >= 2) return false;
    const int n = op->side;
    const int lmax = std::max(op->kh, op->kw);
    const int64_t N = (int64_t)n * n;
    const int vec = op->dtype == KB_F32 ? 4 : 2;
    if (N % vec != 0 || st->ld_s % vec != 0 || st->ld_q % vec != 0) return false;
    if (((uintptr_t)st->s_basis % 16) || ((uintptr_t)st->q_basis % 16) || ((uintptr_t)y0 % 16)) return false;
    const int cap = st->capacity;
    PkParams P{};
    P.K = op->k;
    P.Kt = op->kt;
    P.kh = op->kh;
    P.kw = op->kw;
    P.n = n;
    P.refl = op->kind == KB_OP_RA_REFLEXIVE;
    P.S = st->s_basis;
    P.Q = st->q_basis;
    P.ld_s = st->ld_s;
    P.ld_q = st->ld_q;
    P.cap = cap;
    P.y0 = y0;
    P.hdr = hdr;
    P.alphas = trace;
    P.ts = trace + cap;
    P.zetas = trace + 2 * cap;
    P.nus = trace + 3 * cap;
    P.tol = tol;
    P.tau = cfg->tau;
    P.k_max = cfg->k_max;
    P.p = cfg->p;
    P.k_min = cfg->k_min;
    P.full_reorth = cfg->full_reorth;
    P.lmax = lmax;
    P.diag_part = scratch;
    P.col_part = scratch + (size_t)PK_SEGS * lmax;
    P.blk_part = scratch + 2 * (size_t)PK_SEGS * lmax;
    P.norm_part = P.blk_part + (size_t)(8 * kSMs) * (cap + 4);
    P.zbuf = P.norm_part + 8 * kSMs * PK_NSTRIDE + 2 * (size_t)cap + 256;
    P.bres = P.zbuf + lmax;
    P.bar = reinterpret_cast<unsigned*>(P.bres + cap + 8);
    P.nbar = (int)pk_bar_words(lmax, cap);
    P.wfix = reinterpret_cast<unsigned long long*>(P.bar + pk_bar_only_words(lmax));
    P.xacc = reinterpret_cast<long long*>(P.wfix + 2 * (size_t)lmax);
    P.raw_s = raw;
    P.raw_q = static_cast<char*>(raw) + (size_t)N * (op->dtype == KB_F32 ? 4 : 8);
    *scales_out = nullptr;
    static unsigned long long* dbg = nullptr;
    static int* dbg_n = nullptr;
    static const bool want_trace = std::getenv("KB_PK_TRACE") != nullptr;
    if (want_trace) {
        if (!dbg) {
            KB_CUDA(cudaMalloc(&dbg, 4096 * sizeof(unsigned long long)));
            KB_CUDA(cudaMalloc(&dbg_n, sizeof(int)));
        }
        KB_CUDA(cudaMemsetAsync(dbg_n, 0, sizeof(int), s));
        P.dbg = dbg;
        P.dbg_n = dbg_n;
    }
    struct Dump {
        bool on; cudaStream_t s; unsigned long long* d; int* n;
        ~Dump() {
            if (!on) return;
            int k = 0;
            cudaMemcpyAsync(&k, n, sizeof(int), cudaMemcpyDeviceToHost, s);
            std::vector<unsigned long long> t(4096);
            cudaMemcpyAsync(t.data(), d, sizeof(unsigned long long) * 4096, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            k = std::min(k, 4096);
            fprintf(stderr, "[kb] pk phases (us):");
            for (int i = 1; i < k; ++i) {
                const unsigned tag = (unsigned)(t[i] & 15);
                if (tag) fprintf(stderr, " %u:%.1f", tag, ((t[i] & ~15ull) - (t[i - 1] & ~15ull)) * 1e-3);
                else fprintf(stderr, " %.1f", (t[i] - t[i - 1]) * 1e-3);
            }
            fprintf(stderr, "\n");
        }
    } dump{want_trace, s, dbg, dbg_n};
    int grid = 0;
    static const bool no_tiled = std::getenv("KB_EGKB_NO_TILED") != nullptr;
    if (!no_tiled && op->dtype == KB_F32 && !P.refl && tiled_launch(P, s)) return true;
    // smallest register footprint that covers N with 2 CTAs per SM
    const int64_t per = (int64_t)2 * kSMs * PK_THREADS * vec;
    const int64_t ng = (N + per - 1) / per;
    if (op->dtype == KB_F32) {
        if (ng <= 4) return pk_launch<float, 4, 4>(P, s, grid);
        if (ng <= 8) return pk_launch<float, 4, 8>(P, s, grid);
        return pk_launch<float, 4, PK_MAXG_F32>(P, s, grid);
    }
    if (ng <= 4) return pk_launch<double, 2, 4>(P, s, grid);
    if (ng <= 8) return pk_launch<double, 2, 8>(P, s, grid);
    return pk_launch<double, 2, PK_MAXG_F64>(P, s, grid);
}

}  // namespace kb
