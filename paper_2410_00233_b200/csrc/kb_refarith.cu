// eGKB in the reference's own fp32 arithmetic, bit for bit (KB_ARITH_OPENBLAS_*).
//
// The reference (lowrank.py:199-277) runs its fp32 recurrence through numpy:
// every norm (np.linalg.norm -> x.dot(x)) and every modified Gram-Schmidt
// coefficient (`b @ v`, lowrank.py:153-156) is one call of OpenBLAS's sdot,
// whose x86-64 kernels accumulate in fp32 FMA lanes -- 64 lanes for the
// SkylakeX/Cooperlake/SapphireRapids kernel (4 x 512-bit accumulators), 32
// for the Haswell/Zen kernel (4 x 256-bit) -- and fold the lanes in a fixed
// tree; the elementwise steps are separately rounded fp32 multiplies,
// subtractions and divisions.  Past the numerical rank the recurrence runs
// on rounding noise, so where it breaks down (k_p) depends on exactly these
// roundings: a more accurate implementation (the fused engine's fp64 sums)
// keeps the noise alive for one or two more steps.  This engine repeats the
// reference's operations in the reference's order:
//
//   * k_update: the elementwise steps, v = u - fl(beta*prev) and the MGS
//     update v = v - fl(c*b), with numpy's two roundings, over the whole grid.
//   * k_chain: one sdot.  Lane l accumulates the elements 64k+l (32k+l) in
//     order with IEEE fp32 FMAs, exactly as the SIMD accumulators do; 8 lanes
//     per CTA (one 32-byte sector per row), the rows streamed through a
//     lane-major shared-memory ring by 4-byte cp.async.  The last CTA folds
//     the lanes in the kernel's order, runs the 32-element block and the
//     scalar tail (fp32 products summed in fp64), and takes sqrtf for norms.
//     A second, independent lane set yields |u| (the breakdown threshold) in
//     the same pass.
//   * k_normalize: s = fl(v / t) (lowrank.py:247, 260).
//   * ref_product: the R(A) products in the port's fixed fp64 order
//     (oracle/structured.py: np.bincount's sequential diagonal sums, the kernel
//     rows summed in index order, one rounding to fp32).
//
// Each coefficient is a dependent chain of N/64 FMAs (4-cycle latency):
// this engine is latency-bound by construction; it exists to reproduce the
// reference's decisions and traces exactly, not to be fast.
#include <cuda_pipeline.h>

#include <algorithm>
#include <cmath>
#include <vector>

#include "kb_common.cuh"

namespace kb {
namespace refa {

constexpr int LPC = 8;      // lanes (chains) per CTA: one 32-byte sector per row
constexpr int ROWS = 128;   // rows per ring stage
constexpr int NS = 12;      // ring stages
constexpr int NARR = 3;     // streamed arrays: x, v, u

struct ChainArgs {
    const float* x;      // chain 0 = sdot(x, v); nullptr: sdot(v, v)
    const float* v;
    const float* u;      // chain 1 = sdot(u, u) when not nullptr
    float* out0;         // chain 0 result (sqrtf'ed when sqrt0)
    float* out1;         // sqrtf(chain 1)
    int sqrt0;
    int64_t n;
    int lanes;           // 64 (SkylakeX kernel) or 32 (Haswell kernel)
    float* lane_acc;     // [2][64]
    unsigned* ticket;
};

// Lane fold + 32-element block + scalar tail of OpenBLAS's x86-64 sdot
// (kernel/x86_64/sdot.c with the skylakex / haswell micro-kernels).
__device__ float sdot_fold(const float* acc, int lanes, const float* x, const float* y, int64_t n) {
    const int64_t n1 = n & ~(int64_t)31, nmain = lanes == 64 ? (n1 & ~(int64_t)63) : n1;
    float r;
    if (lanes == 64) {
        float q[4][8];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 8; ++j) q[k][j] = __fadd_rn(acc[16 * k + j], acc[16 * k + j + 8]);
        if (n1 > nmain)   // the 256-bit loop after the 512-bit one: one block of 32
#pragma unroll
            for (int k = 0; k < 4; ++k)
#pragma unroll
                for (int j = 0; j < 8; ++j) q[k][j] = fmaf(x[nmain + 8 * k + j], y[nmain + 8 * k + j], q[k][j]);
        float s8[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) s8[j] = __fadd_rn(__fadd_rn(__fadd_rn(q[0][j], q[1][j]), q[2][j]), q[3][j]);
        float h[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) h[j] = __fadd_rn(s8[j], s8[j + 4]);
        r = __fadd_rn(__fadd_rn(h[0], h[1]), __fadd_rn(h[2], h[3]));
    } else {
        float f[4][4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int j = 0; j < 4; ++j) f[k][j] = __fadd_rn(acc[8 * k + j], acc[8 * k + j + 4]);
        float t[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) t[j] = __fadd_rn(__fadd_rn(f[0][j], f[1][j]), __fadd_rn(f[2][j], f[3][j]));
        r = __fadd_rn(__fadd_rn(t[0], t[1]), __fadd_rn(t[2], t[3]));
    }
    double d = (double)r;   // the scalar tail: fp32 products summed in fp64
    for (int64_t e = n1; e < n; ++e) d += (double)__fmul_rn(x[e], y[e]);
    return (float)d;
}

// The sdot lanes: lane l = 8 * blockIdx.x + threadIdx.x (< 8) accumulates rows k of the
// element 64k + l (32k + l) with fp32 FMAs in order.  A CTA's 8 lanes are one 32-byte
// sector per row; the rows reach a row-major shared-memory ring by cp.async (VEC bytes
// per copy, one pointer increment per copy), so per row a lane issues one shared load
// per array and one FMA: the 4-cycle FMA chain is the limit.
template <bool HAS_X, bool HAS_U, int VEC>
__global__ void __launch_bounds__(32) k_chain(ChainArgs a) {
    extern __shared__ float4 smv[];
    float* sm = reinterpret_cast<float*>(smv);
    const int c = blockIdx.x, t = threadIdx.x;
    const int L = a.lanes;
    const int64_t n1 = a.n & ~(int64_t)31;
    const int64_t nmain = L == 64 ? (n1 & ~(int64_t)63) : n1;
    const int K = (int)(nmain / L);
    constexpr int SLOT = NARR * ROWS * LPC;          // floats per stage: [array][row][lane]
    constexpr int PER = LPC * 4 / VEC;               // copies per row per array
    constexpr int RSTEP = 32 / PER;                  // rows between one thread's copies
    const int nst = (K + ROWS - 1) / ROWS;
    const int part = t % PER, crow = t / PER;
    // this thread's source pointers at row crow of stage 0, and its destination offset
    const float* gv = a.v + (int64_t)crow * L + c * LPC + part * (VEC / 4);
    const float* gx = HAS_X ? a.x + (int64_t)crow * L + c * LPC + part * (VEC / 4) : nullptr;
    const float* gu = HAS_U ? a.u + (int64_t)crow * L + c * LPC + part * (VEC / 4) : nullptr;
    const int soff = crow * LPC + part * (VEC / 4);
    const int64_t gstep = (int64_t)RSTEP * L;

    auto issue = [&](int st) {
        if (st < nst) {
            float* dst = sm + (st % NS) * SLOT + soff;
            const int r0 = st * ROWS;
            const int rows = min(ROWS, K - r0);
            const int64_t g0 = (int64_t)r0 * L;
#pragma unroll
            for (int i = 0; i < ROWS / RSTEP; ++i) {
                if (crow + i * RSTEP < rows) {
                    const int64_t go = g0 + i * gstep;
                    const int so = i * RSTEP * LPC;
                    __pipeline_memcpy_async(dst + 1 * ROWS * LPC + so, gv + go, VEC);
                    if (HAS_X) __pipeline_memcpy_async(dst + 0 * ROWS * LPC + so, gx + go, VEC);
                    if (HAS_U) __pipeline_memcpy_async(dst + 2 * ROWS * LPC + so, gu + go, VEC);
                }
            }
        }
        __pipeline_commit();
    };

    for (int st = 0; st < NS - 1; ++st) issue(st);
    float acc0 = 0.f, acc1 = 0.f;
    for (int st = 0; st < nst; ++st) {
        __pipeline_wait_prior(NS - 2);
        __syncwarp();
        issue(st + NS - 1);
        if (t < LPC) {
            const float* __restrict__ base = sm + (st % NS) * SLOT + t;
            const int rows = min(ROWS, K - st * ROWS);
            if (rows == ROWS) {
                // software-pipelined: the shared loads of the next 16 rows are issued before
                // the 16 dependent FMAs of this group, so the FMA chain never waits on them
                constexpr int GR = 16;
                float cv[GR], cx[GR], cu[GR], nv[GR], nx[GR], nu[GR];
                auto ld = [&](int r0, float* a, float* b, float* c) {
#pragma unroll
                    for (int j = 0; j < GR; ++j) {
                        a[j] = base[(1 * ROWS + r0 + j) * LPC];
                        if (HAS_X) b[j] = base[(0 * ROWS + r0 + j) * LPC];
                        if (HAS_U) c[j] = base[(2 * ROWS + r0 + j) * LPC];
                    }
                };
                ld(0, cv, cx, cu);
#pragma unroll
                for (int r0 = 0; r0 < ROWS; r0 += GR) {
                    if (r0 + GR < ROWS) ld(r0 + GR, nv, nx, nu);
#pragma unroll
                    for (int j = 0; j < GR; ++j) {
                        acc0 = fmaf(HAS_X ? cx[j] : cv[j], cv[j], acc0);
                        if (HAS_U) acc1 = fmaf(cu[j], cu[j], acc1);
                    }
#pragma unroll
                    for (int j = 0; j < GR; ++j) {
                        cv[j] = nv[j];
                        if (HAS_X) cx[j] = nx[j];
                        if (HAS_U) cu[j] = nu[j];
                    }
                }
            } else {
                for (int r = 0; r < rows; ++r) {
                    const float v = base[(1 * ROWS + r) * LPC];
                    acc0 = fmaf(HAS_X ? base[(0 * ROWS + r) * LPC] : v, v, acc0);
                    if (HAS_U) {
                        const float u = base[(2 * ROWS + r) * LPC];
                        acc1 = fmaf(u, u, acc1);
                    }
                }
            }
        }
        __syncwarp();
    }
    __pipeline_wait_prior(0);
    const int lane = c * LPC + t;
    if (t < LPC) {
        a.lane_acc[lane] = acc0;
        a.lane_acc[64 + lane] = acc1;
    }
    __threadfence();
    __syncwarp();
    unsigned prev = 0;
    if (t == 0) prev = atomicAdd(a.ticket, 1u);
    prev = __shfl_sync(0xffffffffu, prev, 0);
    if (prev != gridDim.x - 1) return;
    __threadfence();
    if (t == 0) {   // last CTA: the folds, the remainder elements, the results
        float acc[64];
        for (int i = 0; i < L; ++i) acc[i] = __ldcg(a.lane_acc + i);
        const float r0 = sdot_fold(acc, L, HAS_X ? a.x : a.v, a.v, a.n);
        *a.out0 = a.sqrt0 ? sqrtf(r0) : r0;
        if (HAS_U) {
            for (int i = 0; i < L; ++i) acc[i] = __ldcg(a.lane_acc + 64 + i);
            *a.out1 = sqrtf(sdot_fold(acc, L, a.u, a.u, a.n));
        }
        *a.ticket = 0u;
    }
}

// The elementwise steps with numpy's roundings (a rounded product, then a rounded
// difference): v = vin - fl(c * b), c a device fp32 scalar -- lowrank.py:239, 252
// (u - alpha s_j, q_raw - t q_j) and the MGS update of lowrank.py:155.
__global__ void k_update(const float* __restrict__ vin, const float* __restrict__ b, const float* __restrict__ cdev,
                         float* __restrict__ vout, int64_t n) {
    const float cv = *cdev;
    const int64_t n4 = n >> 2;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const float4* v4 = reinterpret_cast<const float4*>(vin);
    const float4* b4 = reinterpret_cast<const float4*>(b);
    float4* o4 = reinterpret_cast<float4*>(vout);
    for (int64_t i = i0; i < n4; i += stride) {
        const float4 x = v4[i], y = b4[i];
        o4[i] = make_float4(__fsub_rn(x.x, __fmul_rn(cv, y.x)), __fsub_rn(x.y, __fmul_rn(cv, y.y)),
                            __fsub_rn(x.z, __fmul_rn(cv, y.z)), __fsub_rn(x.w, __fmul_rn(cv, y.w)));
    }
    for (int64_t i = 4 * n4 + i0; i < n; i += stride) vout[i] = __fsub_rn(vin[i], __fmul_rn(cv, b[i]));
}

__global__ void k_normalize(const float* __restrict__ v, const float* __restrict__ tdev, float* __restrict__ out,
                            int64_t n) {
    const float tv = *tdev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        out[i] = __fdiv_rn(v[i], tv);
}

// ---- reference-order R(A) products (oracle/structured.py ra_matvec / ra_rmatvec):
// w[u] = sequential fp64 sum over the cells hitting u in np.bincount's input order
// (Toeplitz family, then the two Hankel families of reflexive BC; cells increasing);
// z = sequential fp64 sum over the kernel rows of rounded products; y = fl32(z)
// (zero BC) or fl32 of the sequential sum of a cell's hits (reflexive).
// The sequential sums keep many loads in flight: a batch of PF loads is issued, then the
// batch is added in order (the additions are the only dependent chain).
constexpr int PF = 32;

__global__ void k_rdiag(const float* __restrict__ x, int n, int c, int len, int refl, double* __restrict__ w) {
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= len) return;
    double acc = 0.0;
    const int o = u - c;   // Toeplitz: b = a + o
    const int a_lo = max(0, -o), a_hi = min(n, n - o);
    {   // the next batch's loads are issued before this batch is added (sequential order kept)
        const int64_t st = (int64_t)n + 1;
        const float* px = x + (int64_t)a_lo * st + o;
        const int cnt = max(0, a_hi - a_lo), nb = cnt / PF;
        float cur[PF], nxt[PF];
        if (nb > 0) {
#pragma unroll
            for (int j = 0; j < PF; ++j) cur[j] = __ldg(px + j * st);
        }
        for (int b = 0; b < nb; ++b) {
            if (b + 1 < nb) {
#pragma unroll
                for (int j = 0; j < PF; ++j) nxt[j] = __ldg(px + ((int64_t)(b + 1) * PF + j) * st);
            }
#pragma unroll
            for (int j = 0; j < PF; ++j) acc = __dadd_rn(acc, (double)cur[j]);
#pragma unroll
            for (int j = 0; j < PF; ++j) cur[j] = nxt[j];
        }
        for (int j = nb * PF; j < cnt; ++j) acc = __dadd_rn(acc, (double)__ldg(px + j * st));
    }
    if (refl) {
        for (int fam = 0; fam < 2; ++fam) {   // a + b + 1 + c = u, then a + b + c + 1 - 2n = u
            const int sb = fam == 0 ? u - 1 - c : u + 2 * n - c - 1;   // b = sb - a
            const int lo = max(0, sb - (n - 1)), hi = min(n - 1, sb);   // a range with 0 <= b < n
            int a0 = lo;
            for (; a0 + PF <= hi + 1; a0 += PF) {
                float q[PF];
#pragma unroll
                for (int j = 0; j < PF; ++j) q[j] = __ldg(x + (int64_t)(a0 + j) * n + sb - (a0 + j));
#pragma unroll
                for (int j = 0; j < PF; ++j) acc = __dadd_rn(acc, (double)q[j]);
            }
            for (; a0 <= hi; ++a0) acc = __dadd_rn(acc, (double)__ldg(x + (int64_t)a0 * n + sb - a0));
        }
    }
    w[u] = acc;
}

// z[o] = sum_i M[i][o] w[i], i sequential (M row-major rows x cols: K for R q, K^T for R^T s)
__global__ void k_rz(const float* __restrict__ M, int rows, int cols, const double* __restrict__ w,
                     double* __restrict__ z) {
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= cols) return;
    double acc = 0.0;
    const int nb = rows / PF;
    float cur[PF], nxt[PF];
    if (nb > 0) {
#pragma unroll
        for (int j = 0; j < PF; ++j) cur[j] = __ldg(M + (int64_t)j * cols + o);
    }
    for (int b = 0; b < nb; ++b) {   // next batch in flight while this one is summed in order
        if (b + 1 < nb) {
#pragma unroll
            for (int j = 0; j < PF; ++j) nxt[j] = __ldg(M + ((int64_t)(b + 1) * PF + j) * cols + o);
        }
#pragma unroll
        for (int j = 0; j < PF; ++j) acc = __dadd_rn(acc, __dmul_rn((double)cur[j], __ldg(w + b * PF + j)));
#pragma unroll
        for (int j = 0; j < PF; ++j) cur[j] = nxt[j];
    }
    for (int i = nb * PF; i < rows; ++i) acc = __dadd_rn(acc, __dmul_rn((double)__ldg(M + (int64_t)i * cols + o), __ldg(w + i)));
    z[o] = acc;
}

__global__ void k_rbcast(const double* __restrict__ z, int n, int c, int len, int refl, float* __restrict__ y) {
    const int64_t N = (int64_t)n * n;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < N; e += (int64_t)gridDim.x * blockDim.x) {
        const int a = (int)(e / n), b = (int)(e - (int64_t)a * n);
        const int u1 = b - a + c;
        if (!refl) {
            y[e] = (u1 >= 0 && u1 < len) ? (float)z[u1] : 0.f;
            continue;
        }
        double acc = 0.0;
        if (u1 >= 0 && u1 < len) acc = __dadd_rn(acc, z[u1]);
        const int u2 = a + b + 1 + c;
        if (u2 >= 0 && u2 < len) acc = __dadd_rn(acc, z[u2]);
        const int u3 = a + b + c + 1 - 2 * n;
        if (u3 >= 0 && u3 < len) acc = __dadd_rn(acc, z[u3]);
        y[e] = (float)acc;
    }
}

// y = R(A) x (transpose = 0) or R(A)^T x, reference order; w, z: device scratch (>= kh + kw doubles each)
void ref_product(const kb_operator* op, const float* x, float* y, int transpose, double* w, double* z,
                 cudaStream_t s) {
    const int n = op->side, kh = op->kh, kw = op->kw, refl = op->kind == KB_OP_RA_REFLEXIVE;
    const int lin = transpose ? kw : kh, cin = lin / 2;     // diagonal sums of the input
    const int lout = transpose ? kh : kw, cout = lout / 2;  // broadcast of z
    k_rdiag<<<(int)cdiv(lin, 32), 32, 0, s>>>(x, n, cin, lin, refl, w);
    KB_LAUNCH_CHECK();
    // R q: z[v] = sum_u K[u][v] w[u] (K: kh x kw);  R^T s: z[u] = sum_v K^T[v][u] w[v] (K^T: kw x kh)
    const float* M = static_cast<const float*>(transpose ? op->kt : op->k);
    k_rz<<<(int)cdiv(lout, 32), 32, 0, s>>>(M, lin, lout, w, z);
    KB_LAUNCH_CHECK();
    const int64_t N = (int64_t)n * n;
    k_rbcast<<<(int)std::min<int64_t>(cdiv(N, 256), kSMs * 16), 256, 0, s>>>(z, n, cout, lout, refl, y);
    KB_LAUNCH_CHECK();
}

__global__ void k_update_scalar(const float* __restrict__ vin, const float* __restrict__ b,
                                const float* __restrict__ cdev, float* __restrict__ vout, int64_t n) {
    const float cv = *cdev;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        vout[i] = __fsub_rn(vin[i], __fmul_rn(cv, b[i]));
}

template <bool X, bool U, int VEC>
static void chain_launch(const ChainArgs& a, size_t smem, cudaStream_t s) {
    static bool cfg = false;
    if (!cfg) {
        KB_CUDA(cudaFuncSetAttribute(k_chain<X, U, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        cfg = true;
    }
    k_chain<X, U, VEC><<<a.lanes / LPC, 32, smem, s>>>(a);
}

void launch_chain(ChainArgs a, cudaStream_t s) {
    const size_t smem = sizeof(float) * NS * NARR * ROWS * LPC;
    const bool al = (uintptr_t)a.v % 16 == 0 && (!a.x || (uintptr_t)a.x % 16 == 0) && (!a.u || (uintptr_t)a.u % 16 == 0);
    if (al) {
        if (a.x && a.u) chain_launch<true, true, 16>(a, smem, s);
        else if (a.x) chain_launch<true, false, 16>(a, smem, s);
        else if (a.u) chain_launch<false, true, 16>(a, smem, s);
        else chain_launch<false, false, 16>(a, smem, s);
    } else {
        if (a.x && a.u) chain_launch<true, true, 4>(a, smem, s);
        else if (a.x) chain_launch<true, false, 4>(a, smem, s);
        else if (a.u) chain_launch<false, true, 4>(a, smem, s);
        else chain_launch<false, false, 4>(a, smem, s);
    }
    KB_LAUNCH_CHECK();
}

void launch_update(const float* vin, const float* b, const float* cdev, float* vout, int64_t n, cudaStream_t s) {
    const bool al = ((uintptr_t)vin % 16 == 0) && ((uintptr_t)b % 16 == 0) && ((uintptr_t)vout % 16 == 0);
    const int grid = (int)std::min<int64_t>(kSMs * 4, std::max<int64_t>(1, cdiv(n, 1024)));
    if (al) {
        k_update<<<grid, 256, 0, s>>>(vin, b, cdev, vout, n);
    } else {
        k_update_scalar<<<grid, 256, 0, s>>>(vin, b, cdev, vout, n);
    }
    KB_LAUNCH_CHECK();
}

void launch_normalize(const float* v, const float* tdev, float* out, int64_t n, cudaStream_t s) {
    const int grid = (int)std::min<int64_t>(kSMs * 8, cdiv(n, 256));
    k_normalize<<<std::max(grid, 1), 256, 0, s>>>(v, tdev, out, n);
    KB_LAUNCH_CHECK();
}

}  // namespace refa

// Scratch of the engine inside the kb_egkb_run workspace.
size_t egkb_openblas_ws_bytes(const kb_operator* op, int capacity) {
    const int64_t len = std::max(op->rows, op->cols);
    const size_t kk = (size_t)std::max(op->kh, 0) + (size_t)std::max(op->kw, 0) + 16;
    return 2 * align_up(sizeof(double) * kk) + 2 * align_up(sizeof(float) * (size_t)len) +
           align_up(sizeof(float) * (capacity + 16)) + align_up(sizeof(float) * 128) + align_up(sizeof(float) * 32) +
           align_up(sizeof(unsigned) * 8) + 2048;
}

struct RefOut {   // also declared in kb_driver.cu
    std::vector<double> alphas, ts, zetas, nus;
    int done = 1, fired = -1, reason = 0, breakdown = 0, tbreak = 0, err = 0;
};

// lowrank.py:199-277 with the reference's fp32 operations, lanes = 64 / 32.
void egkb_openblas(const kb_operator* op, const kb_egkb_config* cfg, const void* y0, kb_egkb_state* st,
                   int lanes, double tol, void* wsp, size_t ws_bytes, RefOut& o, cudaStream_t s) {
    KB_REQUIRE(op->dtype == KB_F32, "the reference-arithmetic engine reproduces the fp32 recurrence only");
    KB_REQUIRE(lanes == 64 || lanes == 32, "unknown sdot kernel");
    KB_REQUIRE(op->kind == KB_OP_RA_ZERO || op->kind == KB_OP_RA_REFLEXIVE,
               "the reference-arithmetic engine needs a matrix-free R(A) operator");
    Arena ar(wsp, ws_bytes);
    const size_t kk = (size_t)op->kh + (size_t)op->kw + 16;
    double* pw = ar.take<double>(kk);
    double* pz = ar.take<double>(kk);
    const int64_t mbar = op->rows, nbar = op->cols, len = std::max(mbar, nbar);
    float* ubuf = ar.take<float>((size_t)len);
    float* vbuf = ar.take<float>((size_t)len);
    float* coef = ar.take<float>((size_t)st->capacity + 16);
    float* sc = ar.take<float>(128);         // lane accumulators of k_chain
    float* scal = ar.take<float>(8 * 4);   // fp32 device scalars (S_*)
    unsigned* ticket = ar.take<unsigned>(8);
    enum { S_T = 0, S_UN = 1, S_A = 2, S_PRE = 3, S_ALPHA = 4 };
    float* S = static_cast<float*>(st->s_basis);
    float* Q = static_cast<float*>(st->q_basis);
    const int cap = st->capacity;
    KB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned) * 8, s));

    static thread_local float* hsc = nullptr;
    if (!hsc) KB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hsc), sizeof(float) * 8));

    // one sdot (or norm, sqrt0) of the lanes; out1 = |u| when u != nullptr
    auto chain = [&](const float* x, const float* v, const float* u, float* out0, int sqrt0, float* out1,
                     int64_t n) {
        refa::ChainArgs a{};
        a.x = x; a.v = v; a.u = u; a.out0 = out0; a.out1 = out1; a.sqrt0 = sqrt0;
        a.n = n; a.lanes = lanes; a.lane_acc = sc; a.ticket = ticket;
        refa::launch_chain(a, s);
    };
    // v = vin - fl(beta*prev) (lowrank.py:239 / 252); MGS against basis[0..m) (lowrank.py:153-156);
    // *norm_out = |v| (the t / alpha of lowrank.py:242 / 254), *pre_out = |vin| (the breakdown
    // thresholds |u| / pre_norm of lowrank.py:243 / 251); the projected vector stays in vbuf
    auto project = [&](const float* vin, const float* prev, const float* beta, const float* basis, int64_t ld,
                       int m, int64_t n, float* norm_out, float* pre_out) {
        refa::launch_update(vin, prev, beta, vbuf, n, s);
        if (m == 0) {
            chain(nullptr, vbuf, vin, norm_out, 1, pre_out, n);
            return;
        }
        chain(basis, vbuf, vin, coef, 0, pre_out, n);
        for (int i = 1; i <= m; ++i) {
            refa::launch_update(vbuf, basis + (int64_t)(i - 1) * ld, coef + i - 1, vbuf, n, s);
            if (i < m) chain(basis + (int64_t)i * ld, vbuf, nullptr, coef + i, 0, nullptr, n);
            else chain(nullptr, vbuf, nullptr, norm_out, 1, nullptr, n);
        }
    };
    auto apply = [&](const float* x, float* y, int tr) { refa::ref_product(op, x, y, tr, pw, pz, s); };
    auto fetch = [&]() {
        KB_CUDA(cudaMemcpyAsync(hsc, scal, sizeof(float) * 8, cudaMemcpyDeviceToHost, s));
        KB_CUDA(cudaStreamSynchronize(s));
    };

    // t1 = |y0|, s1 = y0 / t1 (lowrank.py:207-210)
    chain(nullptr, static_cast<const float*>(y0), nullptr, scal + S_T, 1, nullptr, mbar);
    refa::launch_normalize(static_cast<const float*>(y0), scal + S_T, S, mbar, s);
    // q = B^T s1, alpha1 = |q| (lowrank.py:211-215)
    apply(S, ubuf, 1);
    chain(nullptr, ubuf, nullptr, scal + S_ALPHA, 1, nullptr, nbar);
    refa::launch_normalize(ubuf, scal + S_ALPHA, Q, nbar, s);
    fetch();
    const double t1 = hsc[S_T], a1 = hsc[S_ALPHA];
    if (t1 == 0.0) { o.err = 1; return; }
    if (a1 == 0.0) { o.err = 2; return; }
    o.alphas.push_back(a1);
    o.ts.push_back(t1);
    o.zetas.push_back(a1 * t1);
    o.nus.push_back(1e308);
    int done = 1, fired = -1;
    for (;;) {
        const int limit = fired >= 0 ? fired + cfg->p + 1 : cfg->k_max + 1;
        if (done >= limit) break;
        KB_REQUIRE(done + 1 <= cap, "eGKB basis capacity exhausted (%d)", cap);
        // s step (lowrank.py:238-247)
        apply(Q + (int64_t)(done - 1) * st->ld_q, ubuf, 0);
        project(ubuf, S + (int64_t)(done - 1) * st->ld_s, scal + S_ALPHA, S, st->ld_s, cfg->full_reorth ? done : 0,
                mbar, scal + S_T, scal + S_UN);
        refa::launch_normalize(vbuf, scal + S_T, S + (int64_t)done * st->ld_s, mbar, s);
        // q step (lowrank.py:250-260), run before the t test is read back: harmless on a t breakdown
        apply(S + (int64_t)done * st->ld_s, ubuf, 1);
        project(ubuf, Q + (int64_t)(done - 1) * st->ld_q, scal + S_T, Q, st->ld_q, done, nbar, scal + S_A,
                scal + S_PRE);
        refa::launch_normalize(vbuf, scal + S_A, Q + (int64_t)done * st->ld_q, nbar, s);
        fetch();
        const double t_new = hsc[S_T], u_norm = hsc[S_UN], a_new = hsc[S_A], pre = hsc[S_PRE];
        if (t_new <= tol * u_norm) {
            o.breakdown = o.tbreak = 1;
            break;
        }
        if (a_new <= tol * pre) {
            o.breakdown = 1;
            o.ts.push_back(t_new);
            break;
        }
        o.ts.push_back(t_new);
        o.alphas.push_back(a_new);
        const double zeta = a_new * t_new;
        const double nu = std::sqrt(zeta * o.zetas.back());
        o.zetas.push_back(zeta);
        o.nus.push_back(nu);
        ++done;
        KB_CUDA(cudaMemcpyAsync(scal + S_ALPHA, scal + S_A, sizeof(float), cudaMemcpyDeviceToDevice, s));
        if (fired < 0) {
            const double nu_prev = o.nus[o.nus.size() - 2];
            if (nu > nu_prev) {
                fired = std::max(done - 1, cfg->k_min);
                o.reason = KB_STOP_NU_ROSE;
            } else if (nu < cfg->tau) {
                fired = std::max(done, cfg->k_min);
                o.reason = KB_STOP_NU_BELOW_TOL;
            }
        }
    }
    o.done = done;
    o.fired = fired;
}

}  // namespace kb

extern "C" int kb_sdot_openblas(int lanes, const float* x, const float* y, int64_t n, float* out_dev,
                                void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(lanes == 64 || lanes == 32, "lanes must be 64 (SkylakeX kernel) or 32 (Haswell kernel)");
        KB_REQUIRE(x && out_dev && n >= 0 && ws && ws_bytes >= 1024, "bad arguments");
        kb::Arena ar(ws, ws_bytes);
        float* acc = ar.take<float>(128);
        unsigned* ticket = ar.take<unsigned>(8);
        cudaStream_t s = kb::as_stream(stream);
        KB_CUDA(cudaMemsetAsync(ticket, 0, sizeof(unsigned) * 8, s));
        kb::refa::ChainArgs a{};
        a.x = y ? x : nullptr;
        a.v = y ? y : x;
        a.out0 = out_dev;
        a.n = n;
        a.lanes = lanes;
        a.lane_acc = acc;
        a.ticket = ticket;
        kb::refa::launch_chain(a, s);
    })
}
