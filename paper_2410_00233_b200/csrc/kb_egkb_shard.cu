// Row-sharded eGKB building blocks (north_star item 4).
//
// The Krylov vectors of R(A) (length n^2, index a*n + b: a = c_in on the s
// side, r_in on the q side) are partitioned into contiguous blocks of image
// rows a in [a0, a1), one block per GPU; K is replicated.  Every cross-shard
// sum of the recurrence (lowrank.py:211, 238-259) -- the diagonal sums of an
// R(A) product, the reorthogonalisation coefficients and the norms -- is a sum
// of per-CHUNK fp64 partials, where a chunk is fixed by the data layout alone
// (one image row for dots and norms; one 8-row block x one diagonal for the
// diagonal sums), never by the partition.  Each chunk partial is cut into three
// 40-bit integer limbs (weights 2^1, 2^-39, 2^-79) and the limbs are added as
// int64 -- exactly, in any order.  So the per-rank partial buffers combine
// with a plain int64 sum-allreduce (NCCL over NVLink; ~3 (2n+1) + 3 (m+2) + 3
// integers per half step), and the recurrence is bit-identical for every
// number of shards G (shard boundaries on 8-row blocks), which the simulated-
// shard test checks on one device against G = 1.
//
// Per half step (R q shown; R^T s swaps K / K^T and the centres):
//   kb_shard_z          z = K^T w from the all-reduced diagonal-sum limbs (every rank, redundantly)
//   kb_shard_bcast_dots y = P z on the own rows; v = y - beta prev; limbs of S^T v, |v|^2, |y|^2
//   -- allreduce --
//   kb_shard_update     v1 = v - S h (h from the limbs, fp32 FMAs in basis order); limbs of |v1|^2
//   -- allreduce --
//   kb_shard_normalize  out = fl(v1 / t), stored; limbs of its diagonal sums for the next product
//   -- allreduce --
#include <cmath>
#include <cstdint>
#include <initializer_list>

#include "kb_common.cuh"

namespace kb {
namespace shard {

constexpr double W2 = 2.0, W1 = 1.8189894035458565e-12 /* 2^-39 */, W0 = 1.6543612251060553e-24 /* 2^-79 */;

// x (|x| < 2^41) -> three truncated integer limbs (exact remainders via fma)
__device__ __forceinline__ void to_limbs(double x, long long& l2, long long& l1, long long& l0) {
    const double q2 = trunc(x * 0.5);
    const double r1 = fma(-q2, 2.0, x);
    const double q1 = trunc(r1 * 549755813888.0);           // 2^39
    const double r0 = fma(-q1, W1, r1);
    const double q0 = trunc(r0 * 604462909807314587353088.0);   // 2^79
    l2 = (long long)q2;
    l1 = (long long)q1;
    l0 = (long long)q0;
}

// limbs -> double, carries normalised first (the same operations on every rank)
__host__ __device__ inline double from_limbs(long long l2, long long l1, long long l0) {
    long long c = l0 >> 40;   // floor division by 2^40 (arithmetic shift)
    l0 -= c * (1ll << 40);
    l1 += c;
    c = l1 >> 40;
    l1 -= c * (1ll << 40);
    l2 += c;
    return ((double)l2 * W2 + (double)l1 * W1) + (double)l0 * W0;
}

__device__ __forceinline__ void limb_add(long long* dst, double x) {
    if (x == 0.0) return;
    long long a, b, c;
    to_limbs(x, a, b, c);
    atomicAdd(reinterpret_cast<unsigned long long*>(dst), (unsigned long long)a);
    atomicAdd(reinterpret_cast<unsigned long long*>(dst + 1), (unsigned long long)b);
    atomicAdd(reinterpret_cast<unsigned long long*>(dst + 2), (unsigned long long)c);
}

__device__ __forceinline__ double warp_sum_fixed(double v) {   // fixed butterfly order
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Diagonal-sum limbs of x over the rows [a0, a1) (8-row blocks): chunk (block, u) =
// sum over the block's rows a (ascending) of x[a n + a + u - c].
__global__ void k_diag(const float* __restrict__ x, int n, int c, int len, int a0, int a1,
                       long long* __restrict__ limbs) {
    const int blk0 = a0 + 8 * blockIdx.x;
    const int blk1 = min(blk0 + 8, a1);
    for (int u = threadIdx.x; u < len; u += blockDim.x) {
        const int o = u - c;   // b = a + o
        double s = 0.0;
        for (int a = blk0; a < blk1; ++a) {
            const int b = a + o;
            if (b >= 0 && b < n) s += (double)x[(int64_t)a * n + b];
        }
        limb_add(limbs + 3 * u, s);
    }
}

// w (fp64) from its limbs, once per product (every rank the same operations)
__global__ void k_wdecode(const long long* __restrict__ wl, int rows, double* __restrict__ w) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < rows) w[i] = from_limbs(wl[3 * i], wl[3 * i + 1], wl[3 * i + 2]);
}

// z[o] = sum_i Mt[o][i] w[i] (Mt: cols x rows row-major -- K^T for R q, K for R^T s):
// one warp per output row, lanes over i, a fixed butterfly at the end (every rank the same).
__global__ void k_z(const float* __restrict__ Mt, int rows, int cols, const double* __restrict__ wd,
                    double* __restrict__ z) {
    const int o = blockIdx.x * 8 + (threadIdx.x >> 5), lane = threadIdx.x & 31;
    if (o >= cols) return;
    const float* row = Mt + (int64_t)o * rows;
    double acc = 0.0;
    for (int i = lane; i < rows; i += 32) acc = fma((double)__ldg(row + i), __ldg(wd + i), acc);
    acc = warp_sum_fixed(acc);
    if (lane == 0) z[o] = acc;
}

// One warp per own row a: y = fl32(z[b - a + c]), v = fl(y - fl(beta * prev)) stored;
// per row, fixed-order fp64 partials of S_i . v (i < m), |v|^2, |y|^2 -> limbs
// (CTA-level int64 in shared memory, then global).
__global__ void k_bcast_dots(const double* __restrict__ z, int n, int c, int len, const double* __restrict__ beta_dev,
                             const float* __restrict__ prev, const float* __restrict__ S, int64_t ld, int m, int a0,
                             int a1, float* __restrict__ v_out, long long* __restrict__ limbs) {
    extern __shared__ long long lsh[];   // [(m + 2) * 3]
    for (int i = threadIdx.x; i < 3 * (m + 2); i += blockDim.x) lsh[i] = 0;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = a0 + blockIdx.x * (blockDim.x >> 5) + warp;
    const float beta = prev ? (float)*beta_dev : 0.f;
    if (a < a1) {
        const int64_t row = (int64_t)a * n;
        double ysq = 0.0, vsq = 0.0;
        for (int b = lane; b < n; b += 32) {
            const int u = b - a + c;
            const float y = (u >= 0 && u < len) ? (float)z[u] : 0.f;
            const float v = prev ? __fsub_rn(y, __fmul_rn(beta, prev[row + b])) : y;
            v_out[row + b] = v;
            ysq = fma((double)y, (double)y, ysq);
            vsq = fma((double)v, (double)v, vsq);
        }
        __syncwarp();
        ysq = warp_sum_fixed(ysq);
        vsq = warp_sum_fixed(vsq);
        for (int i = 0; i < m; ++i) {
            const float* s = S + (int64_t)i * ld + row;
            double d = 0.0;
            for (int b = lane; b < n; b += 32) d = fma((double)s[b], (double)v_out[row + b], d);
            d = warp_sum_fixed(d);
            if (lane == 0 && d != 0.0) {
                long long l2, l1, l0;
                to_limbs(d, l2, l1, l0);
                atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * i), (unsigned long long)l2);
                atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * i + 1), (unsigned long long)l1);
                atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * i + 2), (unsigned long long)l0);
            }
        }
        if (lane == 0) {
            long long l2, l1, l0;
            to_limbs(vsq, l2, l1, l0);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m), (unsigned long long)l2);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m + 1), (unsigned long long)l1);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m + 2), (unsigned long long)l0);
            to_limbs(ysq, l2, l1, l0);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m + 3), (unsigned long long)l2);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m + 4), (unsigned long long)l1);
            atomicAdd(reinterpret_cast<unsigned long long*>(lsh + 3 * m + 5), (unsigned long long)l0);
        }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 3 * (m + 2); i += blockDim.x)
        if (lsh[i]) atomicAdd(reinterpret_cast<unsigned long long*>(limbs + i), (unsigned long long)lsh[i]);
}

// v1 = v - sum_i fl32(h_i) S_i (fp32 FMAs in basis order), stored in place; row partials
// of |v1|^2 -> limbs.  CTA 0 also decodes |y| (the breakdown threshold) into scal[1].
__global__ void k_update(float* __restrict__ v, const float* __restrict__ S, int64_t ld, int m,
                         const long long* __restrict__ dl, int n, int a0, int a1, long long* __restrict__ nl,
                         double* __restrict__ scal) {
    extern __shared__ float hsh[];
    for (int i = threadIdx.x; i < m; i += blockDim.x) hsh[i] = (float)from_limbs(dl[3 * i], dl[3 * i + 1], dl[3 * i + 2]);
    if (blockIdx.x == 0 && threadIdx.x == 0)
        scal[1] = sqrt(from_limbs(dl[3 * m + 3], dl[3 * m + 4], dl[3 * m + 5]));
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = a0 + blockIdx.x * (blockDim.x >> 5) + warp;
    if (a >= a1) return;
    const int64_t row = (int64_t)a * n;
    double sq = 0.0;
    for (int b = lane; b < n; b += 32) {
        float x = v[row + b];
        for (int i = 0; i < m; ++i) x = fmaf(-hsh[i], S[(int64_t)i * ld + row + b], x);
        v[row + b] = x;
        sq = fma((double)x, (double)x, sq);
    }
    sq = warp_sum_fixed(sq);
    if (lane == 0) limb_add(nl, sq);
}

// t = sqrt(|v1|^2) (scal[0]), out = fl(v1 / fl32(t)) stored, and the diagonal-sum limbs of
// out for the next product (centre c, length len) over the same 8-row blocks as k_diag.
__global__ void k_normalize(const float* __restrict__ v, const long long* __restrict__ nl, float* __restrict__ out,
                            int n, int c, int len, int a0, int a1, long long* __restrict__ limbs,
                            double* __restrict__ scal) {
    extern __shared__ float tile[];   // [8][n]
    const double t = sqrt(from_limbs(nl[0], nl[1], nl[2]));
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[0] = t;
    const float tf = (float)t;
    const int blk0 = a0 + 8 * blockIdx.x, blk1 = min(blk0 + 8, a1);
    for (int e = threadIdx.x; e < (blk1 - blk0) * n; e += blockDim.x) {
        const int r = e / n, b = e - r * n;
        const int64_t idx = (int64_t)(blk0 + r) * n + b;
        const float o = __fdiv_rn(v[idx], tf);
        out[idx] = o;
        tile[r * n + b] = o;
    }
    __syncthreads();
    if (!limbs) return;
    for (int u = threadIdx.x; u < len; u += blockDim.x) {
        const int o = u - c;
        double s = 0.0;
        for (int a = blk0; a < blk1; ++a) {
            const int b = a + o;
            if (b >= 0 && b < n) s += (double)tile[(a - blk0) * n + b];
        }
        limb_add(limbs + 3 * u, s);
    }
}

// ---- vectorised kernels (n % 4 == 0, 16-byte aligned rows).  A persistent grid (the
// resident CTAs, one row at a time per CTA): each CTA adds its rows' limbs in shared
// memory (exact int64) before ONE set of global atomics, so the atomics per address are
// bounded by the grid, not by the row count.  Same chunks as the scalar kernels (one
// image row per dot / norm partial, 8-row blocks for the diagonal sums), so they keep
// the shard-count invariance; only the in-row summation order differs.
__device__ __forceinline__ void flush_limbs(const long long* sh, long long* dst, int count) {
    __syncthreads();
    for (int i = threadIdx.x; i < count; i += blockDim.x)
        if (sh[i]) atomicAdd(reinterpret_cast<unsigned long long*>(dst + i), (unsigned long long)sh[i]);
}

__device__ __forceinline__ double dot4(const float4& a, const float4& b, double acc) {
    acc = fma((double)a.x, (double)b.x, acc);
    acc = fma((double)a.y, (double)b.y, acc);
    acc = fma((double)a.z, (double)b.z, acc);
    return fma((double)a.w, (double)b.w, acc);
}

// Row-per-CTA kernels: the CTA (blockDim = min(256, n/4 rounded to warps)) walks the own
// rows, thread t owning the float4s t, t + blockDim, ... (NT of them) of the current row;
// the basis rows are requested four at a time (4 NT 16-byte loads in flight per thread).
// A row's partial is the warps' fixed butterflies added in warp order, so it depends on
// the row only.
template <int NT>
__global__ void __launch_bounds__(256) k_bcast_dots_r(const double* __restrict__ z, int n, int c, int len,
                                                      const double* __restrict__ beta_dev,
                                                      const float* __restrict__ prev, const float* __restrict__ S,
                                                      int64_t ld, int m, int a0, int a1, float* __restrict__ v_out,
                                                      long long* __restrict__ limbs) {
    extern __shared__ long long lsh[];   // [(m + 2) * 3] limbs, then [nwarps][m + 2] doubles
    const int W = m + 2, nw = blockDim.x >> 5;
    double* part = reinterpret_cast<double*>(lsh + 3 * W);
    for (int i = threadIdx.x; i < 3 * W; i += blockDim.x) lsh[i] = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const float beta = prev ? (float)*beta_dev : 0.f;
    const int n4 = n >> 2;
    for (int a = a0 + blockIdx.x; a < a1; a += gridDim.x) {
        const int64_t row = (int64_t)a * n;
        float4 v[NT];
        double ysq = 0.0, vsq = 0.0;
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            const int j = threadIdx.x + k * blockDim.x;
            float4 y = make_float4(0.f, 0.f, 0.f, 0.f), w = y;
            if (j < n4) {
                const float4 p = prev ? __ldg(reinterpret_cast<const float4*>(prev + row) + j) : y;
                const int u = 4 * j - a + c;
                float* yy = reinterpret_cast<float*>(&y);
#pragma unroll
                for (int q = 0; q < 4; ++q) yy[q] = (u + q >= 0 && u + q < len) ? (float)__ldg(z + u + q) : 0.f;
                w = y;
                if (prev) {
                    w.x = __fsub_rn(y.x, __fmul_rn(beta, p.x));
                    w.y = __fsub_rn(y.y, __fmul_rn(beta, p.y));
                    w.z = __fsub_rn(y.z, __fmul_rn(beta, p.z));
                    w.w = __fsub_rn(y.w, __fmul_rn(beta, p.w));
                }
                reinterpret_cast<float4*>(v_out + row)[j] = w;
            }
            v[k] = w;
            ysq = dot4(y, y, ysq);
            vsq = dot4(w, w, vsq);
        }
        for (int i0 = 0; i0 < m; i0 += 4) {
            float4 sv[4][NT];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int k = 0; k < NT; ++k) {
                    const int j = threadIdx.x + k * blockDim.x;
                    sv[r][k] = (i0 + r < m && j < n4)
                                   ? __ldg(reinterpret_cast<const float4*>(S + (int64_t)(i0 + r) * ld + row) + j)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (i0 + r >= m) break;
                float d = 0.f;   // fp32 FMAs over the thread's 4 NT cells, then fp64 across lanes
#pragma unroll
                for (int k = 0; k < NT; ++k) {
                    d = fmaf(sv[r][k].x, v[k].x, d);
                    d = fmaf(sv[r][k].y, v[k].y, d);
                    d = fmaf(sv[r][k].z, v[k].z, d);
                    d = fmaf(sv[r][k].w, v[k].w, d);
                }
                const double dw = warp_sum_fixed((double)d);
                if (lane == 0) part[warp * W + i0 + r] = dw;
            }
        }
        ysq = warp_sum_fixed(ysq);
        vsq = warp_sum_fixed(vsq);
        if (lane == 0) {
            part[warp * W + m] = vsq;
            part[warp * W + m + 1] = ysq;
        }
        __syncthreads();
        for (int i = threadIdx.x; i < W; i += blockDim.x) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += part[w * W + i];
            if (t != 0.0) {
                long long l2, l1, l0;
                to_limbs(t, l2, l1, l0);
                lsh[3 * i] += l2;   // one thread per entry: no atomics needed
                lsh[3 * i + 1] += l1;
                lsh[3 * i + 2] += l0;
            }
        }
        __syncthreads();
    }
    flush_limbs(lsh, limbs, 3 * W);
}

template <int NT>
__global__ void __launch_bounds__(256) k_update_r(float* __restrict__ v, const float* __restrict__ S, int64_t ld, int m,
                                                  const long long* __restrict__ dl, int n, int a0, int a1,
                                                  long long* __restrict__ nl, double* __restrict__ scal) {
    extern __shared__ float hsh[];   // [m] (padded to 2), 3 limbs, [nwarps] doubles
    long long* lsh = reinterpret_cast<long long*>(hsh + ((m + 1) & ~1));
    double* part = reinterpret_cast<double*>(lsh + 3);
    const int nw = blockDim.x >> 5, warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = threadIdx.x; i < m; i += blockDim.x) hsh[i] = (float)from_limbs(dl[3 * i], dl[3 * i + 1], dl[3 * i + 2]);
    if (threadIdx.x < 3) lsh[threadIdx.x] = 0;
    if (blockIdx.x == 0 && threadIdx.x == 0)
        scal[1] = sqrt(from_limbs(dl[3 * m + 3], dl[3 * m + 4], dl[3 * m + 5]));
    __syncthreads();
    const int n4 = n >> 2;
    for (int a = a0 + blockIdx.x; a < a1; a += gridDim.x) {
        const int64_t row = (int64_t)a * n;
        float4 x[NT];
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            const int j = threadIdx.x + k * blockDim.x;
            x[k] = j < n4 ? reinterpret_cast<const float4*>(v + row)[j] : make_float4(0.f, 0.f, 0.f, 0.f);
        }
        for (int i0 = 0; i0 < m; i0 += 4) {
            float4 sv[4][NT];
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int k = 0; k < NT; ++k) {
                    const int j = threadIdx.x + k * blockDim.x;
                    sv[r][k] = (i0 + r < m && j < n4)
                                   ? __ldg(reinterpret_cast<const float4*>(S + (int64_t)(i0 + r) * ld + row) + j)
                                   : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
            for (int r = 0; r < 4; ++r) {
                if (i0 + r >= m) break;
                const float h = -hsh[i0 + r];   // basis order: one fp32 FMA per cell per vector
#pragma unroll
                for (int k = 0; k < NT; ++k) {
                    x[k].x = fmaf(h, sv[r][k].x, x[k].x);
                    x[k].y = fmaf(h, sv[r][k].y, x[k].y);
                    x[k].z = fmaf(h, sv[r][k].z, x[k].z);
                    x[k].w = fmaf(h, sv[r][k].w, x[k].w);
                }
            }
        }
        double sq = 0.0;
#pragma unroll
        for (int k = 0; k < NT; ++k) {
            const int j = threadIdx.x + k * blockDim.x;
            if (j < n4) {
                reinterpret_cast<float4*>(v + row)[j] = x[k];
                sq = dot4(x[k], x[k], sq);
            }
        }
        sq = warp_sum_fixed(sq);
        if (lane == 0) part[warp] = sq;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int w = 0; w < nw; ++w) t += part[w];
            if (t != 0.0) {
                long long l2, l1, l0;
                to_limbs(t, l2, l1, l0);
                lsh[0] += l2;
                lsh[1] += l1;
                lsh[2] += l0;
            }
        }
        __syncthreads();
    }
    flush_limbs(lsh, nl, 3);
}

// out = fl(v / t) over the CTA's NB 8-row blocks (float4, grid-stride inside the CTA),
// then the (8-row block, diagonal) partials from the CTA's own stores of out, the CTA's
// blocks added as int64 limbs before the atomics.
__global__ void __launch_bounds__(512) k_normalize_v(const float* __restrict__ v, const long long* __restrict__ nl,
                                                     float* out, int n, int c, int len, int a0, int a1,
                                                     long long* __restrict__ limbs, double* __restrict__ scal, int NB) {
    const double t = sqrt(from_limbs(nl[0], nl[1], nl[2]));
    if (blockIdx.x == 0 && threadIdx.x == 0) scal[0] = t;
    const float tf = (float)t;
    const int r0 = a0 + 8 * NB * blockIdx.x, r1 = min(r0 + 8 * NB, a1);
    if (r0 >= r1) return;
    {
        const int64_t e0 = (int64_t)r0 * n / 4, e1 = (int64_t)r1 * n / 4;
        const float4* src = reinterpret_cast<const float4*>(v);
        float4* dst = reinterpret_cast<float4*>(out);
        int64_t e = e0 + threadIdx.x;
        for (; e + 3 * blockDim.x < e1; e += 4 * blockDim.x) {
            float4 q[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) q[j] = __ldg(src + e + j * blockDim.x);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                q[j].x = __fdiv_rn(q[j].x, tf);
                q[j].y = __fdiv_rn(q[j].y, tf);
                q[j].z = __fdiv_rn(q[j].z, tf);
                q[j].w = __fdiv_rn(q[j].w, tf);
                dst[e + j * blockDim.x] = q[j];
            }
        }
        for (; e < e1; e += blockDim.x) {
            float4 q = __ldg(src + e);
            q.x = __fdiv_rn(q.x, tf);
            q.y = __fdiv_rn(q.y, tf);
            q.z = __fdiv_rn(q.z, tf);
            q.w = __fdiv_rn(q.w, tf);
            dst[e] = q;
        }
    }
    if (!limbs) return;
    __syncthreads();   // the CTA's stores of out are visible to the CTA from here on
    // diagonals that meet the CTA's rows: b = a + u - c in [0, n) for some a in [r0, r1)
    const int u_lo = max(0, c - (r1 - 1)), u_hi = min(len, c - r0 + n);
    for (int u = u_lo + threadIdx.x; u < u_hi; u += blockDim.x) {
        const int o = u - c;   // b = a + o
        long long l2 = 0, l1 = 0, l0 = 0;
        for (int blk = r0; blk < r1; blk += 8) {
            const int bend = min(blk + 8, r1);
            float q[8];   // the block's 8 cells of this diagonal requested together
#pragma unroll
            for (int r = 0; r < 8; ++r) {
                const int a = blk + r, b = a + o;
                q[r] = (a < bend && b >= 0 && b < n) ? out[(int64_t)a * n + b] : 0.f;
            }
            double s = 0.0;   // rows in ascending order (absent cells add an exact 0)
#pragma unroll
            for (int r = 0; r < 8; ++r) s += (double)q[r];
            if (s != 0.0) {
                long long q2, q1, q0;
                to_limbs(s, q2, q1, q0);
                l2 += q2;
                l1 += q1;
                l0 += q0;
            }
        }
        if (l2) atomicAdd(reinterpret_cast<unsigned long long*>(limbs + 3 * u), (unsigned long long)l2);
        if (l1) atomicAdd(reinterpret_cast<unsigned long long*>(limbs + 3 * u + 1), (unsigned long long)l1);
        if (l0) atomicAdd(reinterpret_cast<unsigned long long*>(limbs + 3 * u + 2), (unsigned long long)l0);
    }
}

// |x|^2 limbs over the own rows (the start vector, lowrank.py:207)
__global__ void k_sqnorm(const float* __restrict__ x, int n, int a0, int a1, long long* __restrict__ nl) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int a = a0 + blockIdx.x * (blockDim.x >> 5) + warp;
    if (a >= a1) return;
    double sq = 0.0;
    for (int b = lane; b < n; b += 32) {
        const double xv = x[(int64_t)a * n + b];
        sq = fma(xv, xv, sq);
    }
    sq = warp_sum_fixed(sq);
    if (lane == 0) limb_add(nl, sq);
}

}  // namespace shard
}  // namespace kb

using namespace kb;

static int rows_grid(int a0, int a1, int per) { return std::max(1, (a1 - a0 + per - 1) / per); }

// float4s per thread for the row-per-CTA kernels (0: use the scalar kernels)
static int row_threads(int n) { return std::min(256, (int)cdiv(n / 4, 32) * 32); }

static bool vec_ok(int n, int64_t ld, std::initializer_list<const void*> ptrs) {
    if (n % 4 || ld % 4) return false;
    for (const void* p : ptrs)
        if (p && (reinterpret_cast<uintptr_t>(p) & 15)) return false;
    return true;
}

// resident CTAs of `kern` at `tpb` threads (the persistent grid), cached per kernel
template <typename K>
static int resident_grid(K kern, int tpb, size_t smem) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, tpb, smem) != cudaSuccess || per_sm < 1) per_sm = 1;
    return per_sm * kSMs;
}

static int vec_nt(int n, int64_t ld, std::initializer_list<const void*> ptrs) {
    if (!vec_ok(n, ld, ptrs)) return 0;
    const int nt = (int)cdiv(n / 4, row_threads(n));
    return nt <= 2 ? nt : 0;
}

extern "C" int kb_shard_diag(const float* x, int n, int c, int len, int a0, int a1, long long* limbs,
                             kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(x && limbs && n > 0 && 0 <= a0 && a0 <= a1 && a1 <= n && a0 % 8 == 0, "bad shard arguments");
        if (a1 == a0) return KB_OK;
        shard::k_diag<<<rows_grid(a0, a1, 8), 256, 0, as_stream(stream)>>>(x, n, c, len, a0, a1, limbs);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_z(const float* Mt, int rows, int cols, const long long* wl, double* z, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(Mt && wl && z && rows > 0 && cols > 0, "bad arguments");
        // the decoded w goes to z's tail: z holds cols entries, the caller's buffer >= rows + cols
        double* wd = z + cols;
        shard::k_wdecode<<<(int)cdiv(rows, 128), 128, 0, as_stream(stream)>>>(wl, rows, wd);
        KB_LAUNCH_CHECK();
        shard::k_z<<<(int)cdiv(cols, 8), 256, 0, as_stream(stream)>>>(Mt, rows, cols, wd, z);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_bcast_dots(const double* z, int n, int c, int len, const double* beta_dev, const float* prev,
                                   const float* S, int64_t ld, int m, int a0, int a1, float* v_out, long long* limbs,
                                   kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(z && v_out && limbs && m >= 0 && (!m || S) && (!prev || beta_dev), "bad arguments");
        if (a1 == a0) return KB_OK;
        const size_t smem = sizeof(long long) * 3 * (m + 2);
        const int nt = vec_nt(n, ld, {prev, S, v_out});
        if (nt) {
            const int tpb = row_threads(n);
            const size_t smem2 = smem + sizeof(double) * (tpb / 32) * (m + 2);
            const int g = std::min(a1 - a0, resident_grid(nt == 1 ? shard::k_bcast_dots_r<1> : shard::k_bcast_dots_r<2>,
                                                          tpb, smem2));
            if (nt == 1)
                shard::k_bcast_dots_r<1><<<g, tpb, smem2, as_stream(stream)>>>(z, n, c, len, beta_dev, prev, S, ld, m,
                                                                              a0, a1, v_out, limbs);
            else
                shard::k_bcast_dots_r<2><<<g, tpb, smem2, as_stream(stream)>>>(z, n, c, len, beta_dev, prev, S, ld, m,
                                                                              a0, a1, v_out, limbs);
        } else {
            shard::k_bcast_dots<<<rows_grid(a0, a1, 8), 256, smem, as_stream(stream)>>>(z, n, c, len, beta_dev, prev, S,
                                                                                       ld, m, a0, a1, v_out, limbs);
        }
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_update(float* v, const float* S, int64_t ld, int m, const long long* dot_limbs, int n,
                               int a0, int a1, long long* norm_limbs, double* scal, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && dot_limbs && norm_limbs && scal && (!m || S), "bad arguments");
        const int nt = vec_nt(n, ld, {v, S});
        if (nt) {
            const int tpb = row_threads(n);
            const size_t smem = sizeof(float) * (((m + 1) & ~1)) + sizeof(long long) * 3 + sizeof(double) * (tpb / 32);
            const int g = std::max(1, std::min(a1 - a0, resident_grid(nt == 1 ? shard::k_update_r<1> : shard::k_update_r<2>,
                                                                      tpb, smem)));
            if (nt == 1)
                shard::k_update_r<1><<<g, tpb, smem, as_stream(stream)>>>(v, S, ld, m, dot_limbs, n, a0, std::max(a0, a1),
                                                                         norm_limbs, scal);
            else
                shard::k_update_r<2><<<g, tpb, smem, as_stream(stream)>>>(v, S, ld, m, dot_limbs, n, a0, std::max(a0, a1),
                                                                         norm_limbs, scal);
        } else {
            shard::k_update<<<rows_grid(a0, a1, 8), 256, sizeof(float) * (m + 1), as_stream(stream)>>>(
                v, S, ld, m, dot_limbs, n, a0, std::max(a0, a1), norm_limbs, scal);
        }
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_normalize(const float* v, const long long* norm_limbs, float* out, int n, int c, int len,
                                  int a0, int a1, long long* diag_limbs, double* scal, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && norm_limbs && out && scal && a0 % 8 == 0, "bad arguments");
        if (vec_ok(n, n, {v, out}) && v != out) {
            const int rows = std::max(a1 - a0, 1);
            const int nb = std::max(1, (int)cdiv(rows, 16 * kSMs));   // 8-row blocks per CTA
            shard::k_normalize_v<<<(int)cdiv(rows, 8 * nb), 512, 0, as_stream(stream)>>>(
                v, norm_limbs, out, n, c, len, a0, std::max(a0, a1), diag_limbs, scal, nb);
            KB_LAUNCH_CHECK();
            return KB_OK;
        }
        const size_t smem = sizeof(float) * 8 * (size_t)n;
        KB_REQUIRE(smem <= 200 * 1024, "image side too large for the sharded normalisation");
        static bool cfg = false;
        if (!cfg) {
            KB_CUDA(cudaFuncSetAttribute(shard::k_normalize, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
            cfg = true;
        }
        shard::k_normalize<<<rows_grid(a0, a1, 8), 256, smem, as_stream(stream)>>>(v, norm_limbs, out, n, c, len, a0,
                                                                                     std::max(a0, a1), diag_limbs, scal);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_sqnorm(const float* x, int n, int a0, int a1, long long* norm_limbs, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(x && norm_limbs, "bad arguments");
        if (a1 == a0) return KB_OK;
        shard::k_sqnorm<<<rows_grid(a0, a1, 8), 256, 0, as_stream(stream)>>>(x, n, a0, a1, norm_limbs);
        KB_LAUNCH_CHECK();
    })
}

extern "C" double kb_shard_limbs_value(const long long* limbs_host) {
    return shard::from_limbs(limbs_host[0], limbs_host[1], limbs_host[2]);
}
