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
        shard::k_bcast_dots<<<rows_grid(a0, a1, 8), 256, sizeof(long long) * 3 * (m + 2), as_stream(stream)>>>(
            z, n, c, len, beta_dev, prev, S, ld, m, a0, a1, v_out, limbs);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_update(float* v, const float* S, int64_t ld, int m, const long long* dot_limbs, int n,
                               int a0, int a1, long long* norm_limbs, double* scal, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && dot_limbs && norm_limbs && scal && (!m || S), "bad arguments");
        shard::k_update<<<rows_grid(a0, a1, 8), 256, sizeof(float) * (m + 1), as_stream(stream)>>>(
            v, S, ld, m, dot_limbs, n, a0, std::max(a0, a1), norm_limbs, scal);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_shard_normalize(const float* v, const long long* norm_limbs, float* out, int n, int c, int len,
                                  int a0, int a1, long long* diag_limbs, double* scal, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && norm_limbs && out && scal && a0 % 8 == 0, "bad arguments");
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
