// Operator, reorthogonalisation and lift kernels for the eGKB / RSVD path
// (fp32 and fp64), sm_100a.
//
// R(A) for a zero-BC PSF blur is never formed:
//   R[c_in*n + c_out, r_in*n + r_out] = K[r_out - r_in + cu, c_out - c_in + cv]
// so  y = R q  is  w[u] = sum of q over the diagonal r_out - r_in = u - cu
//                  z    = K^T w                        (kw coefficients)
//                  y[c_in*n + c_out] = z[c_out - c_in + cv]   (Toeplitz)
// Reference sites replaced: lowrank.py:211,238,250 (b_mat @ q, b_mat.T @ s)
// on R from rearrange.py:67-75 o blurmodel.py:87-121.
//
// Bandwidth plan (one product): read the n x n band once (diagonal sums,
// coalesced along the diagonal index), read K once (column sums, coalesced
// along K rows), and never write y: the Toeplitz broadcast is regenerated
// inside the reorthogonalisation passes that consume it.
#include <algorithm>

#include "kb_ops.cuh"

#include <type_traits>

namespace kb {

// ------------------------------------------------------------------ diag sums
// Segmented variant used by the R(A) product: a CTA owns 32 consecutive
// diagonals (lane = diagonal, so a warp load is one 128-byte row segment)
// over one of RA_SEGS row segments (warp = row phase, 8 rows in flight per
// row step, 16+ independent loads per thread at n >= 1024).  The last CTA of
// a diagonal chunk sums the RA_SEGS partials in fixed order (deterministic).
constexpr int RA_SEGS = 8;

template <typename T>
__global__ void __launch_bounds__(256)
k_diag_seg(const VecRef xr, int n, int center, int L, int refl, double* __restrict__ part,
           double* __restrict__ w, unsigned* counters) {
    const T* __restrict__ X = resolve<const T>(xr);
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int u = blockIdx.x * 32 + lane;
    const int seg = blockIdx.y, nseg = gridDim.y;
    const int s0 = (int)((int64_t)n * seg / nseg), s1 = (int)((int64_t)n * (seg + 1) / nseg);
    double acc = 0.0;
    if (u < L) acc = ra_gather_rows<T, false>(X, n, u, center, s0, s1, warp, refl != 0);
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && u < L) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += red[q][lane];
        part[(int64_t)seg * L + u] = t;
    }
    if (last_block_ticket(&counters[blockIdx.x], nseg)) {
        if (warp == 0 && u < L) {
            double t = 0.0;
            for (int q = 0; q < nseg; ++q) t += __ldcg(&part[(int64_t)q * L + u]);
            w[u] = t;
        }
    }
}

// z[c] = sum_r M[r, c] w[r]: CTA = 32 columns x one row segment (same layout).
template <typename TM>
__global__ void __launch_bounds__(256)
k_colsum_seg(const TM* __restrict__ M, int64_t ld, int rows, int cols, const double* __restrict__ w,
             double* __restrict__ part, double* __restrict__ z, unsigned* counters) {
    __shared__ double red[8][33];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c = blockIdx.x * 32 + lane;
    const int seg = blockIdx.y, nseg = gridDim.y;
    const int r0 = (int)((int64_t)rows * seg / nseg), r1 = (int)((int64_t)rows * (seg + 1) / nseg);
    double acc = 0.0;
    if (c < cols) {
        int r = r0 + warp;
        for (; r + 56 < r1; r += 64) {                  // 8 independent loads per trip
            TM mv[8];
            double wv[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                mv[q] = __ldg(M + (int64_t)(r + 8 * q) * ld + c);
                wv[q] = __ldg(w + r + 8 * q);
            }
#pragma unroll
            for (int q = 0; q < 8; ++q) acc += (double)mv[q] * wv[q];
        }
        for (; r < r1; r += 8) acc += (double)__ldg(M + (int64_t)r * ld + c) * __ldg(w + r);
    }
    red[warp][lane] = acc;
    __syncthreads();
    if (warp == 0 && c < cols) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += red[q][lane];
        part[(int64_t)seg * cols + c] = t;
    }
    if (last_block_ticket(&counters[blockIdx.x], nseg)) {
        if (warp == 0 && c < cols) {
            double t = 0.0;
            for (int q = 0; q < nseg; ++q) t += __ldcg(&part[(int64_t)q * cols + c]);
            z[c] = t;
        }
    }
}

// ------------------------------------------------------------------ column sums
// z[c] = sum_r M[r, c] w[r]   (M row-major rows x cols, leading dim ld)
template <typename TM, typename TW>
__global__ void __launch_bounds__(256)
k_colsum(const TM* __restrict__ M, int64_t ld, int rows, int cols, const VecRef wr,
         int rb_rows, double* __restrict__ part, double* __restrict__ z, unsigned* counters) {
    const TW* __restrict__ w = resolve<const TW>(wr);
    __shared__ double red[8][128];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int c0 = blockIdx.x * 128;
    const int r0 = blockIdx.y * rb_rows, r1 = min(r0 + rb_rows, rows);
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int r = r0 + warp; r < r1; r += 8) {
        const double wr = (double)w[r];
        const TM* row = M + (int64_t)r * ld;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int c = c0 + lane + 32 * j;
            if (c < cols) acc[j] += (double)__ldg(row + c) * wr;
        }
    }
#pragma unroll
    for (int j = 0; j < 4; ++j) red[warp][lane + 32 * j] = acc[j];
    __syncthreads();
    const int c = c0 + threadIdx.x;
    if (threadIdx.x < 128 && c < cols) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) s += red[q][threadIdx.x];
        part[(int64_t)blockIdx.y * cols + c] = s;
    }
    if (last_block_ticket(&counters[blockIdx.x], gridDim.y)) {
        if (threadIdx.x < 128 && c < cols) {
            double s = 0.0;
#pragma unroll 8
            for (int r = 0; r < (int)gridDim.y; ++r) s += __ldcg(&part[(int64_t)r * cols + c]);
            z[c] = s;
        }
    }
}

// ------------------------------------------------------------------ row dots
// z[r] = sum_c A[r, c] x[c]  (one warp per row; dense b_mat @ q)
template <typename T>
__global__ void __launch_bounds__(256)
k_rowdot(const T* __restrict__ A, int64_t lda, int rows, int cols, const VecRef xr,
         double* __restrict__ z) {
    const T* __restrict__ x = resolve<const T>(xr);
    const int lane = threadIdx.x & 31;
    const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
    if (r >= rows) return;
    const T* row = A + (int64_t)r * lda;
    double acc = 0.0;
    for (int c = lane; c < cols; c += 32) acc += (double)__ldg(row + c) * (double)__ldg(x + c);
    acc = warp_sum(acc);
    if (lane == 0) z[r] = acc;
}

// z[r] = sum_j val[j] x[col[j]] over CSR row r (R(A) of a sparse A):
// one warp per row, lane-strided then a fixed shuffle tree -> deterministic.
// HBM-bound: 12 B per nonzero (value + index) + the gathered x.
template <typename T>
__global__ void __launch_bounds__(256)
k_csr_rows(const int64_t* __restrict__ rowptr, const int* __restrict__ col, const T* __restrict__ val,
           const VecRef xr, double* __restrict__ z, int64_t rows) {
    const T* __restrict__ x = resolve<const T>(xr);
    const int lane = threadIdx.x & 31;
    for (int64_t r = (int64_t)blockIdx.x * 8 + (threadIdx.x >> 5); r < rows; r += (int64_t)gridDim.x * 8) {
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        double acc = 0.0;
        for (int64_t j = b + lane; j < e; j += 32) acc += (double)__ldg(val + j) * (double)__ldg(x + __ldg(col + j));
        acc = warp_sum(acc);
        if (lane == 0) z[r] = acc;
    }
}

// ------------------------------------------------------------------ sources
template <typename T>
struct Gen {
    const double* z;   // global fp64 source (BUF64 / TOEP)
    const T* zt;       // T source (BUFT)
    const double* zs;  // toeplitz coefficients in shared memory
    const T* prev;
    T beta;
    int mode, side, center, L;
    __device__ __forceinline__ T y(int64_t e) const {
        if (mode == SRC_BUF64) return (T)z[e];
        if (mode == SRC_BUFT) return zt[e];
        return (T)ra_bcast(zs, (unsigned)e, side, center, L, mode == SRC_TOEP_REFL);   // n^2 < 2^32
    }
};

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ float div_rn(float a, float b) { return __fdiv_rn(a, b); }
__device__ __forceinline__ double div_rn(double a, double b) { return __ddiv_rn(a, b); }

template <typename T>
__global__ void k_src_write(const VecRef zr, int mode, int side, int center, int L, T* __restrict__ y,
                            int64_t len) {
    const double* z = resolve<const double>(zr);
    Gen<T> g{z, resolve<const T>(zr), z, nullptr, T(0), mode, side, center, L};
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x)
        y[e] = g.y(e);
}

// ------------------------------------------------------------------ reorth pass
template <typename T, int VEC>
struct VecIO;
template <>
struct VecIO<float, 4> {
    static __device__ __forceinline__ void load(const float* p, double* v) {
        float4 q = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = q.x; v[1] = q.y; v[2] = q.z; v[3] = q.w;
    }
};
template <>
struct VecIO<double, 2> {
    static __device__ __forceinline__ void load(const double* p, double* v) {
        double2 q = __ldg(reinterpret_cast<const double2*>(p));
        v[0] = q.x; v[1] = q.y;
    }
};
template <typename T>
struct VecIO<T, 1> {
    static __device__ __forceinline__ void load(const T* p, double* v) { v[0] = (double)__ldg(p); }
};

// One pass over the basis.  smem: [L toeplitz] [mmax coef] [8 x (mmax+2) warp acc] [mmax+4 fin]
// Each thread owns R groups of VEC consecutive elements per tile (groups
// strided by 256*VEC so every warp load is contiguous); per basis vector it
// issues R independent vector loads and does ONE warp reduction per tile.
// All vector / size arguments may be resolved on the device (VecRef/MRef),
// so the same launch serves every iteration of a captured eGKB graph.
template <typename T, int VEC, int R>
__global__ void __launch_bounds__(256)
k_reorth(const VecRef zr, int mode, int side, int center, int L, const VecRef prevr,
         const double* __restrict__ beta_p, const T* __restrict__ S, int64_t ld, const MRef mr,
         const double* __restrict__ coefA, const double* __restrict__ coefB, int dots, const VecRef outr,
         const double* __restrict__ div_p, int64_t len, double* __restrict__ part,
         double* __restrict__ red, double* __restrict__ fix, unsigned* counter) {
    extern __shared__ double sm[];
    const int m = mr.idx ? (*mr.idx) * mr.mul + mr.add : mr.add;
    const int mmax = mr.max;
    const int Ls = (mode >= SRC_TOEP) ? L : 0;
    double* zs = sm;
    double* coef = zs + Ls;
    double* accw = coef + mmax;            // [8][m+2]
    double* fin = accw + 8 * (mmax + 2);   // [m+4]
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int W = m + 2;
    const double* zsrc = resolve<const double>(zr);
    for (int i = threadIdx.x; i < Ls; i += blockDim.x) zs[i] = zsrc[i];
    const bool proj = (coefA != nullptr) || (coefB != nullptr);
    for (int i = threadIdx.x; i < m; i += blockDim.x)
        coef[i] = (coefA ? coefA[i] : 0.0) + (coefB ? coefB[i] : 0.0);
    for (int i = threadIdx.x; i < 8 * W; i += blockDim.x) accw[i] = 0.0;
    __syncthreads();
    const T* prev = prevr.base ? resolve<const T>(prevr) : nullptr;
    T* out = outr.base ? resolve<T>(outr) : nullptr;
    Gen<T> g{zsrc, resolve<const T>(zr), zs, prev, beta_p ? (T)(*beta_p) : T(0), mode, side, center, L};
    const T tdiv = div_p ? (T)(*div_p) : T(1);

    constexpr int64_t GROUP = 256 * VEC;
    constexpr int64_t TILE = GROUP * R;
    const int64_t ntiles = (len + TILE - 1) / TILE;
    double ysq = 0.0, vsq = 0.0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const int64_t base = tile * TILE + (int64_t)threadIdx.x * VEC;
        double v[R][VEC];
#pragma unroll
        for (int r = 0; r < R; ++r) {
#pragma unroll
            for (int q = 0; q < VEC; ++q) {
                const int64_t e = base + r * GROUP + q;
                if (e < len) {
                    const T yv = g.y(e);
                    const T vv = prev ? sub_rn(yv, mul_rn(g.beta, prev[e])) : yv;
                    v[r][q] = (double)vv;
                    ysq += (double)yv * (double)yv;
                } else {
                    v[r][q] = 0.0;
                }
            }
        }
        if (proj) {
#pragma unroll 2
            for (int i = 0; i < m; ++i) {
                const T* Si = S + (int64_t)i * ld + base;
                double sv[R][VEC];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t e0 = base + r * GROUP;
                    if (e0 + VEC <= len) {
                        VecIO<T, VEC>::load(Si + r * GROUP, sv[r]);
                    } else {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) sv[r][q] = (e0 + q < len) ? (double)Si[r * GROUP + q] : 0.0;
                    }
                }
                const double c = coef[i];
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int q = 0; q < VEC; ++q) v[r][q] -= c * sv[r][q];
            }
        }
        if (dots) {
#pragma unroll 2
            for (int i = 0; i < m; ++i) {
                const T* Si = S + (int64_t)i * ld + base;
                double sv[R][VEC];
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const int64_t e0 = base + r * GROUP;
                    if (e0 + VEC <= len) {
                        VecIO<T, VEC>::load(Si + r * GROUP, sv[r]);
                    } else {
#pragma unroll
                        for (int q = 0; q < VEC; ++q) sv[r][q] = (e0 + q < len) ? (double)Si[r * GROUP + q] : 0.0;
                    }
                }
                double d = 0.0;
#pragma unroll
                for (int r = 0; r < R; ++r)
#pragma unroll
                    for (int q = 0; q < VEC; ++q) d += sv[r][q] * v[r][q];
                d = warp_sum(d);
                if (lane == 0) accw[warp * W + i] += d;
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
            for (int q = 0; q < VEC; ++q) vsq += v[r][q] * v[r][q];
        if (out) {
#pragma unroll
            for (int r = 0; r < R; ++r)
#pragma unroll
                for (int q = 0; q < VEC; ++q) {
                    const int64_t e = base + r * GROUP + q;
                    if (e < len) out[e] = div_rn((T)v[r][q], tdiv);
                }
        }
    }
    vsq = warp_sum(vsq);
    ysq = warp_sum(ysq);
    if (lane == 0) {
        accw[warp * W + m] += vsq;
        accw[warp * W + m + 1] += ysq;
    }
    __syncthreads();
    for (int j = threadIdx.x; j < W; j += blockDim.x) {
        double t = 0.0;
#pragma unroll
        for (int q = 0; q < 8; ++q) t += accw[q * W + j];
        part[(int64_t)blockIdx.x * W + j] = t;
    }
    if (last_block_ticket(counter, gridDim.x)) {
        for (int j = warp; j < W; j += 8) {
            double t = 0.0;
            for (int b = lane; b < (int)gridDim.x; b += 32) t += __ldcg(&part[(int64_t)b * W + j]);
            t = warp_sum(t);
            if (lane == 0) fin[j] = t;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double h2 = 0.0;
            if (dots)
                for (int i = 0; i < m; ++i) h2 += fin[i] * fin[i];
            fix[0] = fin[m];
            fix[1] = fin[m + 1];
            fix[2] = sqrt(fmax(fin[m] - h2, 0.0));
            fix[3] = sqrt(fin[m]);
        }
        if (red)
            for (int j = threadIdx.x; j < m; j += blockDim.x) red[j] = fin[j];
    }
}

// ------------------------------------------------------------------ lift
// out_c = sum_i W[i, c] S_i for CB output columns per pass, accumulated in T
// (fp32 like the reference's sgemm for the fp32 path).  One element per
// thread, W broadcast from shared memory.
// TO = T: out_c = sum_i W[i,c] S_i in T (fp32 FMA chain, as the reference's
// working-precision GEMM).  TO = double: the same T value, then scaled in fp64:
// out_c = scale[c] * (double)lift_c -- kron_assemble fused into the lift
// (kronop.py:117-119: ax_i = sigma_i * u_i promoted to fp64), bit-identical to
// lift-then-assemble without writing or re-reading the working-precision u.
// Two adjacent elements per thread (float2 loads, double2 stores) for the
// fp32 -> fp64 assemble when the layout allows; each element keeps exactly
// the FMA order of the one-element path (bit-identical results).
template <int CB>
__global__ void __launch_bounds__(256)
k_lift2_asm(const float* __restrict__ S, int64_t ld, int rows, const float* __restrict__ W, int cols, int c0,
            double* __restrict__ out, int64_t ld_out, int64_t len, const double* __restrict__ scale) {
    extern __shared__ double wraw[];
    float* wsm = reinterpret_cast<float*>(wraw);  // [rows][CB]
    const int nc = min(CB, cols - c0);
    for (int i = threadIdx.x; i < rows * CB; i += blockDim.x) {
        const int r = i / CB, c = i % CB;
        wsm[i] = (c < nc) ? W[(int64_t)r * cols + c0 + c] : 0.f;
    }
    __syncthreads();
    const int64_t len2 = len / 2;
    for (int64_t e2 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e2 < len2;
         e2 += (int64_t)gridDim.x * blockDim.x) {
        float a0[CB], a1[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) a0[c] = a1[c] = 0.f;
        int i = 0;
        for (; i + 8 <= rows; i += 8) {   // 8 rows of loads in flight per thread
            float2 s8[8];
#pragma unroll
            for (int j = 0; j < 8; ++j) s8[j] = __ldg(reinterpret_cast<const float2*>(S + (int64_t)(i + j) * ld) + e2);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const float* wr = wsm + (i + j) * CB;
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    a0[c] = fmaf(s8[j].x, wr[c], a0[c]);
                    a1[c] = fmaf(s8[j].y, wr[c], a1[c]);
                }
            }
        }
        for (; i + 4 <= rows; i += 4) {
            float2 s4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) s4[j] = __ldg(reinterpret_cast<const float2*>(S + (int64_t)(i + j) * ld) + e2);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float* wr = wsm + (i + j) * CB;
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    a0[c] = fmaf(s4[j].x, wr[c], a0[c]);
                    a1[c] = fmaf(s4[j].y, wr[c], a1[c]);
                }
            }
        }
        for (; i < rows; ++i) {
            const float2 sv = __ldg(reinterpret_cast<const float2*>(S + (int64_t)i * ld) + e2);
            const float* wr = wsm + i * CB;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                a0[c] = fmaf(sv.x, wr[c], a0[c]);
                a1[c] = fmaf(sv.y, wr[c], a1[c]);
            }
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            if (c < nc) {
                const double u0 = (double)a0[c], u1 = (double)a1[c];
                const double sc = scale ? scale[c0 + c] : 1.0;
                const double2 o = scale ? make_double2(__dmul_rn(sc, u0), __dmul_rn(sc, u1)) : make_double2(u0, u1);
                __stcs(reinterpret_cast<double2*>(out + (int64_t)(c0 + c) * ld_out) + e2, o);
            }
        }
    }
}

// fp32 -> fp32 lift with four adjacent elements per thread (float4 loads and stores);
// every element keeps the FMA order of k_lift (bit-identical results).
template <int CB>
__global__ void __launch_bounds__(256)
k_lift4(const float* __restrict__ S, int64_t ld, int rows, const float* __restrict__ W, int cols, int c0,
        float* __restrict__ out, int64_t ld_out, int64_t len) {
    extern __shared__ double wraw[];
    float* wsm = reinterpret_cast<float*>(wraw);  // [rows][CB]
    const int nc = min(CB, cols - c0);
    for (int i = threadIdx.x; i < rows * CB; i += blockDim.x) {
        const int r = i / CB, c = i % CB;
        wsm[i] = (c < nc) ? W[(int64_t)r * cols + c0 + c] : 0.f;
    }
    __syncthreads();
    const int64_t len4 = len / 4;
    for (int64_t e4 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e4 < len4;
         e4 += (int64_t)gridDim.x * blockDim.x) {
        float4 acc[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) acc[c] = make_float4(0.f, 0.f, 0.f, 0.f);
        int i = 0;
        for (; i + 4 <= rows; i += 4) {   // 4 basis rows of loads in flight per thread
            float4 s4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) s4[j] = __ldg(reinterpret_cast<const float4*>(S + (int64_t)(i + j) * ld) + e4);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const float* wr = wsm + (i + j) * CB;
#pragma unroll
                for (int c = 0; c < CB; ++c) {
                    acc[c].x = fmaf(s4[j].x, wr[c], acc[c].x);
                    acc[c].y = fmaf(s4[j].y, wr[c], acc[c].y);
                    acc[c].z = fmaf(s4[j].z, wr[c], acc[c].z);
                    acc[c].w = fmaf(s4[j].w, wr[c], acc[c].w);
                }
            }
        }
        for (; i < rows; ++i) {
            const float4 sv = __ldg(reinterpret_cast<const float4*>(S + (int64_t)i * ld) + e4);
            const float* wr = wsm + i * CB;
#pragma unroll
            for (int c = 0; c < CB; ++c) {
                acc[c].x = fmaf(sv.x, wr[c], acc[c].x);
                acc[c].y = fmaf(sv.y, wr[c], acc[c].y);
                acc[c].z = fmaf(sv.z, wr[c], acc[c].z);
                acc[c].w = fmaf(sv.w, wr[c], acc[c].w);
            }
        }
#pragma unroll
        for (int c = 0; c < CB; ++c)
            if (c < nc) __stcs(reinterpret_cast<float4*>(out + (int64_t)(c0 + c) * ld_out) + e4, acc[c]);
    }
}

template <typename T, int CB, typename TO = T, bool ASM = false>
__global__ void __launch_bounds__(256)
k_lift(const T* __restrict__ S, int64_t ld, int rows, const T* __restrict__ W, int cols, int c0,
       TO* __restrict__ out, int64_t ld_out, int64_t len, const double* __restrict__ scale = nullptr) {
    extern __shared__ double wraw[];
    T* wsm = reinterpret_cast<T*>(wraw);  // [rows][CB]
    const int nc = min(CB, cols - c0);
    for (int i = threadIdx.x; i < rows * CB; i += blockDim.x) {
        const int r = i / CB, c = i % CB;
        wsm[i] = (c < nc) ? W[(int64_t)r * cols + c0 + c] : T(0);
    }
    __syncthreads();
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x) {
        T acc[CB];
#pragma unroll
        for (int c = 0; c < CB; ++c) acc[c] = T(0);
        int i = 0;
        for (; i + 4 <= rows; i += 4) {        // 4 basis loads in flight, then the same FMA order
            T s4[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) s4[j] = __ldg(S + (int64_t)(i + j) * ld + e);
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const T* wr = wsm + (i + j) * CB;
#pragma unroll
                for (int c = 0; c < CB; ++c) acc[c] = fma(s4[j], wr[c], acc[c]);
            }
        }
        for (; i < rows; ++i) {
            const T s = __ldg(S + (int64_t)i * ld + e);
            const T* wr = wsm + i * CB;
#pragma unroll
            for (int c = 0; c < CB; ++c) acc[c] = fma(s, wr[c], acc[c]);
        }
#pragma unroll
        for (int c = 0; c < CB; ++c) {
            if (c < nc) {
                if constexpr (!ASM) {
                    out[(int64_t)(c0 + c) * ld_out + e] = acc[c];
                } else {
                    const double u = (double)acc[c];
                    out[(int64_t)(c0 + c) * ld_out + e] = scale ? __dmul_rn(scale[c0 + c], u) : u;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ host side
static void ra_geom(const kb_operator* op, int transpose, int& center_in, int& L_in,
                    int& center_out, int& L_out, const void*& M) {
    // forward: diag sums over r_out - r_in (centre cu, kh bins) -> z = K^T w (kw)
    // transpose: diag sums over c_out - c_in (centre cv, kw bins) -> z = K w (kh)
    const int cu = op->kh / 2, cv = op->kw / 2;
    if (!transpose) {
        center_in = cu; L_in = op->kh; center_out = cv; L_out = op->kw; M = op->k;
    } else {
        center_in = cv; L_in = op->kw; center_out = cu; L_out = op->kh; M = op->kt;
    }
}

static int rb_for(int rows, int chunks, int target_blocks = 4 * kSMs) {
    int nrb = target_blocks / (chunks > 0 ? chunks : 1);
    if (nrb < 1) nrb = 1;
    if (nrb > rows) nrb = rows > 0 ? rows : 1;
    int rb = (int)cdiv(rows, nrb);
    return rb < 1 ? 1 : rb;
}

void op_plan_size(const kb_operator* op, Sizer& s) {
    if (ra_is_operator(op->kind)) {
        const int L = op->kh > op->kw ? op->kh : op->kw;
        const int n = op->side;
        const int nrb_max = 4 * kSMs;
        s.take<double>((size_t)nrb_max * L + 2 * L);   // diag partials (upper bound)
        s.take<double>(L);                              // w
        s.take<double>((size_t)nrb_max * L + 2 * L);   // colsum partials
        s.take<double>(L);                              // z
        s.take<unsigned>(2 * 64 + 64);
        (void)n;
    } else if (op->kind == KB_OP_SPARSE) {
        const int64_t big = op->rows > op->cols ? op->rows : op->cols;
        s.take<double>(64);
        s.take<double>(big);                            // z
        s.take<unsigned>(64);
    } else {
        const int64_t big = op->rows > op->cols ? op->rows : op->cols;
        s.take<double>((size_t)(4 * kSMs) * big);       // colsum partials (upper bound)
        s.take<double>(big);                            // z
        s.take<unsigned>((size_t)cdiv(big, 128) + 64);
    }
}

OpPlan op_plan_make(const kb_operator* op, Arena& a) {
    OpPlan p;
    p.op = op;
    if (ra_is_operator(op->kind)) {
        const int L = op->kh > op->kw ? op->kh : op->kw;
        const int nrb_max = 4 * kSMs;
        p.part = a.take<double>((size_t)nrb_max * L + 2 * L);
        p.w = a.take<double>(L);
        (void)a.take<double>((size_t)nrb_max * L + 2 * L);
        p.z = a.take<double>(L);
        p.counters = a.take<unsigned>(2 * 64 + 64);
        p.n_counters = 2 * 64 + 64;
        p.z_len = L;
    } else if (op->kind == KB_OP_SPARSE) {
        const int64_t big = op->rows > op->cols ? op->rows : op->cols;
        p.part = a.take<double>(64);
        p.z = a.take<double>(big);
        p.counters = a.take<unsigned>(64);
        p.n_counters = 64;
        p.z_len = big;
    } else {
        const int64_t big = op->rows > op->cols ? op->rows : op->cols;
        p.part = a.take<double>((size_t)(4 * kSMs) * big);
        p.z = a.take<double>(big);
        p.counters = a.take<unsigned>((size_t)cdiv(big, 128) + 64);
        p.n_counters = cdiv(big, 128) + 64;
        p.z_len = big;
    }
    return p;
}

template <typename T>
static Src op_source_t(const OpPlan& p, const VecRef& x, int transpose, cudaStream_t st) {
    const kb_operator* op = p.op;
    Src s;
    if (ra_is_operator(op->kind)) {
        int ci, Li, co, Lo;
        const void* Mv;
        ra_geom(op, transpose, ci, Li, co, Lo, Mv);
        const int n = op->side;
        const int segs = std::max(1, std::min(RA_SEGS, n / 64));
        KB_REQUIRE(cdiv(Li, 32) <= 64 && cdiv(Lo, 32) <= 64, "R(A): PSF support too large (%d x %d)",
                   op->kh, op->kw);
        // diagonal sums: 32 diagonals x 1 row segment per CTA
        {
            double band = 0;
            for (int u = 0; u < Li; ++u) {
                band += std::max(n - std::abs(u - ci), 0);
                if (op->kind == KB_OP_RA_REFLEXIVE && u != ci) {   // anti-diagonal a + b = s
                    const int sa = u > ci ? u - ci - 1 : u - ci - 1 + 2 * n;
                    band += std::max(std::min(sa + 1, 2 * n - 1 - sa), 0);
                }
            }
            ProfScope ps(st, PROF_RA_DIAG, band * sizeof(T));
            k_diag_seg<T><<<dim3((unsigned)cdiv(Li, 32), segs), 256, 0, st>>>(
                x, n, ci, Li, op->kind == KB_OP_RA_REFLEXIVE, p.part, p.w, p.counters);
            KB_LAUNCH_CHECK();
        }
        // z = M^T w with M = K (forward) or K^T (transpose): rows Li, cols Lo
        {
            const int segs2 = std::max(1, std::min(RA_SEGS, Li / 64));
            ProfScope ps(st, PROF_RA_COLSUM, (double)Li * Lo * sizeof(T));
            k_colsum_seg<T><<<dim3((unsigned)cdiv(Lo, 32), segs2), 256, 0, st>>>(
                static_cast<const T*>(Mv), Lo, Li, Lo, p.w, p.part, p.z, p.counters + 64);
            KB_LAUNCH_CHECK();
        }
        s.z = VecRef::at(p.z);
        s.mode = op->kind == KB_OP_RA_REFLEXIVE ? SRC_TOEP_REFL : SRC_TOEP;
        s.side = n;
        s.center = co;
        s.L = Lo;
    } else if (op->kind == KB_OP_SPARSE) {
        const int64_t rows = transpose ? op->cols : op->rows;
        const int64_t* rp = transpose ? op->spt_rowptr : op->sp_rowptr;
        const int* ci = transpose ? op->spt_col : op->sp_col;
        const T* va = static_cast<const T*>(transpose ? op->spt_val : op->sp_val);
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(rows, 8), 16 * kSMs);
        ProfScope ps(st, PROF_RA_COLSUM, (double)op->nnz * (sizeof(T) + 4) + 8.0 * (rows + 1) + 8.0 * rows);
        k_csr_rows<T><<<blocks, 256, 0, st>>>(rp, ci, va, x, p.z, rows);
        KB_LAUNCH_CHECK();
        s.z = VecRef::at(p.z);
        s.mode = SRC_BUF64;
    } else {
        const T* A = static_cast<const T*>(op->a);
        if (!transpose) {
            const int rows = (int)op->rows, cols = (int)op->cols;
            ProfScope ps(st, PROF_RA_COLSUM, (double)rows * cols * sizeof(T));
            k_rowdot<T><<<(unsigned)cdiv(rows, 8), 256, 0, st>>>(A, op->lda, rows, cols, x, p.z);
            KB_LAUNCH_CHECK();
        } else {
            const int rows = (int)op->rows, cols = (int)op->cols;
            const int cchunks = (int)cdiv(cols, 128);
            const int rb = rb_for(rows, cchunks);
            const int nrb = (int)cdiv(rows, rb);
            dim3 g(cchunks, nrb);
            ProfScope ps(st, PROF_RA_COLSUM, (double)rows * cols * sizeof(T));
            k_colsum<T, T><<<g, 256, 0, st>>>(A, op->lda, rows, cols, x, rb, p.part, p.z,
                                              p.counters);
            KB_LAUNCH_CHECK();
        }
        s.z = VecRef::at(p.z);
        s.mode = SRC_BUF64;
    }
    return s;
}

Src op_source(const OpPlan& p, const VecRef& x, int transpose, cudaStream_t st) {
    return p.op->dtype == KB_F32 ? op_source_t<float>(p, x, transpose, st)
                                 : op_source_t<double>(p, x, transpose, st);
}

void src_write(int dtype, const Src& s, void* y, int64_t len, cudaStream_t st) {
    const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(len, 256), 8 * kSMs);
    if (dtype == KB_F32)
        k_src_write<float><<<blocks, 256, 0, st>>>(s.z, s.mode, s.side, s.center, s.L,
                                                   static_cast<float*>(y), len);
    else
        k_src_write<double><<<blocks, 256, 0, st>>>(s.z, s.mode, s.side, s.center, s.L,
                                                    static_cast<double*>(y), len);
    KB_LAUNCH_CHECK();
}

constexpr int REORTH_R = 2;
static int reorth_blocks(int64_t len) {
    const int64_t tiles = cdiv(len, 256 * REORTH_R);   // VEC >= 1
    return (int)std::max<int64_t>(1, std::min<int64_t>(tiles, 4 * kSMs));
}

void reorth_ws_size(int64_t len, int max_m, Sizer& s) {
    s.take<double>((size_t)reorth_blocks(len) * (max_m + 2) + 64);
    s.take<unsigned>(64);
}

ReorthWs reorth_ws_make(int64_t len, int max_m, Arena& a) {
    ReorthWs w;
    w.max_blocks = reorth_blocks(len);
    w.max_m = max_m;
    w.part = a.take<double>((size_t)w.max_blocks * (max_m + 2) + 64);
    w.counter = a.take<unsigned>(64);
    return w;
}

template <typename T, int VEC>
static void launch_reorth(const Src& src, const void* S, int64_t ld, const MRef& m, const double* cA,
                          const double* cB, bool dots, const VecRef& out, const double* div, int64_t len,
                          double* red, double* fix, const ReorthWs& ws, cudaStream_t st) {
    const int Ls = (src.mode >= SRC_TOEP) ? src.L : 0;
    const int mm = m.max;
    const size_t smem = sizeof(double) * ((size_t)Ls + mm + 8 * (mm + 2) + (mm + 4));
    auto kern = k_reorth<T, VEC, REORTH_R>;
    static bool configured = false;
    if (!configured) {
        KB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        configured = true;
    }
    const int blocks = std::max(1, std::min<int>(ws.max_blocks, (int)cdiv(len, 256 * VEC * REORTH_R)));
    // algorithmic bytes (with m at its upper bound when resolved on the device)
    double vecs = (double)(m.acct >= 0 ? m.acct : mm) + (src.prev.null() ? 0 : 1) + (out.null() ? 0 : 1) + (src.mode == SRC_BUFT ? 1 : 0);
    double bytes = vecs * len * sizeof(T) + (src.mode == SRC_BUF64 ? 8.0 * len : 0.0);
    ProfScope ps(st, PROF_REORTH, bytes);
    kern<<<blocks, 256, smem, st>>>(src.z, src.mode, src.side, src.center, src.L, src.prev, src.beta,
                                    static_cast<const T*>(S), ld, m, cA, cB, dots ? 1 : 0, out, div, len,
                                    ws.part, red, fix, ws.counter);
    KB_LAUNCH_CHECK();
}

void reorth_pass(int dtype, const Src& src, const void* S, int64_t ld, const MRef& m,
                 const double* coefA, const double* coefB, bool dots, const VecRef& out,
                 const double* div, int64_t len, double* red, double* fix, const ReorthWs& ws,
                 cudaStream_t st) {
    KB_REQUIRE(m.max <= ws.max_m, "reorth: basis size %d exceeds workspace capacity %d", m.max, ws.max_m);
    auto aligned = [](const void* p, size_t a) { return p == nullptr || ((uintptr_t)p % a) == 0; };
    if (dtype == KB_F32) {
        const bool v4 = (ld % 4 == 0) && (len % 4 == 0) && aligned(S, 16);
        if (v4)
            launch_reorth<float, 4>(src, S, ld, m, coefA, coefB, dots, out, div, len, red, fix, ws, st);
        else
            launch_reorth<float, 1>(src, S, ld, m, coefA, coefB, dots, out, div, len, red, fix, ws, st);
    } else {
        const bool v2 = (ld % 2 == 0) && (len % 2 == 0) && aligned(S, 16);
        if (v2)
            launch_reorth<double, 2>(src, S, ld, m, coefA, coefB, dots, out, div, len, red, fix, ws, st);
        else
            launch_reorth<double, 1>(src, S, ld, m, coefA, coefB, dots, out, div, len, red, fix, ws, st);
    }
}

void dense_gemv64(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* x,
                  double* y, int transpose, double* part, unsigned* counters, cudaStream_t st) {
    ProfScope ps(st, PROF_RA_COLSUM, 8.0 * rows * cols);
    if (!transpose) {
        k_rowdot<double><<<(unsigned)cdiv(rows, 8), 256, 0, st>>>(A, lda, (int)rows, (int)cols, VecRef::at(x), y);
    } else {
        const int cchunks = (int)cdiv(cols, 128);
        const int rb = rb_for((int)rows, cchunks);
        dim3 g(cchunks, (unsigned)cdiv(rows, rb));
        k_colsum<double, double><<<g, 256, 0, st>>>(A, lda, (int)rows, (int)cols, VecRef::at(x), rb, part, y, counters);
    }
    KB_LAUNCH_CHECK();
}

template <typename T, int CB, typename TO, bool ASM>
static void launch_lift(const void* S, int64_t ld, int rows, const void* W, int cols, int c0, void* out,
                        int64_t ld_out, int64_t len, const double* scale, cudaStream_t st) {
    static bool configured = false;
    if (!configured) {
        KB_CUDA(cudaFuncSetAttribute(k_lift<T, CB, TO, ASM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
        configured = true;
    }
    const size_t smem = sizeof(T) * (size_t)rows * CB;
    const unsigned blocks = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(len, 256), 8 * kSMs));
    ProfScope ps(st, PROF_LIFT, (double)len * (sizeof(T) * rows + sizeof(TO) * std::min(CB, cols - c0)));
    if constexpr (ASM && sizeof(T) == 4) {
        if (len % 2 == 0 && ld % 2 == 0 && ld_out % 2 == 0 && ((uintptr_t)S % 8) == 0 && ((uintptr_t)out % 16) == 0) {
            static bool cfg2 = false;
            if (!cfg2) {
                KB_CUDA(cudaFuncSetAttribute(k_lift2_asm<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
                cfg2 = true;
            }
            const unsigned b2 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(len / 2, 256), 4 * kSMs));
            k_lift2_asm<CB><<<b2, 256, smem, st>>>(static_cast<const float*>(S), ld, rows, static_cast<const float*>(W),
                                                   cols, c0, static_cast<double*>(out), ld_out, len, scale);
            KB_LAUNCH_CHECK();
            return;
        }
    }
    if constexpr (!ASM && sizeof(T) == 4 && sizeof(TO) == 4 && CB <= 16) {   // (CB = 32: 128 accumulators)
        if (len % 4 == 0 && ld % 4 == 0 && ld_out % 4 == 0 && ((uintptr_t)S % 16) == 0 && ((uintptr_t)out % 16) == 0) {
            static bool cfg4 = false;
            if (!cfg4) {
                KB_CUDA(cudaFuncSetAttribute(k_lift4<CB>, cudaFuncAttributeMaxDynamicSharedMemorySize, 160 * 1024));
                cfg4 = true;
            }
            const unsigned b4 = (unsigned)std::max<int64_t>(1, std::min<int64_t>(cdiv(len / 4, 256), 4 * kSMs));
            k_lift4<CB><<<b4, 256, smem, st>>>(static_cast<const float*>(S), ld, rows, static_cast<const float*>(W), cols,
                                               c0, static_cast<float*>(out), ld_out, len);
            KB_LAUNCH_CHECK();
            return;
        }
    }
    k_lift<T, CB, TO, ASM><<<blocks, 256, smem, st>>>(static_cast<const T*>(S), ld, rows, static_cast<const T*>(W),
                                                 cols, c0, static_cast<TO*>(out), ld_out, len, scale);
    KB_LAUNCH_CHECK();
}

template <typename T, typename TO, bool ASM>
static void lift_cols(const void* S, int64_t ld, int rows, const void* W, int cols, void* out, int64_t ld_out,
                      int64_t len, const double* scale, cudaStream_t st) {
    for (int c0 = 0; c0 < cols; c0 += 32) {
        const int nc = std::min(32, cols - c0);
        if (nc <= 8) launch_lift<T, 8, TO, ASM>(S, ld, rows, W, cols, c0, out, ld_out, len, scale, st);
        else if (nc <= 16) launch_lift<T, 16, TO, ASM>(S, ld, rows, W, cols, c0, out, ld_out, len, scale, st);
        else launch_lift<T, 32, TO, ASM>(S, ld, rows, W, cols, c0, out, ld_out, len, scale, st);
    }
}

void ts_lift(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols, void* out,
             int64_t ld_out, int64_t len, cudaStream_t st) {
    KB_REQUIRE(rows <= 1024, "lift: too many basis vectors (%d)", rows);
    if (dtype == KB_F32) lift_cols<float, float, false>(S, ld, rows, W, cols, out, ld_out, len, nullptr, st);
    else lift_cols<double, double, false>(S, ld, rows, W, cols, out, ld_out, len, nullptr, st);
}

void ts_lift_f64(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols, double* out,
                 int64_t ld_out, int64_t len, const double* scale, cudaStream_t st) {
    KB_REQUIRE(rows <= 1024, "lift: too many basis vectors (%d)", rows);
    if (dtype == KB_F32) lift_cols<float, double, true>(S, ld, rows, W, cols, out, ld_out, len, scale, st);
    else lift_cols<double, double, true>(S, ld, rows, W, cols, out, ld_out, len, scale, st);
}

}  // namespace kb

// ---------------------------------------------------------------- PSF normalisation
// dst = (T)(src / divisor): the reference's Psf normalisation k / k.sum()
// (blurmodel.py:25-65) followed by the working-precision cast, on the device
// (IEEE division and round-to-nearest cast: bitwise numpy's (k / total).astype(T)).
namespace kb {
template <typename T>
__global__ void __launch_bounds__(256) k_div_cast(const double* __restrict__ src, double divisor, T* __restrict__ dst,
                                                  int64_t count) {
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < count; e += (int64_t)gridDim.x * blockDim.x)
        dst[e] = (T)__ddiv_rn(src[e], divisor);
}
}  // namespace kb

extern "C" int kb_div_cast(const double* src, double divisor, int dtype, void* dst, int64_t count, kb_stream_t stream) {
    using namespace kb;
    KB_GUARD({
        KB_REQUIRE(src && dst && count >= 0, "bad arguments");
        KB_REQUIRE(dtype == KB_F32 || dtype == KB_F64, "dtype must be KB_F32 or KB_F64");
        if (count == 0) return KB_OK;
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(count, 256), 8 * kSMs);
        if (dtype == KB_F32)
            k_div_cast<float><<<blocks, 256, 0, as_stream(stream)>>>(src, divisor, static_cast<float*>(dst), count);
        else
            k_div_cast<double><<<blocks, 256, 0, as_stream(stream)>>>(src, divisor, static_cast<double*>(dst), count);
        KB_LAUNCH_CHECK();
    })
}

// ---------------------------------------------------------------- PSF transpose
// K^T for the column-coalesced R(A)^T products; done on the device so the
// host uploads the PSF once.
namespace kb {
template <typename T>
__global__ void __launch_bounds__(256) k_transpose(const T* __restrict__ src, int64_t rows, int64_t cols,
                                                   T* __restrict__ dst) {
    __shared__ T tile[32][33];
    const int64_t c0 = (int64_t)blockIdx.x * 32, r0 = (int64_t)blockIdx.y * 32;
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t r = r0 + i, c = c0 + threadIdx.x;
        if (r < rows && c < cols) tile[i][threadIdx.x] = src[r * cols + c];
    }
    __syncthreads();
    for (int i = threadIdx.y; i < 32; i += 8) {
        const int64_t c = c0 + i, r = r0 + threadIdx.x;
        if (r < rows && c < cols) dst[c * rows + r] = tile[threadIdx.x][i];
    }
}
}  // namespace kb

extern "C" int kb_transpose(int dtype, const void* src, int64_t rows, int64_t cols, void* dst,
                            kb_stream_t stream) {
    using namespace kb;
    KB_GUARD({
        KB_REQUIRE(src && dst && rows >= 0 && cols >= 0, "bad arguments");
        KB_REQUIRE(dtype == KB_F32 || dtype == KB_F64, "dtype must be KB_F32 or KB_F64");
        if (rows == 0 || cols == 0) return KB_OK;
        KB_REQUIRE(cdiv(rows, 32) < 65536, "too many rows");
        const dim3 grid((unsigned)cdiv(cols, 32), (unsigned)cdiv(rows, 32)), block(32, 8);
        if (dtype == KB_F32)
            k_transpose<float><<<grid, block, 0, as_stream(stream)>>>(static_cast<const float*>(src), rows, cols,
                                                                      static_cast<float*>(dst));
        else
            k_transpose<double><<<grid, block, 0, as_stream(stream)>>>(static_cast<const double*>(src), rows,
                                                                       cols, static_cast<double*>(dst));
        KB_LAUNCH_CHECK();
    })
}
