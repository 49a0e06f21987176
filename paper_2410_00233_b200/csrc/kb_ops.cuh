// Kernel launch wrappers shared between translation units (host side).
#pragma once

#include "kb_common.cuh"

namespace kb {

// A vector argument that may be resolved on the device at run time:
//   ptr = base + (idx ? (*idx + off) : 0) * ld        (in elements)
// so that one captured CUDA graph can address basis slot `done` of the
// iteration it is executing (the eGKB loop body is a graph while-node).
struct VecRef {
    const void* base = nullptr;
    const int* idx = nullptr;
    int off = 0;
    int64_t ld = 0;
    static VecRef at(const void* p) { VecRef r; r.base = p; return r; }
    static VecRef slot(const void* b, const int* i, int o, int64_t l) {
        VecRef r; r.base = b; r.idx = i; r.off = o; r.ld = l; return r;
    }
    bool null() const { return base == nullptr; }
};

template <typename T>
__device__ __forceinline__ T* resolve(const VecRef& r) {
    T* p = reinterpret_cast<T*>(const_cast<void*>(r.base));
    return r.idx ? p + (int64_t)(*r.idx + r.off) * r.ld : p;
}

// ------------------------------------------------------------------ R(A) index families
// R(A) = P_c K^T P_r^T.  Row (a, b) of P (image cell
// a*n + b) hits index u = b - a + c (Toeplitz, zero and reflexive BC) and, for
// the reflexive BC (blurmodel.py:80-84, 122-126), also u = a + b + 1 + c and
// u = a + b + c + 1 - 2n (Hankel: the reflections below 0 and above n-1).
inline bool ra_is_operator(int kind) { return kind == KB_OP_RA_ZERO || kind == KB_OP_RA_REFLEXIVE; }

// Broadcast P z at cell e = a*n + b (fp64; z in shared memory, length L).
__device__ __forceinline__ double ra_bcast(const double* zs, unsigned e, int n, int c, int L, bool refl) {
    const unsigned a = e / (unsigned)n;
    const int b = (int)(e - a * (unsigned)n);
    const int u = b - (int)a + c;
    double y = (u >= 0 && u < L) ? zs[u] : 0.0;
    if (refl) {
        const int s = (int)a + b + 1 + c;
        if (s < L) y += zs[s];
        if (s - 2 * n >= 0) y += zs[s - 2 * n];
    }
    return y;
}

// Sum of X[a*stride + off] over rows a in [lo, hi) with a = lo + phase (mod 8),
// U independent loads in flight (CG: coherent loads for data written in-kernel).
// The summation order (U-row batches, then the tail) depends on U only through
// the batching of the same ascending row sequence.
template <typename T, bool CG, int U = 8>
__device__ __forceinline__ double band_rows(const T* X, int64_t stride, int64_t off, int lo, int hi, int phase) {
    double acc = 0.0;
    int a = lo + phase;
    const T* p = X + (int64_t)a * stride + off;
    const int64_t step = 8 * stride;
    for (; a + 8 * (U - 1) < hi; a += 8 * U, p += U * step) {
        T q[U];
#pragma unroll
        for (int k = 0; k < U; ++k) q[k] = CG ? __ldcg(p + k * step) : __ldg(p + k * step);
#pragma unroll
        for (int k = 0; k < U; ++k) acc += (double)q[k];
    }
    for (; a < hi; a += 8, p += step) acc += (double)(CG ? __ldcg(p) : __ldg(p));
    return acc;
}

// (P^T x)[u] restricted to image rows [s0, s1), summed by row phase `phase`
// (the caller reduces over the 8 phases and the row segments).
template <typename T, bool CG, int U = 8>
__device__ __forceinline__ double ra_gather_rows(const T* X, int n, int u, int c, int s0, int s1, int phase,
                                                 bool refl) {
    const int d = u - c;   // diagonal b - a = d
    double acc = band_rows<T, CG, U>(X, n + 1, d, max(s0, -d), min(s1, n - d), phase);
    if (refl && u != c) {
        const int s = u > c ? d - 1 : d - 1 + 2 * n;   // anti-diagonal a + b = s
        acc += band_rows<T, CG, U>(X, n - 1, s, max(s0, s - n + 1), min(s1, s + 1), phase);
    }
    return acc;
}

// ra_bcast for the 4 consecutive cells e0..e0+3 (one division when they share a row).
__device__ __forceinline__ void ra_bcast4(const double* zs, unsigned e0, int n, int c, int L, bool refl,
                                          double (&out)[4]) {
    const unsigned a = e0 / (unsigned)n;
    const int b0 = (int)(e0 - a * (unsigned)n);
    if (b0 + 3 < n) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int b = b0 + q;
            const int u = b - (int)a + c;
            double y = (u >= 0 && u < L) ? zs[u] : 0.0;
            if (refl) {
                const int s = (int)a + b + 1 + c;
                if (s < L) y += zs[s];
                if (s - 2 * n >= 0) y += zs[s - 2 * n];
            }
            out[q] = y;
        }
    } else {
#pragma unroll
        for (int q = 0; q < 4; ++q) out[q] = ra_bcast(zs, e0 + q, n, c, L, refl);
    }
}

// Basis size resolved on the device: m = idx ? (*idx) * mul + add : add.
struct MRef {
    const int* idx = nullptr;
    int mul = 0;
    int add = 0;
    int max = 0;   // upper bound (shared-memory sizing)
    int acct = -1; // host-known value for byte accounting (-1: unknown, use max)
    static MRef fixed(int m) { MRef r; r.add = m; r.max = m; r.acct = m; return r; }
};

// Source of the generated vector v in the reorthogonalisation passes:
//   SRC_BUFT   : y[e] = x[e]       (a stored vector in T, e.g. y0 or a slot)
//   SRC_BUF64  : y[e] = (T) z[e]   (dense operator product, fp64 accumulated)
//   SRC_TOEP   : y[a*n+b] = (T) z[b - a + center], 0 outside [0,L)  (R(A))
//   SRC_TOEP_REFL : the same plus the Hankel families (reflexive BC, ra_bcast)
enum SrcMode { SRC_BUFT = 0, SRC_BUF64 = 1, SRC_TOEP = 2, SRC_TOEP_REFL = 3 };

struct Src {
    VecRef z;                     // BUFT: T vector; BUF64/TOEP: fp64 array
    int mode = SRC_BUF64;
    int side = 0;
    int center = 0;
    int L = 0;
    VecRef prev;                  // v = y - beta * prev   (prev in T)
    const double* beta = nullptr; // device scalar
};

// Matrix-vector product into an fp64 "source" (either the full vector or
// the Toeplitz coefficient array z for R(A)).
struct OpPlan {
    const kb_operator* op;
    double* part = nullptr;      // partial sums
    double* w = nullptr;         // diagonal sums (R(A))
    double* z = nullptr;         // output coefficients / full vector
    unsigned* counters = nullptr;
    int64_t n_counters = 0;
    int64_t z_len = 0;
};

void op_plan_size(const kb_operator* op, Sizer& s);
OpPlan op_plan_make(const kb_operator* op, Arena& a);
// Computes the fp64 source for y = op x (or op^T x); returns the Src.
Src op_source(const OpPlan& p, const VecRef& x, int transpose, cudaStream_t st);
// Writes y (dtype T) from a source.
void src_write(int dtype, const Src& s, void* y, int64_t len, cudaStream_t st);

// Reorthogonalisation pass over basis S (m vectors at stride ld):
//   v = y - beta*prev - S (coefA + coefB)       (coef may be null)
//   red[0..m) = S^T v (if dots)
//   fix[0] = ||v||^2, fix[1] = ||y||^2, fix[2] = sqrt(max(fix[0] - sum red_i^2, 0)),
//   fix[3] = sqrt(fix[0])               (four fixed-address scalars)
//   out = v / *div (if out; div may be null)
struct ReorthWs {
    double* part = nullptr;
    unsigned* counter = nullptr;
    int max_blocks = 0;
    int max_m = 0;
};
void reorth_ws_size(int64_t len, int max_m, Sizer& s);
ReorthWs reorth_ws_make(int64_t len, int max_m, Arena& a);
void reorth_pass(int dtype, const Src& src, const void* S, int64_t ld, const MRef& m,
                 const double* coefA, const double* coefB, bool dots, const VecRef& out,
                 const double* div, int64_t len, double* red, double* fix, const ReorthWs& ws,
                 cudaStream_t st);

void ts_lift(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols, void* out,
             int64_t ld_out, int64_t len, cudaStream_t st);
// Same lift with fp64 output out_c = scale[c] * (double)lift_c (scale may be null).
void ts_lift_f64(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols, double* out,
                 int64_t ld_out, int64_t len, const double* scale, cudaStream_t st);

}  // namespace kb
