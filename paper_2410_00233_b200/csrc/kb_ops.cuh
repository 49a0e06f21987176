// Kernel launch wrappers shared between translation units (host side).
#pragma once

#include "kb_common.cuh"

namespace kb {

// Source of the generated vector v in the reorthogonalisation passes:
//   SRC_BUFT   : y[e] = ((const T*) z)[e]                          (a stored vector)
//   SRC_BUF64  : y[e] = (T) z[e]                                   (dense op)
//   SRC_TOEP   : y[a*n+b] = (T) z[b - a + center], 0 outside [0,L) (R(A))
enum SrcMode { SRC_BUFT = 0, SRC_BUF64 = 1, SRC_TOEP = 2 };

struct Src {
    const double* z = nullptr;
    int mode = SRC_BUF64;
    int side = 0;
    int center = 0;
    int L = 0;
    const void* prev = nullptr;   // v = y - beta * prev   (prev in T)
    const double* beta = nullptr; // device scalar
};

// Matrix-vector product into an fp64 "source" (either the full vector or
// the Toeplitz coefficient array z for R(A)).
struct OpPlan {
    const kb_operator* op;
    // workspace pieces
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
Src op_source(const OpPlan& p, const void* x, int transpose, cudaStream_t st);
// Writes y (dtype T) from a source.
void src_write(int dtype, const Src& s, void* y, int64_t len, cudaStream_t st);

// Reorthogonalisation pass over basis S (m vectors at stride ld):
//   v = y - beta*prev - S (coefA + coefB)       (coef may be null)
//   red[0..m) = S^T v (if dots), red[m] = ||v||^2, red[m+1] = ||y||^2,
//   red[m+2] = sqrt(max(red[m] - sum_i red[i]^2, 0)), red[m+3] = sqrt(red[m])
//   out = v / *div (if out)
struct ReorthWs {
    double* part = nullptr;
    unsigned* counter = nullptr;
    int max_blocks = 0;
    int max_m = 0;
};
void reorth_ws_size(int64_t len, int max_m, Sizer& s);
ReorthWs reorth_ws_make(int64_t len, int max_m, Arena& a);
void reorth_pass(int dtype, const Src& src, const void* S, int64_t ld, int m, const double* coefA,
                 const double* coefB, bool dots, void* out, const double* div, int64_t len,
                 double* red, const ReorthWs& ws, cudaStream_t st);

void ts_lift(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols, void* out,
             int64_t ld_out, int64_t len, cudaStream_t st);

}  // namespace kb
