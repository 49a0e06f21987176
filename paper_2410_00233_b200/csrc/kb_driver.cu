// C ABI for the low-rank engines: operator products, tall-skinny kernels,
// orthonormalize, the eGKB driver loop, lifts and factor assembly.
//
// The eGKB loop (lowrank.py:207-303) runs here in C++: each iteration queues
// ~12 kernels (two operator products, 3+3 reorthogonalisation passes and a
// scalar collect) and performs ONE device->host read of four scalars
// (t, ||u||, alpha, ||B^T s||) for the breakdown tests and the rank rule.
#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "kb_ops.cuh"

namespace kb {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

// ------------------------------------------------------------------ profiling
bool g_prof = false;
struct ProfRec { cudaEvent_t a, b; int cls; double bytes, flops; };
static std::vector<ProfRec> g_recs;
static size_t g_nrec = 0;

void prof_record(cudaStream_t st, int cls, double bytes, double flops, bool start) {
    if (start) {
        if (g_nrec == g_recs.size()) {
            ProfRec r{};
            cudaEventCreate(&r.a);
            cudaEventCreate(&r.b);
            g_recs.push_back(r);
        }
        ProfRec& r = g_recs[g_nrec];
        r.cls = cls;
        r.bytes = bytes;
        r.flops = flops;
        cudaEventRecord(r.a, st);
    } else {
        cudaEventRecord(g_recs[g_nrec].b, st);
        ++g_nrec;
    }
}

void prof_set_last_bytes(double bytes) {
    if (g_nrec > 0) g_recs[g_nrec - 1].bytes = bytes;
}

void dense_gemv64(const double* A, int64_t lda, int64_t rows, int64_t cols, const double* x,
                  double* y, int transpose, double* part, unsigned* counters, cudaStream_t st);

// copy up to 4 device scalars into destinations (single tiny launch)
__global__ void k_scalars(const double* a0, double* d0, const double* a1, double* d1,
                          const double* a2, double* d2, const double* a3, double* d3) {
    if (threadIdx.x == 0) {
        if (a0) *d0 = *a0;
        if (a1) *d1 = *a1;
        if (a2) *d2 = *a2;
        if (a3) *d3 = *a3;
    }
}
static void scalars(cudaStream_t st, const double* a0, double* d0, const double* a1 = nullptr,
                    double* d1 = nullptr, const double* a2 = nullptr, double* d2 = nullptr,
                    const double* a3 = nullptr, double* d3 = nullptr) {
    k_scalars<<<1, 32, 0, st>>>(a0, d0, a1, d1, a2, d2, a3, d3);
    KB_LAUNCH_CHECK();
}

template <typename T>
__global__ void k_toeplitz_lift(const T* __restrict__ coef, int64_t ldc, int L, int center, int k,
                                int side, T* __restrict__ out, int64_t ld_out, int refl) {
    const int64_t len = (int64_t)side * side;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x) {
        const unsigned a = (unsigned)e / (unsigned)side;
        const int b = (int)((unsigned)e - a * (unsigned)side);
        const int u = b - (int)a + center;
        const bool ok = (u >= 0 && u < L);
        if (!refl) {
            for (int c = 0; c < k; ++c) out[(int64_t)c * ld_out + e] = ok ? coef[(int64_t)c * ldc + u] : T(0);
        } else {
            // Toeplitz + Hankel families of the reflexive BC (kb_ops.cuh ra_bcast)
            const int s = (int)a + b + 1 + center, h = s - 2 * side;
            for (int c = 0; c < k; ++c) {
                const T* cc = coef + (int64_t)c * ldc;
                double y = ok ? (double)cc[u] : 0.0;
                if (s < L) y += (double)cc[s];
                if (h >= 0) y += (double)cc[h];
                out[(int64_t)c * ld_out + e] = (T)y;
            }
        }
    }
}

struct SigmaParam {
    double v[256];
};

template <typename T>
__global__ void k_assemble(const T* __restrict__ u, int64_t ldu, const T* __restrict__ v, int64_t ldv,
                           const SigmaParam sigma, int k, int64_t len_u, int64_t len_v,
                           double* __restrict__ f, double* __restrict__ g) {
    const int i = blockIdx.y;
    const double s = sigma.v[i];
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len_u || e < len_v;
         e += (int64_t)gridDim.x * blockDim.x) {
        if (e < len_u) f[(int64_t)i * len_u + e] = s * (double)u[(int64_t)i * ldu + e];
        if (e < len_v) g[(int64_t)i * len_v + e] = (double)v[(int64_t)i * ldv + e];
    }
}

static void validate_op(const kb_operator* op) {
    KB_REQUIRE(op != nullptr, "null operator");
    KB_REQUIRE(op->dtype == KB_F32 || op->dtype == KB_F64, "unsupported dtype code %d", op->dtype);
    KB_REQUIRE(op->rows >= 1 && op->cols >= 1, "operator has an empty shape");
    if (ra_is_operator(op->kind)) {
        KB_REQUIRE(op->k && op->kt, "R(A) operator needs the PSF and its transpose");
        KB_REQUIRE(op->kh >= 1 && op->kw >= 1 && (op->kh % 2) == 1 && (op->kw % 2) == 1,
                   "PSF support must be odd in both dimensions, got (%d, %d)", op->kh, op->kw);
        KB_REQUIRE(op->side >= 1 && (int64_t)op->side * op->side == op->rows && op->rows == op->cols,
                   "R(A) shape must be n^2 x n^2");
        // blurmodel.py:100-101: one reflection must cover the support
        KB_REQUIRE(op->kind == KB_OP_RA_ZERO || (op->kh <= 2 * op->side - 1 && op->kw <= 2 * op->side - 1),
                   "PSF support too large for single reflection at this image size");
    } else if (op->kind == KB_OP_SPARSE) {
        KB_REQUIRE(op->sp_rowptr && op->sp_col && op->sp_val && op->spt_rowptr && op->spt_col && op->spt_val,
                   "sparse operator needs the CSR arrays of R and R^T");
        KB_REQUIRE(op->nnz >= 0 && op->rows < (1ll << 31) && op->cols < (1ll << 31), "bad sparse operator");
    } else {
        KB_REQUIRE(op->kind == KB_OP_DENSE, "unknown operator kind %d", op->kind);
        KB_REQUIRE(op->a != nullptr && op->lda >= op->cols, "bad dense operator");
        KB_REQUIRE(op->rows < (1ll << 31) && op->cols < (1ll << 31), "dense operator too large");
    }
}

static int64_t op_len(const kb_operator* op) { return std::max(op->rows, op->cols); }

// kb_refarith.cu: the reference-arithmetic engine (KB_ARITH_OPENBLAS_*)
struct RefOut {
    std::vector<double> alphas, ts, zetas, nus;
    int done = 1, fired = -1, reason = 0, breakdown = 0, tbreak = 0, err = 0;
};
size_t egkb_openblas_ws_bytes(const kb_operator* op, int capacity);
void egkb_openblas(const kb_operator* op, const kb_egkb_config* cfg, const void* y0, kb_egkb_state* st,
                   int lanes, double tol, void* wsp, size_t ws_bytes, RefOut& o, cudaStream_t s);

// ------------------------------------------------------------------ eGKB
// The whole bidiagonalisation (lowrank.py:207-303) is ONE CUDA graph: an
// init stage (s1 = y0/|y0|, q1 = B^T s1/alpha1) followed by a conditional
// WHILE node whose body is one Golub-Kahan iteration (two operator products,
// the reorthogonalisation passes) plus a one-thread control kernel that
// applies the reference's breakdown tests and nu rank rule on the device and
// sets the loop condition.  Kernels address basis slot `done` through
// device-resolved references, so the body is captured once and replayed.
// The host reads the trace back once, after the graph.  A host-driven
// ("eager") replay of the same body is used when kernel profiling is on.
enum { H_DONE = 0, H_FIRED, H_REASON, H_STOP, H_BREAK, H_TBREAK, H_OVERFLOW, H_ERR, H_NA, H_NT, H_NN,
       H_COUNT = 16 };

struct EgkbCtl {
    int* hdr;
    double *alphas, *ts, *zetas, *nus;
    const double *t_ptr, *u2_ptr, *a_ptr, *p2_ptr;
    double tol, tau;
    int k_max, p, k_min, cap;
    cudaGraphConditionalHandle handle;
    int use_cond;
};

__global__ void k_egkb_init(EgkbCtl c) {
    if (threadIdx.x != 0) return;
    int* h = c.hdr;
    for (int i = 0; i < H_COUNT; ++i) h[i] = 0;
    h[H_FIRED] = -1;
    h[H_DONE] = 1;
    const double t1 = *c.t_ptr, a1 = *c.a_ptr;   // here: |y0| and |B^T s1|
    c.ts[0] = t1;
    c.alphas[0] = a1;
    c.zetas[0] = a1 * t1;
    c.nus[0] = 1e308;
    h[H_NA] = h[H_NT] = h[H_NN] = 1;
    if (t1 == 0.0) h[H_ERR] = 1;          // ValidationError: zero starting vector
    else if (a1 == 0.0) h[H_ERR] = 2;     // NumericalError: operator annihilates y0
    if (h[H_ERR]) h[H_STOP] = 1;
    if (c.use_cond) cudaGraphSetConditional(c.handle, h[H_STOP] ? 0u : 1u);
}

__global__ void k_egkb_control(EgkbCtl c) {
    if (threadIdx.x != 0) return;
    int* h = c.hdr;
    const double t_new = *c.t_ptr, unorm = sqrt(*c.u2_ptr);
    const double a_new = *c.a_ptr, pre = sqrt(*c.p2_ptr);
    if (t_new <= c.tol * unorm) {                        // lowrank.py:243-246
        h[H_BREAK] = h[H_TBREAK] = 1;
        h[H_STOP] = 1;
    } else if (a_new <= c.tol * pre) {                   // lowrank.py:255-259
        h[H_BREAK] = 1;
        c.ts[h[H_NT]++] = t_new;
        h[H_STOP] = 1;
    } else {                                             // lowrank.py:260-277
        c.ts[h[H_NT]++] = t_new;
        c.alphas[h[H_NA]++] = a_new;
        const double zeta = a_new * t_new;
        const double nu = sqrt(zeta * c.zetas[h[H_NN] - 1]);
        c.zetas[h[H_NN]] = zeta;
        c.nus[h[H_NN]] = nu;
        h[H_NN]++;
        const int done = ++h[H_DONE];
        if (h[H_FIRED] < 0) {
            const double prev = c.nus[h[H_NN] - 2];
            if (nu > prev) {
                h[H_FIRED] = max(done - 1, c.k_min);
                h[H_REASON] = KB_STOP_NU_ROSE;
            } else if (nu < c.tau) {
                h[H_FIRED] = max(done, c.k_min);
                h[H_REASON] = KB_STOP_NU_BELOW_TOL;
            }
        }
        const int limit = h[H_FIRED] >= 0 ? h[H_FIRED] + c.p + 1 : c.k_max + 1;
        if (done >= limit) h[H_STOP] = 1;
        if (done + 1 > c.cap) { h[H_STOP] = 1; h[H_OVERFLOW] = 1; }
    }
    if (c.use_cond) cudaGraphSetConditional(c.handle, h[H_STOP] ? 0u : 1u);
}

size_t pk_scratch_doubles(int lmax, int cap);
bool egkb_persistent(const kb_operator* op, const kb_egkb_config* cfg, kb_egkb_state* st, const void* y0,
                     int* hdr, double* trace, double* scratch, void* raw, double tol, double** scales_out,
                     cudaStream_t s);
void prof_set_last_bytes(double bytes);
size_t ra_block_scratch_doubles(int n, int lmax, int nv);
bool ra_block_apply(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy, int nv,
                    int transpose, double* scratch, cudaStream_t st);
constexpr int KB_BLOCK_MAXV = 16;

struct EgkbWs {
    double* pk = nullptr;  // persistent-kernel scratch
    void* pkraw = nullptr; // two pending vectors (2 N elements)
    OpPlan plan;
    ReorthWs rw;
    double* red_s;      // coefficient slots (capacity + 8)
    double* red_s2;
    double* red_q;
    double* red_q2;
    double* fx;         // fixed scalars: [0..15] s-step, [16..31] q-step, [32..47] init
    int* hdr;
    double* trace;      // alphas | ts | zetas | nus   (4 x capacity)
    void* y0slot;       // private copy of y0 (graph input)
};

static void egkb_ws_size(const kb_operator* op, int capacity, Sizer& s) {
    op_plan_size(op, s);
    reorth_ws_size(op_len(op), capacity + 1, s);
    for (int i = 0; i < 4; ++i) s.take<double>(capacity + 16);
    s.take<double>(64);
    s.take<int>(H_COUNT);
    s.take<double>(4 * (size_t)capacity);
    s.take<double>((size_t)op->rows);
    s.take<double>(pk_scratch_doubles(std::max(op->kh, op->kw), capacity));
    s.take<double>(2 * (size_t)op_len(op));
}

static EgkbWs egkb_ws_make(const kb_operator* op, int capacity, Arena& a) {
    EgkbWs w;
    w.plan = op_plan_make(op, a);
    w.rw = reorth_ws_make(op_len(op), capacity + 1, a);
    w.red_s = a.take<double>(capacity + 16);
    w.red_s2 = a.take<double>(capacity + 16);
    w.red_q = a.take<double>(capacity + 16);
    w.red_q2 = a.take<double>(capacity + 16);
    w.fx = a.take<double>(64);
    w.hdr = a.take<int>(H_COUNT);
    w.trace = a.take<double>(4 * (size_t)capacity);
    w.y0slot = a.take<double>((size_t)op->rows);
    w.pk = a.take<double>(pk_scratch_doubles(std::max(op->kh, op->kw), capacity));
    w.pkraw = a.take<double>(2 * (size_t)op_len(op));
    return w;
}

static double eps_of(int dtype) { return dtype == KB_F32 ? 1.1920928955078125e-07 : 2.220446049250313e-16; }

// Thin SVD of the lower-bidiagonal C (rows x k; C[i,i] = alphas[i],
// C[i+1,i] = ts[i+1]; lowrank.py:308-316) on the host: one-sided (Hestenes)
// Jacobi in fp64, cyclic pair order, converged to 1e-15 (high relative
// accuracy on a bidiagonal; ~10 us for k = 13), sorted descending.  Then
// W_u = U_C[:, :chosen], W_v = V_C[:, :chosen] (working dtype, row stride
// chosen) and sigma (fp64 of the working-precision values) go to the device
// in one stream-ordered copy from pinned memory -- the lift reads them there.
static void svd_c_upload(int dtype, const double* alphas, const double* ts, int rows, int k, int chosen,
                         kb_egkb_state* st, cudaStream_t s) {
    std::vector<double> A((size_t)rows * k, 0.0), V((size_t)k * k, 0.0);   // column-major
    for (int j = 0; j < k; ++j) {
        A[(size_t)j * rows + j] = alphas[j];
        if (j + 1 < rows) A[(size_t)j * rows + j + 1] = ts[j + 1];
        V[(size_t)j * k + j] = 1.0;
    }
    for (int sweep = 0; sweep < 60; ++sweep) {
        bool rot = false;
        for (int p = 0; p < k - 1; ++p)
            for (int q = p + 1; q < k; ++q) {
                double* Ap = &A[(size_t)p * rows];
                double* Aq = &A[(size_t)q * rows];
                double al = 0.0, be = 0.0, ga = 0.0;
                for (int i = 0; i < rows; ++i) {
                    al += Ap[i] * Ap[i];
                    be += Aq[i] * Aq[i];
                    ga += Ap[i] * Aq[i];
                }
                if (ga == 0.0 || !(ga * ga > 1e-30 * al * be)) continue;
                const double zeta = (be - al) / (2.0 * ga);
                const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (std::fabs(zeta) + std::sqrt(1.0 + zeta * zeta));
                const double c = 1.0 / std::sqrt(1.0 + t * t), sn = c * t;
                for (int i = 0; i < rows; ++i) {
                    const double u = Ap[i], w = Aq[i];
                    Ap[i] = c * u - sn * w;
                    Aq[i] = sn * u + c * w;
                }
                double* Vp = &V[(size_t)p * k];
                double* Vq = &V[(size_t)q * k];
                for (int i = 0; i < k; ++i) {
                    const double u = Vp[i], w = Vq[i];
                    Vp[i] = c * u - sn * w;
                    Vq[i] = sn * u + c * w;
                }
                rot = true;
            }
        if (!rot) break;
    }
    std::vector<double> sig(k);
    std::vector<int> perm(k);
    for (int j = 0; j < k; ++j) {
        double s2 = 0.0;
        for (int i = 0; i < rows; ++i) s2 += A[(size_t)j * rows + i] * A[(size_t)j * rows + i];
        sig[j] = std::sqrt(s2);
        perm[j] = j;
    }
    std::stable_sort(perm.begin(), perm.end(), [&](int a, int b) { return sig[a] > sig[b]; });
    // staging: [W_u | W_v | sigma], 16-byte aligned blocks (pinned, reused once the copy is done)
    const size_t esz = dtype == KB_F32 ? 4 : 8;
    const size_t bu = (size_t)rows * chosen * esz, bv = (size_t)k * chosen * esz, bs = sizeof(double) * chosen;
    static thread_local char* stage = nullptr;
    static thread_local size_t stage_bytes = 0;
    static thread_local cudaEvent_t done = nullptr;
    if (!done) KB_CUDA(cudaEventCreateWithFlags(&done, cudaEventDisableTiming));
    KB_CUDA(cudaEventSynchronize(done));   // the previous upload out of `stage` has finished
    // one copy when the device blocks follow each other inside their declared
    // capacity^2-element extents (lowrank.egkb's svdbuf): the staging then mirrors
    // the device offsets, and the gap bytes it also writes lie inside the W_u / W_v
    // blocks the header gives to the library -- never in a neighbouring allocation
    const char* du = static_cast<const char*>(st->wu_dev);
    const char* dv = static_cast<const char*>(st->wv_dev);
    const char* ds = reinterpret_cast<const char*>(st->sigma_dev);
    const size_t ext = (size_t)st->capacity * (size_t)st->capacity * esz;
    const bool one = dv >= du + bu && ds >= dv + bv && (size_t)(dv - du) <= ext && (size_t)(ds - dv) <= ext &&
                     ((uintptr_t)(dv - du) % 8 == 0) && ((uintptr_t)(ds - du) % 8 == 0);
    const size_t ov = one ? (size_t)(dv - du) : bu, os = one ? (size_t)(ds - du) : bu + bv;
    const size_t need = os + bs;
    if (stage_bytes < need) {
        if (stage) cudaFreeHost(stage);
        KB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage), need));
        stage_bytes = need;
    }
    char* pu = stage;
    char* pv = stage + ov;
    double* ps = reinterpret_cast<double*>(stage + os);
    for (int c = 0; c < chosen; ++c) {
        const int j = perm[c];
        const double sv = sig[j];
        ps[c] = dtype == KB_F32 ? (double)(float)sv : sv;
        st->sigma_host[c] = ps[c];
        // lift weights for the STORED basis vectors: basis i is stored as (normalised_i / scale_i)
        for (int i = 0; i < rows; ++i) {
            const double u = (sv > 0.0 ? A[(size_t)j * rows + i] / sv : 0.0) * (st->s_scale_host ? st->s_scale_host[i] : 1.0);
            if (dtype == KB_F32) reinterpret_cast<float*>(pu)[(size_t)i * chosen + c] = (float)u;
            else reinterpret_cast<double*>(pu)[(size_t)i * chosen + c] = u;
        }
        for (int i = 0; i < k; ++i) {
            const double w = V[(size_t)j * k + i] * (st->q_scale_host ? st->q_scale_host[i] : 1.0);
            if (dtype == KB_F32) reinterpret_cast<float*>(pv)[(size_t)i * chosen + c] = (float)w;
            else reinterpret_cast<double*>(pv)[(size_t)i * chosen + c] = w;
        }
    }
    if (one) {
        KB_CUDA(cudaMemcpyAsync(st->wu_dev, pu, need, cudaMemcpyHostToDevice, s));
    } else {
        KB_CUDA(cudaMemcpyAsync(st->wu_dev, pu, bu, cudaMemcpyHostToDevice, s));
        KB_CUDA(cudaMemcpyAsync(st->wv_dev, pv, bv, cudaMemcpyHostToDevice, s));
        KB_CUDA(cudaMemcpyAsync(st->sigma_dev, ps, bs, cudaMemcpyHostToDevice, s));
    }
    KB_CUDA(cudaEventRecord(done, s));
}

static int egkb_capacity(const kb_egkb_config* c) {
    // Loop limit is fired_k + p + 1 with fired_k <= max(k_max, k_min), else
    // k_max + 1; the left basis may hold one more vector than iterations.
    return std::max(c->k_max, c->k_min) + c->p + 3;
}

// One half step on device-resolved slots: out[done] = normalise(reorth(B x - beta prev)).
// Returns pointers to the new norm (t or alpha) and |B x|^2 (fixed addresses).
static void half_step(const kb_operator* op, EgkbWs& w, int transpose, const VecRef& x, const VecRef& prev,
                      const double* beta, const void* S, int64_t ld, const MRef& m, int passes,
                      const VecRef& out, double* red1, double* red2, double* fx, const double** norm,
                      const double** y2, cudaStream_t st) {
    const int64_t len = transpose ? op->cols : op->rows;
    Src src = op_source(w.plan, x, transpose, st);
    src.prev = prev;
    src.beta = beta;
    const bool proj = m.max > 0;
    reorth_pass(op->dtype, src, S, ld, m, nullptr, nullptr, proj, VecRef(), nullptr, len, red1, fx + 0, w.rw, st);
    *y2 = fx + 1;
    if (!proj) {
        *norm = fx + 3;
        reorth_pass(op->dtype, src, S, ld, m, nullptr, nullptr, false, out, fx + 3, len, nullptr, fx + 8, w.rw, st);
    } else if (passes >= 2) {
        reorth_pass(op->dtype, src, S, ld, m, red1, nullptr, true, VecRef(), nullptr, len, red2, fx + 4, w.rw, st);
        *norm = fx + 6;   // Pythagorean norm after the second projection
        reorth_pass(op->dtype, src, S, ld, m, red1, red2, false, out, fx + 6, len, nullptr, fx + 8, w.rw, st);
    } else {
        // one classical GS pass: write the projected vector, then normalise in place
        reorth_pass(op->dtype, src, S, ld, m, red1, nullptr, false, out, nullptr, len, nullptr, fx + 4, w.rw, st);
        *norm = fx + 7;
        Src self;
        self.z = out;
        self.mode = SRC_BUFT;
        reorth_pass(op->dtype, self, S, ld, MRef::fixed(0), nullptr, nullptr, false, out, fx + 7, len, nullptr,
                    fx + 8, w.rw, st);
    }
}

struct EgkbPlan {
    int done_host = -1;   // eager mode: iteration count known on the host (byte accounting)
    const kb_operator* op;
    const kb_egkb_config* cfg;
    kb_egkb_state* st;
    EgkbWs w;
    EgkbCtl ctl;
};

static void enqueue_init(EgkbPlan& P, cudaStream_t s) {
    const kb_operator* op = P.op;
    EgkbWs& w = P.w;
    double* fxi = w.fx + 32;
    // s1 = y0 / |y0|   (lowrank.py:207-210)
    Src sy;
    sy.z = VecRef::at(w.y0slot);
    sy.mode = SRC_BUFT;
    reorth_pass(op->dtype, sy, nullptr, 0, MRef::fixed(0), nullptr, nullptr, false, VecRef(), nullptr, op->rows,
                nullptr, fxi + 0, w.rw, s);
    reorth_pass(op->dtype, sy, nullptr, 0, MRef::fixed(0), nullptr, nullptr, false, VecRef::at(P.st->s_basis),
                fxi + 3, op->rows, nullptr, fxi + 4, w.rw, s);
    // q1 = B^T s1 / alpha1   (lowrank.py:211-215); alpha1 lands where the loop reads alpha
    Src src = op_source(w.plan, VecRef::at(P.st->s_basis), 1, s);
    double* fq = w.fx + 16;
    reorth_pass(op->dtype, src, nullptr, 0, MRef::fixed(0), nullptr, nullptr, false, VecRef(), nullptr, op->cols,
                nullptr, fq + 4, w.rw, s);
    reorth_pass(op->dtype, src, nullptr, 0, MRef::fixed(0), nullptr, nullptr, false, VecRef::at(P.st->q_basis),
                fq + 7, op->cols, nullptr, fq + 8, w.rw, s);
    EgkbCtl c = P.ctl;
    c.t_ptr = fxi + 3;
    c.a_ptr = fq + 7;
    k_egkb_init<<<1, 32, 0, s>>>(c);
    KB_LAUNCH_CHECK();
}

static void enqueue_body(EgkbPlan& P, cudaStream_t s) {
    const kb_operator* op = P.op;
    const kb_egkb_config* cfg = P.cfg;
    kb_egkb_state* st = P.st;
    EgkbWs& w = P.w;
    const int* done = w.hdr + H_DONE;
    const int cap = st->capacity;
    const int passes = cfg->reorth_passes >= 2 ? 2 : 1;
    double* fs = w.fx;
    double* fq = w.fx + 16;
    const double *t_ptr, *u2, *a_ptr, *p2;
    // s step (lowrank.py:237-247): u = B q_done-1 ; s_raw = u - alpha s_done-1 ; MGS vs S
    MRef ms;
    if (cfg->full_reorth) { ms.idx = done; ms.mul = 1; ms.add = 0; ms.max = cap; ms.acct = P.done_host; }
    half_step(op, w, 0, VecRef::slot(st->q_basis, done, -1, st->ld_q), VecRef::slot(st->s_basis, done, -1, st->ld_s),
              fq + (passes >= 2 ? 6 : 7), st->s_basis, st->ld_s, ms, passes,
              VecRef::slot(st->s_basis, done, 0, st->ld_s), w.red_s, w.red_s2, fs, &t_ptr, &u2, s);
    // q step (lowrank.py:249-260): B^T s_new - t q_done-1 ; MGS vs Q (always)
    MRef mq;
    mq.idx = done; mq.mul = 1; mq.add = 0; mq.max = cap; mq.acct = P.done_host;
    half_step(op, w, 1, VecRef::slot(st->s_basis, done, 0, st->ld_s), VecRef::slot(st->q_basis, done, -1, st->ld_q),
              t_ptr, st->q_basis, st->ld_q, mq, passes, VecRef::slot(st->q_basis, done, 0, st->ld_q), w.red_q,
              w.red_q2, fq, &a_ptr, &p2, s);
    EgkbCtl c = P.ctl;
    c.t_ptr = t_ptr;
    c.u2_ptr = u2;
    c.a_ptr = a_ptr;
    c.p2_ptr = p2;
    k_egkb_control<<<1, 32, 0, s>>>(c);
    KB_LAUNCH_CHECK();
}

// graph cache (one entry per distinct argument set)
struct GraphKey {
    kb_operator op;
    kb_egkb_config cfg;
    void *s_basis, *q_basis, *ws;
    int64_t ld_s, ld_q;
    int cap;
    size_t ws_bytes;
    bool operator==(const GraphKey& o) const { return std::memcmp(this, &o, sizeof(GraphKey)) == 0; }
};
struct GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
};
static std::vector<GraphEntry> g_graphs;
static cudaStream_t g_capture_stream = nullptr;

static cudaGraphExec_t build_graph(EgkbPlan& P) {
    if (!g_capture_stream) KB_CUDA(cudaStreamCreateWithFlags(&g_capture_stream, cudaStreamNonBlocking));
    cudaStream_t cs = g_capture_stream;
    const bool prof = g_prof;
    g_prof = false;   // no event timing inside a graph
    cudaGraph_t g = nullptr;
    try {
        KB_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
        cudaStreamCaptureStatus cst;
        cudaGraph_t capg;
        const cudaGraphNode_t* deps = nullptr;
        size_t ndeps = 0;
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphConditionalHandle h;
        KB_CUDA(cudaGraphConditionalHandleCreate(&h, capg, 1, cudaGraphCondAssignDefault));
        P.ctl.handle = h;
        P.ctl.use_cond = 1;
        enqueue_init(P, cs);
        KB_CUDA(cudaStreamGetCaptureInfo(cs, &cst, nullptr, &capg, &deps, &ndeps));
        cudaGraphNodeParams cp = {};
        cp.type = cudaGraphNodeTypeConditional;
        cp.conditional.handle = h;
        cp.conditional.type = cudaGraphCondTypeWhile;
        cp.conditional.size = 1;
        cudaGraphNode_t cnode;
        KB_CUDA(cudaGraphAddNode(&cnode, capg, deps, ndeps, &cp));
        cudaGraph_t body = cp.conditional.phGraph_out[0];
        KB_CUDA(cudaStreamUpdateCaptureDependencies(cs, &cnode, 1, cudaStreamSetCaptureDependencies));
        KB_CUDA(cudaStreamEndCapture(cs, &g));
        // body: one iteration, captured into the while node's graph
        KB_CUDA(cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0, cudaStreamCaptureModeThreadLocal));
        enqueue_body(P, cs);
        cudaGraph_t body_out;
        KB_CUDA(cudaStreamEndCapture(cs, &body_out));
        cudaGraphExec_t exec;
        KB_CUDA(cudaGraphInstantiate(&exec, g, 0));
        KB_CUDA(cudaGraphDestroy(g));
        g_prof = prof;
        return exec;
    } catch (...) {
        g_prof = prof;
        cudaStreamCaptureStatus cst;
        if (cudaStreamIsCapturing(cs, &cst) == cudaSuccess && cst != cudaStreamCaptureStatusNone) {
            cudaGraph_t junk;
            cudaStreamEndCapture(cs, &junk);
            if (junk) cudaGraphDestroy(junk);
        }
        if (g) cudaGraphDestroy(g);
        cudaGetLastError();
        throw;
    }
}

static void egkb_run(const kb_operator* op, const kb_egkb_config* cfg, const void* y0,
                     kb_egkb_state* st, void* wsp, size_t ws_bytes, cudaStream_t s) {
    validate_op(op);
    KB_REQUIRE(cfg && st && y0, "null argument");
    KB_REQUIRE(cfg->k_max >= 1, "k_max must be >= 1");
    KB_REQUIRE(cfg->p >= 0, "p must be >= 0");
    KB_REQUIRE(cfg->k_min >= 1, "k_min must be >= 1");
    const int cap = st->capacity;
    KB_REQUIRE(cap >= egkb_capacity(cfg), "basis capacity %d < required %d", cap, egkb_capacity(cfg));
    KB_REQUIRE(st->s_basis && st->q_basis && st->alphas_host && st->ts_host && st->zetas_host &&
                   st->nus_host, "missing basis / trace buffers");
    const size_t esz = op->dtype == KB_F32 ? 4 : 8;
    if (cfg->arith != KB_ARITH_FAST) {
        KB_REQUIRE(cfg->arith == KB_ARITH_OPENBLAS_SKX || cfg->arith == KB_ARITH_OPENBLAS_HSW,
                   "unknown arithmetic %d", cfg->arith);
        const double tol = cfg->break_tol >= 0 ? cfg->break_tol : std::sqrt(eps_of(op->dtype));
        RefOut o;
        egkb_openblas(op, cfg, y0, st, cfg->arith == KB_ARITH_OPENBLAS_SKX ? 64 : 32, tol, wsp, ws_bytes, o, s);
        if (o.err == 1) {
            set_error("starting vector must be nonzero");
            throw Fail{KB_EVALIDATION};
        }
        if (o.err == 2) {
            set_error("operator annihilates the starting vector");
            throw Fail{KB_ENUMERICAL};
        }
        int k_p, rows;
        if (o.breakdown && o.tbreak) { k_p = o.done; rows = o.done; }
        else if (o.breakdown) { k_p = o.done; rows = o.done + 1; }
        else { k_p = o.done - 1; rows = o.done; }
        int chosen, reason;
        if (o.fired >= 0) { chosen = std::min(o.fired, k_p); reason = o.reason; }
        else if (o.breakdown) { chosen = k_p; reason = KB_STOP_BREAKDOWN; }
        else { chosen = std::min(cfg->k_max, k_p); reason = KB_STOP_HIT_KMAX; }
        if (chosen < 1 || k_p < 1) {
            set_error("bidiagonalization broke down before producing any factors");
            throw Fail{KB_ENUMERICAL};
        }
        const int na = (int)o.alphas.size(), nt = (int)o.ts.size(), nn = (int)o.nus.size();
        o.alphas.resize(std::max<size_t>(o.alphas.size(), (size_t)rows + 1), 0.0);
        o.ts.resize(std::max<size_t>(o.ts.size(), (size_t)rows + 1), 0.0);
        if (st->s_scale_host && st->q_scale_host)   // normalised vectors stored: unit scales (before the lift weights)
            for (int i = 0; i < cap; ++i) st->s_scale_host[i] = st->q_scale_host[i] = 1.0;
        if (st->wu_dev) {
            KB_REQUIRE(st->wv_dev && st->sigma_dev && st->sigma_host, "SVD outputs incomplete");
            svd_c_upload(op->dtype, o.alphas.data(), o.ts.data(), rows, k_p, chosen, st, s);
        }
        st->n_alphas = na;
        st->n_ts = nt;
        st->n_nus = nn;
        std::copy(o.alphas.begin(), o.alphas.begin() + st->n_alphas, st->alphas_host);
        std::copy(o.ts.begin(), o.ts.begin() + st->n_ts, st->ts_host);
        std::copy(o.zetas.begin(), o.zetas.end(), st->zetas_host);
        std::copy(o.nus.begin(), o.nus.end(), st->nus_host);
        st->chosen_k = chosen;
        st->k_p = k_p;
        st->rows = rows;
        st->stop_reason = reason;
        st->breakdown = o.breakdown;
        KB_CUDA(cudaStreamSynchronize(s));
        return;
    }
    Arena a(wsp, ws_bytes);
    EgkbPlan P;
    P.op = op;
    P.cfg = cfg;
    P.st = st;
    P.w = egkb_ws_make(op, cap, a);
    EgkbCtl& c = P.ctl;
    c.hdr = P.w.hdr;
    c.alphas = P.w.trace;
    c.ts = P.w.trace + cap;
    c.zetas = P.w.trace + 2 * cap;
    c.nus = P.w.trace + 3 * cap;
    c.tol = cfg->break_tol >= 0 ? cfg->break_tol : std::sqrt(eps_of(op->dtype));
    c.tau = cfg->tau;
    c.k_max = cfg->k_max;
    c.p = cfg->p;
    c.k_min = cfg->k_min;
    c.cap = cap;
    c.handle = 0;
    c.use_cond = 0;

    static thread_local char* hbuf = nullptr;   // pinned trace mailbox
    static thread_local size_t hbuf_bytes = 0;
    // header and trace are adjacent in the workspace (egkb_ws_make): one read-back
    const size_t toff = (size_t)(reinterpret_cast<char*>(P.w.trace) - reinterpret_cast<char*>(P.w.hdr));
    const size_t need = toff + sizeof(double) * 4 * (size_t)cap;
    if (hbuf_bytes < need) {
        if (hbuf) cudaFreeHost(hbuf);
        KB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&hbuf), need));
        hbuf_bytes = need;
    }
    int* hh = reinterpret_cast<int*>(hbuf);
    double* ht = reinterpret_cast<double*>(hbuf + toff);

    static const bool force_eager = std::getenv("KB_EGKB_EAGER") != nullptr;  // e.g. for ncu, which
    // cannot profile kernel nodes of graphs that contain conditional nodes
    static const bool no_pk = std::getenv("KB_EGKB_NO_PERSISTENT") != nullptr;
    bool pk_done = false;
    double* pk_scales = nullptr;
    if (!force_eager && !no_pk)
        pk_done = egkb_persistent(op, cfg, st, y0, P.w.hdr, P.w.trace, P.w.pk, P.w.pkraw, c.tol, &pk_scales, s);
    if (!pk_done) {   // graph / eager engines: counters zeroed, y0 copied into the graph's input slot
        KB_CUDA(cudaMemsetAsync(P.w.plan.counters, 0, sizeof(unsigned) * P.w.plan.n_counters, s));
        KB_CUDA(cudaMemsetAsync(P.w.rw.counter, 0, sizeof(unsigned) * 64, s));
        KB_CUDA(cudaMemcpyAsync(P.w.y0slot, y0, esz * (size_t)op->rows, cudaMemcpyDeviceToDevice, s));
    }
    if (pk_done) {
        // single persistent kernel ran the whole loop
    } else if (!g_prof && !force_eager) {
        GraphKey key;
        std::memset(&key, 0, sizeof(key));
        key.op = *op;
        key.cfg = *cfg;
        key.s_basis = st->s_basis;
        key.q_basis = st->q_basis;
        key.ws = wsp;
        key.ld_s = st->ld_s;
        key.ld_q = st->ld_q;
        key.cap = cap;
        key.ws_bytes = ws_bytes;
        cudaGraphExec_t exec = nullptr;
        for (auto& e : g_graphs)
            if (e.key == key) exec = e.exec;
        if (!exec) {
            exec = build_graph(P);
            if (g_graphs.size() >= 16) {
                cudaGraphExecDestroy(g_graphs.front().exec);
                g_graphs.erase(g_graphs.begin());
            }
            g_graphs.push_back({key, exec});
        }
        KB_CUDA(cudaGraphLaunch(exec, s));
    } else {
        // eager replay of the same kernels (per-kernel event timing)
        enqueue_init(P, s);
        for (;;) {
            KB_CUDA(cudaMemcpyAsync(hh, P.w.hdr, sizeof(int) * H_COUNT, cudaMemcpyDeviceToHost, s));
            KB_CUDA(cudaStreamSynchronize(s));
            if (hh[H_STOP]) break;
            P.done_host = hh[H_DONE];
            enqueue_body(P, s);
        }
    }
    KB_CUDA(cudaMemcpyAsync(hbuf, P.w.hdr, need, cudaMemcpyDeviceToHost, s));
    if (pk_done && pk_scales && st->s_scale_host && st->q_scale_host) {
        KB_CUDA(cudaMemcpyAsync(st->s_scale_host, pk_scales, sizeof(double) * cap, cudaMemcpyDeviceToHost, s));
        KB_CUDA(cudaMemcpyAsync(st->q_scale_host, pk_scales + cap, sizeof(double) * cap, cudaMemcpyDeviceToHost, s));
    }
    KB_CUDA(cudaStreamSynchronize(s));
    if ((!pk_done || !pk_scales) && st->s_scale_host && st->q_scale_host)
        for (int i = 0; i < cap; ++i) st->s_scale_host[i] = st->q_scale_host[i] = 1.0;
    if (hh[H_ERR] == 1) {
        set_error("starting vector must be nonzero");
        throw Fail{KB_EVALIDATION};
    }
    if (hh[H_ERR] == 2) {
        set_error("operator annihilates the starting vector");
        throw Fail{KB_ENUMERICAL};
    }
    KB_REQUIRE(!hh[H_OVERFLOW], "eGKB basis capacity exhausted (%d)", cap);
    const int done = hh[H_DONE];
    const bool breakdown = hh[H_BREAK] != 0, t_break = hh[H_TBREAK] != 0;
    const int fired = hh[H_FIRED];
    int k_p, rows;
    if (breakdown && t_break) { k_p = done; rows = done; }
    else if (breakdown) { k_p = done; rows = done + 1; }
    else { k_p = done - 1; rows = done; }
    int chosen, reason;
    if (fired >= 0) { chosen = std::min(fired, k_p); reason = hh[H_REASON]; }
    else if (breakdown) { chosen = k_p; reason = KB_STOP_BREAKDOWN; }
    else { chosen = std::min(cfg->k_max, k_p); reason = KB_STOP_HIT_KMAX; }
    if (chosen < 1 || k_p < 1) {
        set_error("bidiagonalization broke down before producing any factors");
        throw Fail{KB_ENUMERICAL};
    }
    if (st->wu_dev) {   // small SVD of C (host, C++) and the lift weights, uploaded stream-ordered
        KB_REQUIRE(st->wv_dev && st->sigma_dev && st->sigma_host, "SVD outputs incomplete");
        svd_c_upload(op->dtype, ht, ht + cap, rows, k_p, chosen, st, s);
    }
    st->n_alphas = hh[H_NA];
    st->n_ts = hh[H_NT];
    st->n_nus = hh[H_NN];
    std::copy(ht, ht + st->n_alphas, st->alphas_host);
    std::copy(ht + cap, ht + cap + st->n_ts, st->ts_host);
    std::copy(ht + 2 * cap, ht + 2 * cap + st->n_nus, st->zetas_host);
    std::copy(ht + 3 * cap, ht + 3 * cap + st->n_nus, st->nus_host);
    st->chosen_k = chosen;
    st->k_p = k_p;
    st->rows = rows;
    st->stop_reason = reason;
    st->breakdown = breakdown ? 1 : 0;
    if (pk_done && g_prof) {
        // algorithmic bytes of the run actually executed, SURVEY §8d's eGKB row without
        // the lift: B_egkb = (2 J + 1) B_mv + sum_{j=1..J} 8 N (2 j + 3) over the J executed
        // iterations -- per iteration two R(A) products and, per side, the coefficient and
        // update passes over the j basis vectors plus the prev, raw and written vectors.
        const double N = (double)op->rows, e = (double)esz;
        const double bmv = e * (2.0 * N + (double)op->kh * op->kw);
        double by = bmv;   // the initial product R^T s1
        for (int j = 1; j < done + (breakdown ? 1 : 0); ++j) {
            const double ms = cfg->full_reorth ? j : 0, mq = j;
            by += 2.0 * bmv;
            by += e * N * (2.0 * ms + 3.0) + e * N * (2.0 * mq + 3.0);
        }
        prof_set_last_bytes(by);
    }
}

// ------------------------------------------------------------------ orthonormalize
static void orth_ws_size(int64_t len, int ncol, Sizer& s) {
    reorth_ws_size(len, ncol + 1, s);
    for (int i = 0; i < 3; ++i) s.take<double>(ncol + 16);
    s.take<double>(2 * (size_t)ncol + 16);
}

static void orthonormalize(int dtype, void* Q, int64_t ld, int ncol, int64_t len, double drop_tol,
                           int* bad_col, void* wsp, size_t ws_bytes, cudaStream_t s) {
    KB_REQUIRE(dtype == KB_F32 || dtype == KB_F64, "unsupported dtype");
    KB_REQUIRE(ncol <= len, "cannot orthonormalize %d columns in dimension %lld", ncol, (long long)len);
    if (bad_col) *bad_col = -1;
    if (ncol == 0) return;
    Arena a(wsp, ws_bytes);
    ReorthWs rw = reorth_ws_make(len, ncol + 1, a);
    double* red[3];
    for (int i = 0; i < 3; ++i) red[i] = a.take<double>(ncol + 16);
    double* hist = a.take<double>(2 * (size_t)ncol + 16);  // [t_j | raw_j]
    KB_CUDA(cudaMemsetAsync(rw.counter, 0, sizeof(unsigned) * 64, s));
    double* fx = red[2];
    const size_t esz = dtype == KB_F32 ? 4 : 8;
    for (int j = 0; j < ncol; ++j) {
        void* col = static_cast<char*>(Q) + (size_t)j * ld * esz;
        Src src;
        src.z = VecRef::at(col);
        src.mode = SRC_BUFT;
        const MRef m = MRef::fixed(j);
        const bool any = j > 0;
        // CGS2: coefficients, second-pass coefficients, then the projected, normalised column
        reorth_pass(dtype, src, Q, ld, m, nullptr, nullptr, any, VecRef(), nullptr, len, red[0], fx + 0, rw, s);
        reorth_pass(dtype, src, Q, ld, m, any ? red[0] : nullptr, nullptr, true, VecRef(), nullptr, len, red[1],
                    fx + 4, rw, s);
        reorth_pass(dtype, src, Q, ld, m, any ? red[0] : nullptr, any ? red[1] : nullptr, false, VecRef::at(col),
                    fx + 6, len, nullptr, fx + 8, rw, s);
        scalars(s, fx + 6, hist + j, fx + 3, hist + ncol + j);
    }
    std::vector<double> h(2 * (size_t)ncol);
    KB_CUDA(cudaMemcpyAsync(h.data(), hist, sizeof(double) * 2 * ncol, cudaMemcpyDeviceToHost, s));
    KB_CUDA(cudaStreamSynchronize(s));
    if (drop_tol < 0) {
        double mx = 0.0;
        for (int j = 0; j < ncol; ++j) mx = std::max(mx, h[ncol + j]);
        drop_tol = eps_of(dtype) * std::sqrt((double)len) * mx;
    }
    for (int j = 0; j < ncol; ++j) {
        if (!std::isfinite(h[j])) {
            if (bad_col) *bad_col = -2 - j;
            set_error("non-finite column norm at column %d", j);
            throw Fail{KB_ENUMERICAL};
        }
        if (h[j] <= drop_tol) {
            if (bad_col) *bad_col = j;
            set_error("column %d became numerically zero during orthonormalization", j);
            throw Fail{KB_ENUMERICAL};
        }
    }
}

}  // namespace kb

// ================================================================ C ABI
using namespace kb;

extern "C" const char* kb_last_error(void) { return g_err; }

extern "C" int kb_version(void) { return 1; }


extern "C" void kb_prof_enable(int on) {
    g_prof = on != 0;
    g_nrec = 0;
}

extern "C" int kb_prof_query(int cls, double* ms, long long* launches, double* bytes, double* flops) {
    KB_GUARD({
        double t = 0, by = 0, fl = 0;
        long long n = 0;
        for (size_t i = 0; i < g_nrec; ++i) {
            const ProfRec& r = g_recs[i];
            if (r.cls != cls) continue;
            KB_CUDA(cudaEventSynchronize(r.b));
            float e = 0;
            KB_CUDA(cudaEventElapsedTime(&e, r.a, r.b));
            t += e;
            by += r.bytes;
            fl += r.flops;
            ++n;
        }
        *ms = t;
        *launches = n;
        *bytes = by;
        *flops = fl;
    })
}
extern "C" int kb_op_workspace_bytes(const kb_operator* op, size_t* bytes) {
    KB_GUARD({
        validate_op(op);
        KB_REQUIRE(bytes, "null argument");
        Sizer s;
        op_plan_size(op, s);
        s.take<unsigned>(8);
        if (ra_is_operator(op->kind)) s.take<double>(ra_block_scratch_doubles(op->side, std::max(op->kh, op->kw), KB_BLOCK_MAXV));
        *bytes = s.off;
    })
}

extern "C" int kb_op_apply(const kb_operator* op, const void* x, void* y, int transpose, void* ws,
                           size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        validate_op(op);
        KB_REQUIRE(x && y, "null argument");
        Arena a(ws, ws_bytes);
        OpPlan p = op_plan_make(op, a);
        (void)a.take<unsigned>(8);
        cudaStream_t s = as_stream(stream);
        if (ra_is_operator(op->kind)) {
            double* scr = a.take<double>(ra_block_scratch_doubles(op->side, std::max(op->kh, op->kw), KB_BLOCK_MAXV));
            if (ra_block_apply(op, x, op->cols, y, op->rows, 1, transpose, scr, s)) return KB_OK;
        }
        KB_CUDA(cudaMemsetAsync(p.counters, 0, sizeof(unsigned) * p.n_counters, s));
        Src src = op_source(p, VecRef::at(x), transpose, s);
        src_write(op->dtype, src, y, transpose ? op->cols : op->rows, s);
    })
}

extern "C" int kb_op_apply_block(const kb_operator* op, const void* X, int64_t ldx, void* Y, int64_t ldy,
                                 int nv, int transpose, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        validate_op(op);
        KB_REQUIRE(X && Y && nv >= 0, "bad arguments");
        cudaStream_t s = as_stream(stream);
        const size_t esz = op->dtype == KB_F32 ? 4 : 8;
        const int64_t in_len = transpose ? op->rows : op->cols, out_len = transpose ? op->cols : op->rows;
        KB_REQUIRE(ldx >= in_len && ldy >= out_len, "leading dimensions too small");
        Arena a(ws, ws_bytes);
        OpPlan p = op_plan_make(op, a);
        (void)a.take<unsigned>(8);
        double* scr = nullptr;
        if (ra_is_operator(op->kind))
            scr = a.take<double>(ra_block_scratch_doubles(op->side, std::max(op->kh, op->kw), KB_BLOCK_MAXV));
        for (int v0 = 0; v0 < nv; v0 += KB_BLOCK_MAXV) {
            const int cnt = std::min(KB_BLOCK_MAXV, nv - v0);
            const char* xs = static_cast<const char*>(X) + (size_t)v0 * ldx * esz;
            char* ys = static_cast<char*>(Y) + (size_t)v0 * ldy * esz;
            if (scr && ra_block_apply(op, xs, ldx, ys, ldy, cnt, transpose, scr, s)) continue;
            KB_CUDA(cudaMemsetAsync(p.counters, 0, sizeof(unsigned) * p.n_counters, s));
            for (int v = 0; v < cnt; ++v) {
                Src src = op_source(p, VecRef::at(xs + (size_t)v * ldx * esz), transpose, s);
                src_write(op->dtype, src, ys + (size_t)v * ldy * esz, out_len, s);
            }
        }
    })
}

extern "C" int kb_ts_dots(int dtype, const void* S, int64_t ld, int m, const void* v, int64_t len,
                          double* out, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && out && (S || m == 0), "null argument");
        Arena a(ws, ws_bytes);
        ReorthWs rw = reorth_ws_make(len, m, a);
        double* red = a.take<double>(m + 16);
        cudaStream_t s = as_stream(stream);
        KB_CUDA(cudaMemsetAsync(rw.counter, 0, sizeof(unsigned) * 64, s));
        Src src;
        src.z = VecRef::at(v);
        src.mode = SRC_BUFT;
        double* fix = red + m + 1;
        reorth_pass(dtype, src, S, ld, MRef::fixed(m), nullptr, nullptr, true, VecRef(), nullptr, len, red, fix, rw, s);
        KB_CUDA(cudaMemcpyAsync(out, red, sizeof(double) * m, cudaMemcpyDeviceToDevice, s));
        KB_CUDA(cudaMemcpyAsync(out + m, fix, sizeof(double), cudaMemcpyDeviceToDevice, s));
    })
}

extern "C" int kb_ts_axpy(int dtype, const void* S, int64_t ld, int m, const double* coef, void* v,
                          int64_t len, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && coef && (S || m == 0), "null argument");
        // small private workspace: the pass only needs its reduction scratch
        static thread_local void* scratch = nullptr;
        static thread_local size_t scratch_bytes = 0;
        Sizer sz;
        reorth_ws_size(len, m, sz);
        sz.take<double>(m + 8);
        if (scratch_bytes < sz.off) {
            if (scratch) cudaFree(scratch);
            KB_CUDA(cudaMalloc(&scratch, sz.off));
            KB_CUDA(cudaMemset(scratch, 0, sz.off));
            scratch_bytes = sz.off;
        }
        Arena a(scratch, scratch_bytes);
        ReorthWs rw = reorth_ws_make(len, m, a);
        double* red = a.take<double>(m + 8);
        Src src;
        src.z = VecRef::at(v);
        src.mode = SRC_BUFT;
        reorth_pass(dtype, src, S, ld, MRef::fixed(m), coef, nullptr, false, VecRef::at(v), nullptr, len, nullptr,
                    red, rw, as_stream(stream));
    })
}

extern "C" int kb_ts_lift(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols,
                          void* out, int64_t ld_out, int64_t len, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(S && W && out, "null argument");
        KB_REQUIRE(rows >= 1 && cols >= 1, "empty lift");
        ts_lift(dtype, S, ld, rows, W, cols, out, ld_out, len, as_stream(stream));
    })
}

extern "C" int kb_lift_assemble(int dtype, const void* S, int64_t ld, int rows, const void* W, int cols,
                                const double* scale_dev, double* out, int64_t ld_out, int64_t len,
                                kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(S && W && out && rows >= 1 && cols >= 1 && len >= 0, "bad arguments");
        KB_REQUIRE(dtype == KB_F32 || dtype == KB_F64, "dtype must be KB_F32 or KB_F64");
        ts_lift_f64(dtype, S, ld, rows, W, cols, out, ld_out, len, scale_dev, as_stream(stream));
    })
}

extern "C" int kb_orth_workspace_bytes(int64_t len, int ncol, size_t* bytes) {
    KB_GUARD({
        Sizer s;
        orth_ws_size(len, ncol, s);
        *bytes = s.off;
    })
}

extern "C" int kb_orthonormalize(int dtype, void* Q, int64_t ld, int ncol, int64_t len,
                                 double drop_tol, int* bad_col, void* ws, size_t ws_bytes,
                                 kb_stream_t stream) {
    KB_GUARD(orthonormalize(dtype, Q, ld, ncol, len, drop_tol, bad_col, ws, ws_bytes, as_stream(stream)))
}

extern "C" int kb_egkb_capacity(const kb_egkb_config* cfg) { return cfg ? egkb_capacity(cfg) : -1; }

extern "C" int kb_egkb_workspace_bytes(const kb_operator* op, int capacity, size_t* bytes) {
    KB_GUARD({
        validate_op(op);
        Sizer s;
        egkb_ws_size(op, capacity, s);
        *bytes = std::max(s.off, egkb_openblas_ws_bytes(op, capacity));
    })
}

extern "C" int kb_egkb_run(const kb_operator* op, const kb_egkb_config* cfg, const void* y0,
                           kb_egkb_state* st, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD(egkb_run(op, cfg, y0, st, ws, ws_bytes, as_stream(stream)))
}

extern "C" int kb_toeplitz_lift(int dtype, const void* coef, int64_t ldc, int len_coef, int center,
                                int k, int side, int reflexive, void* out, int64_t ld_out, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(coef && out && k >= 1 && side >= 1, "bad arguments");
        const int64_t len = (int64_t)side * side;
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(len, 256), 8 * kSMs);
        cudaStream_t s = as_stream(stream);
        if (dtype == KB_F32)
            k_toeplitz_lift<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(coef), ldc, len_coef,
                                                          center, k, side, static_cast<float*>(out), ld_out,
                                                          reflexive);
        else
            k_toeplitz_lift<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(coef), ldc, len_coef,
                                                           center, k, side, static_cast<double*>(out), ld_out,
                                                           reflexive);
        KB_LAUNCH_CHECK();
    })
}

extern "C" int kb_kron_assemble(int dtype, const void* u, int64_t ldu, const void* v, int64_t ldv,
                                const double* sigma_host, int k, int64_t len_u, int64_t len_v, double* f,
                                double* g, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(u && v && sigma_host && f && g && k >= 1, "bad arguments");
        KB_REQUIRE(k <= 256, "too many terms (%d > 256)", k);
        cudaStream_t s = as_stream(stream);
        SigmaParam sig{};
        for (int i = 0; i < k; ++i) sig.v[i] = sigma_host[i];
        dim3 grid((unsigned)std::min<int64_t>(cdiv(std::max(len_u, len_v), 256), 4 * kSMs), (unsigned)k);
        if (dtype == KB_F32)
            k_assemble<float><<<grid, 256, 0, s>>>(static_cast<const float*>(u), ldu,
                                                   static_cast<const float*>(v), ldv, sig, k, len_u, len_v, f, g);
        else
            k_assemble<double><<<grid, 256, 0, s>>>(static_cast<const double*>(u), ldu,
                                                    static_cast<const double*>(v), ldv, sig, k, len_u, len_v, f, g);
        KB_LAUNCH_CHECK();
    })
}
