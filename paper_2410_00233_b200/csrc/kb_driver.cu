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
                                int side, T* __restrict__ out, int64_t ld_out) {
    const int64_t len = (int64_t)side * side;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < len;
         e += (int64_t)gridDim.x * blockDim.x) {
        const unsigned a = (unsigned)e / (unsigned)side;
        const int u = (int)((unsigned)e - a * (unsigned)side) - (int)a + center;
        const bool ok = (u >= 0 && u < L);
        for (int c = 0; c < k; ++c) out[(int64_t)c * ld_out + e] = ok ? coef[(int64_t)c * ldc + u] : T(0);
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
    if (op->kind == KB_OP_RA_ZERO) {
        KB_REQUIRE(op->k && op->kt, "R(A) operator needs the PSF and its transpose");
        KB_REQUIRE(op->kh >= 1 && op->kw >= 1 && (op->kh % 2) == 1 && (op->kw % 2) == 1,
                   "PSF support must be odd in both dimensions, got (%d, %d)", op->kh, op->kw);
        KB_REQUIRE(op->side >= 1 && (int64_t)op->side * op->side == op->rows && op->rows == op->cols,
                   "R(A) shape must be n^2 x n^2");
    } else {
        KB_REQUIRE(op->kind == KB_OP_DENSE, "unknown operator kind %d", op->kind);
        KB_REQUIRE(op->a != nullptr && op->lda >= op->cols, "bad dense operator");
        KB_REQUIRE(op->rows < (1ll << 31) && op->cols < (1ll << 31), "dense operator too large");
    }
}

static int64_t op_len(const kb_operator* op) { return std::max(op->rows, op->cols); }

// ------------------------------------------------------------------ eGKB
struct EgkbWs {
    OpPlan plan;
    ReorthWs rw;
    double* red[6];     // s1 s2 s3 q1 q2 q3, each capacity + 8
    double* cur;        // [0]=alpha, [1]=t
    double* hist;       // [4]: t, |u|^2, alpha, |B^T s|^2
};

static void egkb_ws_size(const kb_operator* op, int capacity, Sizer& s) {
    op_plan_size(op, s);
    reorth_ws_size(op_len(op), capacity + 1, s);
    for (int i = 0; i < 6; ++i) s.take<double>(capacity + 16);
    s.take<double>(8);
    s.take<double>(8);
}

static EgkbWs egkb_ws_make(const kb_operator* op, int capacity, Arena& a) {
    EgkbWs w;
    w.plan = op_plan_make(op, a);
    w.rw = reorth_ws_make(op_len(op), capacity + 1, a);
    for (int i = 0; i < 6; ++i) w.red[i] = a.take<double>(capacity + 16);
    w.cur = a.take<double>(8);
    w.hist = a.take<double>(8);
    return w;
}

// One half step: out = normalise(reorth(y - beta*prev)) with y = B x (or B^T x).
// Returns the device pointer of the new norm (t or alpha) and of |y|^2.
struct HalfOut {
    const double* norm;
    const double* ynorm2;
};

static HalfOut half_step(const kb_operator* op, EgkbWs& w, int transpose, const void* x,
                         const void* prev, const double* beta, const void* S, int64_t ld, int m,
                         int passes, void* out, double** red, cudaStream_t st) {
    const int64_t len = transpose ? op->cols : op->rows;
    Src src = op_source(w.plan, x, transpose, st);
    src.prev = prev;
    src.beta = beta;
    HalfOut h;
    reorth_pass(op->dtype, src, S, ld, m, nullptr, nullptr, m > 0, nullptr, nullptr, len, red[0],
                w.rw, st);
    h.ynorm2 = red[0] + m + 1;
    if (m == 0) {
        h.norm = red[0] + m + 3;
        reorth_pass(op->dtype, src, S, ld, 0, nullptr, nullptr, false, out, h.norm, len, red[2], w.rw, st);
    } else if (passes >= 2) {
        reorth_pass(op->dtype, src, S, ld, m, red[0], nullptr, true, nullptr, nullptr, len, red[1],
                    w.rw, st);
        h.norm = red[1] + m + 2;
        reorth_pass(op->dtype, src, S, ld, m, red[0], red[1], false, out, h.norm, len, red[2], w.rw, st);
    } else {
        // classical GS: write the projected vector, then normalise in place
        reorth_pass(op->dtype, src, S, ld, m, red[0], nullptr, false, out, nullptr, len, red[1], w.rw, st);
        h.norm = red[1] + m + 3;
        Src self;
        self.z = static_cast<const double*>(out);
        self.mode = SRC_BUFT;
        reorth_pass(op->dtype, self, S, ld, 0, nullptr, nullptr, false, out, h.norm, len, red[2], w.rw, st);
    }
    return h;
}

static double eps_of(int dtype) { return dtype == KB_F32 ? 1.1920928955078125e-07 : 2.220446049250313e-16; }

static int egkb_capacity(const kb_egkb_config* c) {
    // Loop limit is fired_k + p + 1 with fired_k <= max(k_max, k_min), else
    // k_max + 1; the left basis may hold one more vector than iterations.
    return std::max(c->k_max, c->k_min) + c->p + 3;
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
    auto slot = [&](void* base, int64_t ld, int i) -> void* {
        return static_cast<char*>(base) + (size_t)i * ld * esz;
    };
    Arena a(wsp, ws_bytes);
    EgkbWs w = egkb_ws_make(op, cap, a);
    KB_CUDA(cudaMemsetAsync(w.plan.counters, 0, sizeof(unsigned) * w.plan.n_counters, s));
    KB_CUDA(cudaMemsetAsync(w.rw.counter, 0, sizeof(unsigned) * 64, s));
    static thread_local double* hp = nullptr;   // pinned scalar mailbox, allocated once per thread
    if (hp == nullptr) KB_CUDA(cudaMallocHost(&hp, sizeof(double) * 8));

    const double tol = cfg->break_tol >= 0 ? cfg->break_tol : std::sqrt(eps_of(op->dtype));
    const int passes = cfg->reorth_passes >= 2 ? 2 : 1;
    const int64_t M = op->rows, N = op->cols;

    // --- s1 = y0 / |y0|   (lowrank.py:207-210)
    Src sy;
    sy.z = static_cast<const double*>(y0);
    sy.mode = SRC_BUFT;
    reorth_pass(op->dtype, sy, nullptr, 0, 0, nullptr, nullptr, false, nullptr, nullptr, M, w.red[0], w.rw, s);
    scalars(s, w.red[0] + 3, w.cur + 1, w.red[0] + 3, w.hist + 0);
    reorth_pass(op->dtype, sy, nullptr, 0, 0, nullptr, nullptr, false, slot(st->s_basis, st->ld_s, 0),
                w.cur + 1, M, w.red[1], w.rw, s);
    // --- q1 = B^T s1 / alpha1   (lowrank.py:211-215)
    {
        Src src = op_source(w.plan, slot(st->s_basis, st->ld_s, 0), 1, s);
        reorth_pass(op->dtype, src, nullptr, 0, 0, nullptr, nullptr, false, nullptr, nullptr, N, w.red[3], w.rw, s);
        scalars(s, w.red[3] + 3, w.cur + 0, w.red[3] + 3, w.hist + 2);
        reorth_pass(op->dtype, src, nullptr, 0, 0, nullptr, nullptr, false, slot(st->q_basis, st->ld_q, 0),
                    w.cur + 0, N, w.red[4], w.rw, s);
    }
    KB_CUDA(cudaMemcpyAsync(hp, w.hist, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
    KB_CUDA(cudaStreamSynchronize(s));
    const double t1 = hp[0];
    if (t1 == 0.0) {
        set_error("starting vector must be nonzero");
        throw Fail{KB_EVALIDATION};
    }
    const double alpha1 = hp[2];
    if (alpha1 == 0.0) {
        set_error("operator annihilates the starting vector");
        throw Fail{KB_ENUMERICAL};
    }
    std::vector<double> alphas{alpha1}, ts{t1}, zetas{alpha1 * t1}, nus{1e308};

    int fired = -1;
    int fired_reason = 0;
    bool breakdown = false, t_break = false;
    int done = 1;
    auto limit = [&]() { return fired >= 0 ? fired + cfg->p + 1 : cfg->k_max + 1; };
    while (done < limit()) {
        KB_REQUIRE(done + 1 <= cap, "eGKB basis capacity exhausted (%d)", cap);
        // s step (lowrank.py:237-247)
        const int ms = cfg->full_reorth ? done : 0;
        HalfOut hs = half_step(op, w, 0, slot(st->q_basis, st->ld_q, done - 1),
                               slot(st->s_basis, st->ld_s, done - 1), w.cur + 0, st->s_basis, st->ld_s,
                               ms, passes, slot(st->s_basis, st->ld_s, done), &w.red[0], s);
        scalars(s, hs.norm, w.cur + 1, hs.norm, w.hist + 0, hs.ynorm2, w.hist + 1);
        // q step (lowrank.py:249-260)
        HalfOut hq = half_step(op, w, 1, slot(st->s_basis, st->ld_s, done),
                               slot(st->q_basis, st->ld_q, done - 1), w.cur + 1, st->q_basis, st->ld_q,
                               done, passes, slot(st->q_basis, st->ld_q, done), &w.red[3], s);
        scalars(s, hq.norm, w.cur + 0, hq.norm, w.hist + 2, hq.ynorm2, w.hist + 3);
        KB_CUDA(cudaMemcpyAsync(hp, w.hist, sizeof(double) * 4, cudaMemcpyDeviceToHost, s));
        KB_CUDA(cudaStreamSynchronize(s));
        const double t_new = hp[0], unorm = std::sqrt(hp[1]);
        const double a_new = hp[2], pre = std::sqrt(hp[3]);
        if (t_new <= tol * unorm) {
            breakdown = t_break = true;
            break;
        }
        if (a_new <= tol * pre) {
            breakdown = true;
            ts.push_back(t_new);
            break;
        }
        ts.push_back(t_new);
        alphas.push_back(a_new);
        const double zeta = a_new * t_new;
        const double nu = std::sqrt(zeta * zetas.back());
        zetas.push_back(zeta);
        nus.push_back(nu);
        done += 1;
        if (fired < 0) {
            const double prev = nus[nus.size() - 2];
            if (nu > prev) {
                fired = std::max(done - 1, cfg->k_min);
                fired_reason = KB_STOP_NU_ROSE;
            } else if (nu < cfg->tau) {
                fired = std::max(done, cfg->k_min);
                fired_reason = KB_STOP_NU_BELOW_TOL;
            }
        }
    }
    int k_p, rows;
    if (breakdown && t_break) { k_p = done; rows = done; }
    else if (breakdown) { k_p = done; rows = done + 1; }
    else { k_p = done - 1; rows = done; }
    int chosen, reason;
    if (fired >= 0) { chosen = std::min(fired, k_p); reason = fired_reason; }
    else if (breakdown) { chosen = k_p; reason = KB_STOP_BREAKDOWN; }
    else { chosen = std::min(cfg->k_max, k_p); reason = KB_STOP_HIT_KMAX; }
    if (chosen < 1 || k_p < 1) {
        set_error("bidiagonalization broke down before producing any factors");
        throw Fail{KB_ENUMERICAL};
    }
    KB_REQUIRE((int)alphas.size() <= cap && (int)ts.size() <= cap, "trace overflow");
    std::copy(alphas.begin(), alphas.end(), st->alphas_host);
    std::copy(ts.begin(), ts.end(), st->ts_host);
    std::copy(zetas.begin(), zetas.end(), st->zetas_host);
    std::copy(nus.begin(), nus.end(), st->nus_host);
    st->n_alphas = (int)alphas.size();
    st->n_ts = (int)ts.size();
    st->n_nus = (int)nus.size();
    st->chosen_k = chosen;
    st->k_p = k_p;
    st->rows = rows;
    st->stop_reason = reason;
    st->breakdown = breakdown ? 1 : 0;
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
    const size_t esz = dtype == KB_F32 ? 4 : 8;
    for (int j = 0; j < ncol; ++j) {
        void* col = static_cast<char*>(Q) + (size_t)j * ld * esz;
        Src src;
        src.z = static_cast<const double*>(col);
        src.mode = SRC_BUFT;
        const int m = j;
        reorth_pass(dtype, src, Q, ld, m, nullptr, nullptr, m > 0, nullptr, nullptr, len, red[0], rw, s);
        reorth_pass(dtype, src, Q, ld, m, m > 0 ? red[0] : nullptr, nullptr, true, nullptr, nullptr, len,
                    red[1], rw, s);
        const double* t = red[1] + m + 2;
        reorth_pass(dtype, src, Q, ld, m, m > 0 ? red[0] : nullptr, m > 0 ? red[1] : nullptr, false, col, t,
                    len, red[2], rw, s);
        scalars(s, t, hist + j, red[0] + m + 3, hist + ncol + j);
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

#define KB_GUARD(...)                                               \
    try {                                                           \
        __VA_ARGS__;                                                \
        return KB_OK;                                               \
    } catch (Fail f) {                                              \
        return f.code;                                              \
    } catch (...) {                                                 \
        set_error("unexpected C++ exception");                      \
        return KB_ERUNTIME;                                         \
    }

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
        cudaStream_t s = as_stream(stream);
        KB_CUDA(cudaMemsetAsync(p.counters, 0, sizeof(unsigned) * p.n_counters, s));
        Src src = op_source(p, x, transpose, s);
        src_write(op->dtype, src, y, transpose ? op->cols : op->rows, s);
    })
}

extern "C" int kb_ts_dots(int dtype, const void* S, int64_t ld, int m, const void* v, int64_t len,
                          double* out, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(v && out && (S || m == 0), "null argument");
        Arena a(ws, ws_bytes);
        ReorthWs rw = reorth_ws_make(len, m, a);
        double* red = a.take<double>(m + 8);
        cudaStream_t s = as_stream(stream);
        KB_CUDA(cudaMemsetAsync(rw.counter, 0, sizeof(unsigned) * 64, s));
        Src src;
        src.z = static_cast<const double*>(v);
        src.mode = SRC_BUFT;
        reorth_pass(dtype, src, S, ld, m, nullptr, nullptr, true, nullptr, nullptr, len, red, rw, s);
        KB_CUDA(cudaMemcpyAsync(out, red, sizeof(double) * (m + 1), cudaMemcpyDeviceToDevice, s));
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
        src.z = static_cast<const double*>(v);
        src.mode = SRC_BUFT;
        reorth_pass(dtype, src, S, ld, m, coef, nullptr, false, v, nullptr, len, red, rw,
                    as_stream(stream));
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
        *bytes = s.off;
    })
}

extern "C" int kb_egkb_run(const kb_operator* op, const kb_egkb_config* cfg, const void* y0,
                           kb_egkb_state* st, void* ws, size_t ws_bytes, kb_stream_t stream) {
    KB_GUARD(egkb_run(op, cfg, y0, st, ws, ws_bytes, as_stream(stream)))
}

extern "C" int kb_toeplitz_lift(int dtype, const void* coef, int64_t ldc, int len_coef, int center,
                                int k, int side, void* out, int64_t ld_out, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(coef && out && k >= 1 && side >= 1, "bad arguments");
        const int64_t len = (int64_t)side * side;
        const unsigned blocks = (unsigned)std::min<int64_t>(cdiv(len, 256), 8 * kSMs);
        cudaStream_t s = as_stream(stream);
        if (dtype == KB_F32)
            k_toeplitz_lift<float><<<blocks, 256, 0, s>>>(static_cast<const float*>(coef), ldc, len_coef,
                                                          center, k, side, static_cast<float*>(out), ld_out);
        else
            k_toeplitz_lift<double><<<blocks, 256, 0, s>>>(static_cast<const double*>(coef), ldc, len_coef,
                                                           center, k, side, static_cast<double*>(out), ld_out);
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
