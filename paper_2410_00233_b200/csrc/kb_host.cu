// Host-side helpers of the e2e path (no device compute): the Psf validation
// scan and the staged upload of the raw PSF.
//
//   kb_psf_scan   -- blurmodel.py:25-65 (Psf.__init__): k.min() and k.sum()
//                    of the C-ordered float64 kernel, and the private copy the
//                    reference's np.array(kernel) takes, in the same pass.  The sum is numpy's
//                    pairwise summation (8 accumulators over blocks of <= 128,
//                    halving splits rounded to multiples of 8), evaluated on
//                    the top subtrees in parallel and combined in the same
//                    tree: bit-identical to k.sum(), in a fraction of the time.
//   kb_stage_upload -- host array -> device through one library-owned pinned
//                    buffer, filled by all host threads chunk by chunk while
//                    the previous chunk is on the wire (pageable copies run at
//                    ~16 GB/s; this pipeline at the link rate).
#include <omp.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "kb_common.cuh"

namespace kb {
namespace {

// numpy/_core/src/umath/loops_utils.h.src: DOUBLE_pairwise_sum (contiguous)
double pairwise_sum(const double* a, int64_t n) {
    if (n < 8) {
        double res = 0.0;
        for (int64_t i = 0; i < n; ++i) res += a[i];
        return res;
    }
    if (n <= 128) {
        double r[8];
        for (int j = 0; j < 8; ++j) r[j] = a[j];
        int64_t i = 8;
        for (; i < n - (n % 8); i += 8)
            for (int j = 0; j < 8; ++j) r[j] += a[i + j];
        double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < n; ++i) res += a[i];
        return res;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return pairwise_sum(a, n2) + pairwise_sum(a + n2, n - n2);
}

struct Leaf {
    int64_t lo, n;
};

// The top `depth` levels of numpy's split tree; leaves in order.
void split_tree(int64_t lo, int64_t n, int depth, std::vector<Leaf>& out) {
    if (depth == 0 || n <= 1024) {
        out.push_back({lo, n});
        return;
    }
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    split_tree(lo, n2, depth - 1, out);
    split_tree(lo + n2, n - n2, depth - 1, out);
}

// Recombine leaf sums with the tree's association.
double combine(int64_t n, int depth, const double* leaf_sum, int& idx) {
    if (depth == 0 || n <= 1024) return leaf_sum[idx++];
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    const double a = combine(n2, depth - 1, leaf_sum, idx);
    const double b = combine(n - n2, depth - 1, leaf_sum, idx);
    return a + b;
}

}  // namespace
}  // namespace kb

namespace kb {
namespace {

// Library-owned pinned staging for the fp32 PSF upload.  One lock serialises
// every user of the buffers (ctypes releases the GIL, so two Python threads
// can upload at once); `done` is the last copy out of buf32.
struct Stage {
    std::mutex mu;
    cudaEvent_t done = nullptr;
    float* buf32 = nullptr;
    size_t cap32 = 0;
};
Stage& stage() {
    static Stage s;
    return s;
}
std::mutex& upload_mutex() {
    static std::mutex m;
    return m;
}

void psf_scan(const double* k, int64_t n, int threads, double* sum_out, double* min_out, char* copy_to = nullptr) {
    if (n == 0) {
        *sum_out = 0.0;
        *min_out = 0.0;
        return;
    }
    const int depth = 4;   // 16 leaves
    std::vector<Leaf> leaves;
    split_tree(0, n, depth, leaves);
    std::vector<double> sums(leaves.size()), mins(leaves.size());
    const int nt = std::max(1, std::min<int>(threads, (int)leaves.size()));
#pragma omp parallel for num_threads(nt) schedule(static, 1)
    for (int i = 0; i < (int)leaves.size(); ++i) {
        const double* a = k + leaves[i].lo;
        sums[i] = pairwise_sum(a, leaves[i].n);
        if (copy_to) std::memcpy(copy_to + sizeof(double) * leaves[i].lo, a, sizeof(double) * leaves[i].n);
        double m = a[0];
        for (int64_t j = 1; j < leaves[i].n; ++j) m = std::min(m, a[j]);   // NaN: caught by the sum / > 0 tests
        mins[i] = m;
    }
    int idx = 0;
    *sum_out = combine(n, depth, sums.data(), idx);
    double m = mins[0];
    for (size_t i = 1; i < mins.size(); ++i) m = std::min(m, mins[i]);
    *min_out = m;
}

void stage_upload(const void* src, size_t bytes, void* dst, int threads, cudaStream_t s) {
    static char* stage = nullptr;
    static size_t cap = 0;
    static cudaEvent_t ev[2] = {nullptr, nullptr};
    if (!ev[0]) {
        KB_CUDA(cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming));
        KB_CUDA(cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming));
    }
    constexpr size_t CH = 1 << 20;   // pipeline chunk
    const size_t want = std::max(std::min(bytes, 2 * CH), (size_t)1 << 16);
    if (cap < want) {
        KB_CUDA(cudaEventSynchronize(ev[0]));
        KB_CUDA(cudaEventSynchronize(ev[1]));
        if (stage) cudaFreeHost(stage);
        cap = want;
        KB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&stage), cap));
    }
    // two halves of the staging buffer: one is filled while the other is on the wire
    const bool dbl = cap >= 2 * CH;
    const size_t half = dbl ? CH : cap;
    const int nt = std::max(1, threads);
    int b = 0;
    for (size_t off = 0; off < bytes; off += half, b ^= 1) {
        const size_t len = std::min(half, bytes - off);
        const int e = dbl ? b : 0;
        char* buf = stage + (dbl ? b * CH : 0);
        KB_CUDA(cudaEventSynchronize(ev[e]));   // this half's previous copy has finished
        const char* from = static_cast<const char*>(src) + off;
        const size_t per = (len + nt - 1) / nt;
#pragma omp parallel for num_threads(nt) schedule(static, 1)
        for (int t = 0; t < nt; ++t) {
            const size_t lo = (size_t)t * per;
            if (lo < len) std::memcpy(buf + lo, from + lo, std::min(per, len - lo));
        }
        KB_CUDA(cudaMemcpyAsync(static_cast<char*>(dst) + off, buf, len, cudaMemcpyHostToDevice, s));
        KB_CUDA(cudaEventRecord(ev[e], s));
    }
}

}  // namespace
}  // namespace kb

extern "C" int kb_psf_scan(const double* k, int64_t n, int threads, double* sum_out, double* min_out,
                           double* copy_to) {
    KB_GUARD({
        KB_REQUIRE(k && n >= 0 && sum_out && min_out, "bad arguments");
        kb::psf_scan(k, n, threads, sum_out, min_out, reinterpret_cast<char*>(copy_to));
    })
}

namespace kb {
namespace {
void commit_f32(Stage& st, const double* src, int64_t n, double total, float* dst, int threads, cudaStream_t s) {
    if (st.cap32 < (size_t)n) {
        if (st.buf32) cudaFreeHost(st.buf32);
        st.buf32 = nullptr;
        st.cap32 = 0;
        KB_CUDA(cudaMallocHost(reinterpret_cast<void**>(&st.buf32), sizeof(float) * (size_t)n));
        st.cap32 = (size_t)n;
    }
    float* out = st.buf32;
    // (k / total).astype(float32): IEEE fp64 division, then round to fp32 (bitwise numpy).
    // Chunked so the copy engine uploads chunk c while the threads normalise c + 1.
    static const int env_ch = std::getenv("KB_STAGE_CHUNKS") ? std::atoi(std::getenv("KB_STAGE_CHUNKS")) : 0;
    const int64_t nch = env_ch > 0 ? env_ch : (n >= (int64_t)1 << 18 ? 8 : 1);
    const int64_t csz = ((n + nch - 1) / nch + 1023) / 1024 * 1024;
    cudaError_t err = cudaSuccess;
#pragma omp parallel num_threads(std::max(1, threads))
    for (int64_t c0 = 0; c0 < n; c0 += csz) {
        const int64_t c1 = std::min(n, c0 + csz);
#pragma omp for schedule(static)
        for (int64_t i = c0; i < c1; ++i) out[i] = (float)(src[i] / total);
#pragma omp master
        {
            const cudaError_t e = cudaMemcpyAsync(dst + c0, out + c0, sizeof(float) * (size_t)(c1 - c0),
                                                  cudaMemcpyHostToDevice, s);
            if (e != cudaSuccess && err == cudaSuccess) err = e;
        }
    }
    KB_CUDA(err);
    KB_CUDA(cudaEventRecord(st.done, s));
}
}  // namespace
}  // namespace kb

extern "C" int kb_psf_commit_f32(const double* src, size_t count, double total, float* dst, int threads,
                                 kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(src && dst, "bad arguments");
        kb::Stage& st = kb::stage();
        std::lock_guard<std::mutex> lock(st.mu);
        if (!st.done) KB_CUDA(cudaEventCreateWithFlags(&st.done, cudaEventDisableTiming));
        KB_CUDA(cudaEventSynchronize(st.done));   // the previous upload out of buf32 has finished
        kb::commit_f32(st, src, (int64_t)count, total, dst, threads, kb::as_stream(stream));
    })
}

extern "C" int kb_stage_upload(const void* src, size_t bytes, void* dst, int threads, kb_stream_t stream) {
    KB_GUARD({
        KB_REQUIRE(src && dst, "bad arguments");
        std::lock_guard<std::mutex> lock(kb::upload_mutex());
        kb::stage_upload(src, bytes, dst, threads, kb::as_stream(stream));
    })
}
