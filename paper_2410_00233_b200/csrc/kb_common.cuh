// Shared helpers for the kronblur_b200 sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>

#include "../../include/kronblur_b200.h"

namespace kb {

constexpr int kSMs = 148;  // B200: 2 dies x 74 SMs

void set_error(const char* fmt, ...);

struct Fail {
    int code;
};

#define KB_CUDA(expr)                                                              \
    do {                                                                           \
        cudaError_t _e = (expr);                                                   \
        if (_e != cudaSuccess) {                                                   \
            ::kb::set_error("%s failed: %s (%s:%d)", #expr, cudaGetErrorString(_e), \
                            __FILE__, __LINE__);                                   \
            throw ::kb::Fail{KB_ERUNTIME};                                         \
        }                                                                          \
    } while (0)

#define KB_REQUIRE(cond, ...)            \
    do {                                 \
        if (!(cond)) {                   \
            ::kb::set_error(__VA_ARGS__); \
            throw ::kb::Fail{KB_EVALIDATION}; \
        }                                \
    } while (0)

#define KB_LAUNCH_CHECK() KB_CUDA(cudaGetLastError())

// Body wrapper of every C-ABI entry point: C++ failures -> status codes.
#define KB_GUARD(...)                                  \
    try {                                              \
        __VA_ARGS__;                                   \
        return KB_OK;                                  \
    } catch (::kb::Fail f) {                           \
        return f.code;                                 \
    } catch (...) {                                    \
        ::kb::set_error("unexpected C++ exception");   \
        return KB_ERUNTIME;                            \
    }

inline cudaStream_t as_stream(kb_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

// Bump allocator over a caller-provided workspace.
struct Arena {
    char* base;
    size_t cap;
    size_t off = 0;
    Arena(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <typename T>
    T* take(size_t count) {
        size_t need = align_up(count * sizeof(T));
        if (base == nullptr || off + need > cap) {
            set_error("workspace too small: need %zu more bytes at offset %zu (capacity %zu)", need,
                      off, cap);
            throw Fail{KB_EVALIDATION};
        }
        T* p = reinterpret_cast<T*>(base + off);
        off += need;
        return p;
    }
};

// Byte counter mirroring Arena::take for workspace-size queries.
struct Sizer {
    size_t off = 0;
    template <typename T>
    T* take(size_t count) {   // same signature as Arena::take (returns no memory)
        off += align_up(count * sizeof(T));
        return nullptr;
    }
};

// Masked GEMM work for batched solves: blocks whose problem is inactive exit.
// rows > 0: problems stacked along M (problem = row / rows); rows == 0: the
// problem is the batch index.  flags[p * stride] != 0 means active.
// band (optional, nseg == 1 only): device int[2] (lo, hi) such that the
// untransposed B operand's row r, column c can be nonzero only when
// lo <= c - r <= hi (kb_kron_band); k tiles outside a CTA's column band are
// all-zero products and are skipped (adding exact zeros never changes a sum,
// so for finite A the result is bit-identical to the dense product).
struct GemmSkip {
    const int* flags = nullptr;
    int stride = 0;
    int rows = 0;
    const int* band = nullptr;     // zero band (col - row) of the stored B blocks: k-tile window from the column tile
    const int* band_a = nullptr;   // zero band (col - row) of the stored A blocks: k-tile window from the row tile
};

// ---------------------------------------------------------------- profiling
// Optional per-kernel-class device timing (CUDA events on the launching
// stream), used by bench.py for the live roofline numbers.  Off by default.
enum ProfClass { PROF_REORTH = 0, PROF_RA_DIAG, PROF_RA_COLSUM, PROF_DGEMM, PROF_SBVEC, PROF_LIFT,
                 PROF_RNG, PROF_NCLASS };
extern bool g_prof;
void prof_record(cudaStream_t st, int cls, double bytes, double flops, bool start);
struct ProfScope {
    cudaStream_t st; int cls; double bytes, flops; bool on;
    ProfScope(cudaStream_t s, int c, double b, double f = 0.0) : st(s), cls(c), bytes(b), flops(f), on(g_prof) {
        if (on) prof_record(st, cls, bytes, flops, true);
    }
    ~ProfScope() { if (on) prof_record(st, cls, bytes, flops, false); }
};

// ---------------------------------------------------------------- device side
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum (blockDim.x multiple of 32, <= 1024); result valid in all threads.
__device__ __forceinline__ double block_sum(double v, double* smem32) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) smem32[warp] = v;
    __syncthreads();
    const int nw = blockDim.x >> 5;
    double t = (threadIdx.x < nw) ? smem32[threadIdx.x] : 0.0;
    if (warp == 0) t = warp_sum(t);
    if (threadIdx.x == 0) smem32[0] = t;
    __syncthreads();
    double r = smem32[0];
    __syncthreads();
    return r;
}

// "Last block" ticket: every block calls after publishing its partials.
// Returns true in exactly one block (the last to arrive), which then reduces
// all partials in a fixed order -> deterministic.  The counter self-resets.
__device__ __forceinline__ bool last_block_ticket(unsigned int* counter, unsigned int nblocks) {
    __shared__ bool s_last;
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned int t = atomicAdd(counter, 1u);
        s_last = (t == nblocks - 1);
        if (s_last) *counter = 0u;
    }
    __syncthreads();
    bool last = s_last;
    if (last) __threadfence();
    return last;
}

}  // namespace kb
