// Grid barrier + fixed-order reduction of per-CTA partials (W slots), the
// pattern of every eGKB half step.  Variants, timed per iteration for
// 296 CTAs x 256 threads:
//   A  cg grid.sync, then every CTA reduces [CTA][slot] partials (lane = slot)
//   B  cg grid.sync, then every CTA reduces [slot][CTA] partials (lanes over CTAs)
//   C  last arriver reduces [CTA][slot] and publishes, others wait on a generation word
//   G  plain cg grid.sync (no reduction), for reference
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_probe red_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

constexpr int TH = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct P {
    double* part;     // [296][64] or [64][296]
    double* res;      // [64]
    unsigned* bar;    // [0] count, [32] gen
    double* out;      // sink
    int W, iters, mode;
};

// lane = slot, warps over CTAs, all loads in flight
__device__ void red_cta_slot(const double* part, int stride, int nblk, int W, double* out, double* tmp) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j0 = 0; j0 < W; j0 += 32) {
        const int j = j0 + lane;
        double s = 0.0;
        if (j < W) {
            double q[40];
#pragma unroll
            for (int k = 0; k < 40; ++k) {
                const int b = warp + 8 * k;
                q[k] = b < nblk ? __ldcg(part + (size_t)b * stride + j) : 0.0;
            }
#pragma unroll
            for (int k = 0; k < 40; ++k) s += q[k];
        }
        tmp[warp * 32 + lane] = s;
        __syncthreads();
        if (warp == 0 && j < W) {
            double t = 0.0;
#pragma unroll
            for (int w = 0; w < 8; ++w) t += tmp[w * 32 + lane];
            out[j] = t;
        }
        __syncthreads();
    }
}

// warp = slot (strided), lanes over CTAs (coalesced [slot][CTA])
__device__ void red_slot_cta(const double* part, int nblk, int W, double* out) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int j = warp; j < W; j += 8) {
        double q[10];
#pragma unroll
        for (int k = 0; k < 10; ++k) {
            const int b = lane + 32 * k;
            q[k] = b < nblk ? __ldcg(part + (size_t)j * 320 + b) : 0.0;
        }
        double s = 0.0;
#pragma unroll
        for (int k = 0; k < 10; ++k) s += q[k];
        s = warp_sum(s);
        if (lane == 0) out[j] = s;
    }
    __syncthreads();
}

__global__ void __launch_bounds__(TH, 2) k_probe(P p) {
    cg::grid_group grid = cg::this_grid();
    __shared__ double out[64];
    __shared__ double tmp[8 * 32];
    __shared__ int s_last;
    const int nblk = gridDim.x, b = blockIdx.x, tid = threadIdx.x;
    unsigned gen = 0;
    if (tid == 0) asm volatile("ld.relaxed.gpu.u32 %0, [%1];" : "=r"(gen) : "l"(p.bar + 32) : "memory");
    double acc = 0.0;
    for (int it = 0; it < p.iters; ++it) {
        // publish partials
        if (tid < p.W) {
            const double v = (double)(b + it + tid);
            if (p.mode == 1) __stcg(p.part + (size_t)tid * 320 + b, v);
            else __stcg(p.part + (size_t)b * 64 + tid, v);
        }
        if (p.mode == 0) {
            grid.sync();
            red_cta_slot(p.part, 64, nblk, p.W, out, tmp);
        } else if (p.mode == 1) {
            grid.sync();
            red_slot_cta(p.part, nblk, p.W, out);
        } else if (p.mode == 2) {
            __syncthreads();
            if (tid == 0) {
                unsigned old;
                asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(p.bar), "r"(1u) : "memory");
                s_last = (old == nblk - 1);
                ++gen;
            }
            __syncthreads();
            if (s_last) {
                red_cta_slot(p.part, 64, nblk, p.W, out, tmp);
                for (int j = tid; j < p.W; j += TH) __stcg(p.res + j, out[j]);
                __syncthreads();
                if (tid == 0) {
                    asm volatile("st.relaxed.gpu.u32 [%0], %1;" ::"l"(p.bar), "r"(0u) : "memory");
                    asm volatile("st.release.gpu.u32 [%0], %1;" ::"l"(p.bar + 32), "r"(gen) : "memory");
                }
            } else {
                if (tid == 0) {
                    unsigned g;
                    do {
                        asm volatile("ld.acquire.gpu.u32 %0, [%1];" : "=r"(g) : "l"(p.bar + 32) : "memory");
                    } while ((int)(g - gen) < 0);
                }
                __syncthreads();
                for (int j = tid; j < p.W; j += TH) out[j] = __ldcg(p.res + j);
            }
            __syncthreads();
        } else {
            grid.sync();
        }
        acc += out[it % (p.W > 0 ? p.W : 1)];
        if (p.mode != 3) grid.sync();   // protects part[] against the next iteration's writes (A/B/C alike)
    }
    if (tid == 0) p.out[b] = acc;
}

int main() {
    P p{};
    cudaMalloc(&p.part, sizeof(double) * 64 * 320);
    cudaMalloc(&p.res, sizeof(double) * 64);
    cudaMalloc(&p.bar, sizeof(unsigned) * 64);
    cudaMalloc(&p.out, sizeof(double) * 320);
    cudaMemset(p.bar, 0, sizeof(unsigned) * 64);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const char* names[] = {"A cg+redundant [cta][slot]", "B cg+redundant [slot][cta]", "C last-arriver reduce",
                           "G cg grid.sync only"};
    int Ws[] = {1, 2, 15, 35};
    for (int mode = 0; mode < 4; ++mode)
        for (int wi = 0; wi < 4; ++wi) {
            p.W = Ws[wi];
            p.mode = mode;
            float best = 1e30f;
            for (int rep = 0; rep < 3; ++rep) {
                float ms[2];
                for (int k = 0; k < 2; ++k) {
                    p.iters = k ? 400 : 100;
                    void* args[] = {&p};
                    cudaEventRecord(e0);
                    cudaLaunchCooperativeKernel((void*)k_probe, 296, TH, args, 0, 0);
                    cudaEventRecord(e1);
                    cudaEventSynchronize(e1);
                    cudaEventElapsedTime(&ms[k], e0, e1);
                }
                const float us = (ms[1] - ms[0]) * 1e3f / 300.0f;
                if (us < best) best = us;
            }
            // A/B/C include one extra grid.sync per iteration (the part[] guard)
            printf("%-28s W=%2d : %.3f us/iter\n", names[mode], p.W, best);
        }
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
