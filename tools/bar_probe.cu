// Grid barrier variants for 296 CTAs x 256 threads (2 per SM): cooperative-groups
// grid.sync vs a two-level barrier (groups of G CTAs count on their own line,
// the group's last arriver counts on a top line, the top's last arriver flips a
// generation word every CTA polls).  nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned atom_add_acqrel(unsigned* p, unsigned v) {
    unsigned old;
    asm volatile("atom.add.acq_rel.gpu.u32 %0,[%1],%2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
    return old;
}
__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
    unsigned v;
    asm volatile("ld.acquire.gpu.u32 %0,[%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned* p, unsigned v) {
    asm volatile("st.release.gpu.u32 [%0],%1;" ::"l"(p), "r"(v) : "memory");
}

// bar layout (unsigned): [0] gen, [32 * (1 + g)] group counters, [32 * 64] top counter
__device__ void bar2(unsigned* bar, unsigned& gen, int G) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const int nblk = gridDim.x, g = blockIdx.x % G, ngrp = G;
        const int gsize = (nblk - g + G - 1) / G;   // CTAs b with b % G == g
        ++gen;
        unsigned* gc = bar + 32 * (1 + g);
        const unsigned old = atom_add_acqrel(gc, 1u);
        if (old == (unsigned)gsize - 1) {
            *gc = 0;                                   // reset (next use after the release below)
            const unsigned t = atom_add_acqrel(bar + 32 * 64, 1u);
            if (t == (unsigned)ngrp - 1) {
                bar[32 * 64] = 0;
                st_release(bar, gen);
            }
        }
        while ((int)(ld_acquire(bar) - gen) < 0) {}
    }
    __syncthreads();
}

__global__ void k_cg(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}
__global__ void k_bar2(int iters, unsigned* bar, int G, int* sink) {
    unsigned gen = 0;
    if (threadIdx.x == 0) gen = ld_acquire(bar);
    for (int i = 0; i < iters; ++i) bar2(bar, gen, G);
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

int main() {
    int* sink;
    unsigned* bar;
    cudaMalloc(&sink, 4);
    cudaMalloc(&bar, 4 * 32 * 80);
    cudaMemset(bar, 0, 4 * 32 * 80);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](auto launch) {
        float best = 1e30f;
        for (int rep = 0; rep < 3; ++rep) {
            float ms[2];
            for (int k = 0; k < 2; ++k) {
                cudaEventRecord(e0);
                launch(k ? 2000 : 200);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms[k], e0, e1);
            }
            best = std::min(best, (ms[1] - ms[0]) * 1e3f / 1800.f);
        }
        return best;
    };
    for (int grid : {296, 148}) {
        const int th = grid == 296 ? 256 : 512;
        float t = timeit([&](int it) {
            void* a[] = {&it, &sink};
            cudaLaunchCooperativeKernel((void*)k_cg, grid, th, a, 0, 0);
        });
        printf("grid %d: cg grid.sync %.3f us\n", grid, t);
        for (int G : {1, 4, 8, 16, 37}) {
            float t2 = timeit([&](int it) {
                void* a[] = {&it, &bar, &G, &sink};
                cudaLaunchCooperativeKernel((void*)k_bar2, grid, th, a, 0, 0);
            });
            printf("grid %d: two-level barrier G=%2d %.3f us\n", grid, G, t2);
        }
    }
    printf("(%s)\n", cudaGetErrorString(cudaGetLastError()));
}
