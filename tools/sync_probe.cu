// Grid-barrier cost on B200: cooperative-groups grid.sync() vs a sense-reversal
// barrier (one atomic per CTA, acquire/release), for 2x148 CTAs of 256 threads
// and 1x148 CTAs of 512 threads.   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o sync_probe sync_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_cg(int iters, int* sink) {
    cg::grid_group g = cg::this_grid();
    for (int i = 0; i < iters; ++i) g.sync();
    if (threadIdx.x == 0 && blockIdx.x == 0) *sink = iters;
}

__device__ __forceinline__ void bar(unsigned* count, volatile unsigned* gen, unsigned nblk) {
    __syncthreads();
    if (threadIdx.x == 0) {
        const unsigned g0 = *gen;
        __threadfence();
        const unsigned t = atomicAdd(count, 1u);
        if (t == nblk - 1) {
            *count = 0;
            __threadfence();
            atomicAdd((unsigned*)gen, 1u);
        } else {
            while (*gen == g0) {}
        }
        __threadfence();
    }
    __syncthreads();
}

__global__ void k_custom(int iters, unsigned* count, unsigned* gen) {
    for (int i = 0; i < iters; ++i) bar(count, gen, gridDim.x);
}

int main() {
    int* sink; unsigned *cnt, *gen;
    cudaMalloc(&sink, 4); cudaMalloc(&cnt, 4); cudaMalloc(&gen, 4);
    cudaMemset(cnt, 0, 4); cudaMemset(gen, 0, 4);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int iters = 2000;
    for (int cfg = 0; cfg < 2; ++cfg) {
        const int grid = cfg == 0 ? 296 : 148, threads = cfg == 0 ? 256 : 512;
        void* args[] = {(void*)&iters, (void*)&sink};
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_cg, grid, threads, args, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        float ms; cudaEventElapsedTime(&ms, a, b);
        void* args2[] = {(void*)&iters, (void*)&cnt, (void*)&gen};
        float ms2 = 0;
        for (int rep = 0; rep < 2; ++rep) {
            cudaEventRecord(a);
            cudaLaunchCooperativeKernel((void*)k_custom, grid, threads, args2, 0, 0);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
        }
        cudaEventElapsedTime(&ms2, a, b);
        printf("grid %d x %d: cg grid.sync %.3f us, custom barrier %.3f us  (%s)\n", grid, threads,
               ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
