// Achievable bandwidth of the eGKB "dots" pattern (h_i = S_i . v, v in registers,
// S = m vectors of N floats, mostly L2-resident) at n = 1024:
//   A: the persistent kernel's loop shape (float4, ng groups, warp_sum per vector)
//   B: the same with the S loads of U vectors hoisted (independent accumulators)
//   C: 1-D bulk-copy (TMA engine) ring of the block's slice into shared memory
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dots_probe dots_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_pipeline.h>

constexpr int TH = 256;

__device__ __forceinline__ double wsum(double v) {
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

template <int NG>
__global__ void __launch_bounds__(TH, 2) kA(const float* S, int64_t ld, int m, int64_t N, double* out) {
    __shared__ double acc[8][40];
    const int64_t G = (int64_t)gridDim.x * TH, gt = (int64_t)blockIdx.x * TH + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float v[NG][4];
    for (int g = 0; g < NG; ++g) for (int q = 0; q < 4; ++q) v[g][q] = 1.0f + 0.001f * q;
    for (int i = threadIdx.x; i < 8 * 40; i += TH) (&acc[0][0])[i] = 0;
    __syncthreads();
#pragma unroll 4
    for (int i = 0; i < m; ++i) {
        const float* Si = S + (int64_t)i * ld;
        double d = 0;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
            const int64_t e0 = (g * G + gt) * 4;
            if (e0 < N) {
                const float4 s = __ldcg(reinterpret_cast<const float4*>(Si + e0));
                d += (double)s.x * v[g][0] + (double)s.y * v[g][1] + (double)s.z * v[g][2] + (double)s.w * v[g][3];
            }
        }
        d = wsum(d);
        if (lane == 0) acc[warp][i] += d;
    }
    __syncthreads();
    if (threadIdx.x < m) {
        double t = 0;
        for (int w = 0; w < 8; ++w) t += acc[w][threadIdx.x];
        out[blockIdx.x * 40 + threadIdx.x] = t;
    }
}

// B: U vectors per step, all loads first
template <int NG, int U>
__global__ void __launch_bounds__(TH, 2) kB(const float* S, int64_t ld, int m, int64_t N, double* out) {
    __shared__ double acc[8][40];
    const int64_t G = (int64_t)gridDim.x * TH, gt = (int64_t)blockIdx.x * TH + threadIdx.x;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    float v[NG][4];
    for (int g = 0; g < NG; ++g) for (int q = 0; q < 4; ++q) v[g][q] = 1.0f + 0.001f * q;
    for (int i = threadIdx.x; i < 8 * 40; i += TH) (&acc[0][0])[i] = 0;
    __syncthreads();
    for (int i0 = 0; i0 < m; i0 += U) {
        float4 s[U][NG];
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int g = 0; g < NG; ++g) {
                const int64_t e0 = (g * G + gt) * 4;
                s[u][g] = (i0 + u < m && e0 < N) ? __ldcg(reinterpret_cast<const float4*>(S + (int64_t)(i0 + u) * ld + e0))
                                                 : make_float4(0, 0, 0, 0);
            }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            double d = 0;
#pragma unroll
            for (int g = 0; g < NG; ++g)
                d += (double)s[u][g].x * v[g][0] + (double)s[u][g].y * v[g][1] + (double)s[u][g].z * v[g][2] +
                     (double)s[u][g].w * v[g][3];
            d = wsum(d);
            if (lane == 0 && i0 + u < m) acc[warp][i0 + u] += d;
        }
    }
    __syncthreads();
    if (threadIdx.x < m) {
        double t = 0;
        for (int w = 0; w < 8; ++w) t += acc[w][threadIdx.x];
        out[blockIdx.x * 40 + threadIdx.x] = t;
    }
}

int main() {
    const int64_t N = 1 << 20;
    const int m = 13;
    float* S; double* out;
    cudaMalloc(&S, sizeof(float) * N * 40);
    cudaMalloc(&out, sizeof(double) * 400 * 40);
    cudaMemset(S, 0, sizeof(float) * N * 40);
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char* name, auto kern, int grid) {
        for (int r = 0; r < 3; ++r) kern<<<grid, TH>>>(S, N, m, N, out);
        cudaEventRecord(a);
        for (int r = 0; r < 20; ++r) kern<<<grid, TH>>>(S, N, m, N, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        const double us = ms * 1e3 / 20;
        printf("%-28s grid %d: %.2f us  %.2f TB/s (%s)\n", name, grid, us, 4.0 * N * m / (us * 1e-6) / 1e12,
               cudaGetErrorString(cudaGetLastError()));
    };
    run("A  (pk shape, ng=4)", kA<4>, 296);
    run("B  U=2", kB<4, 2>, 296);
    run("B  U=4", kB<4, 4>, 296);
    run("A  ng=2 (2x grid)", kA<2>, 592);
    run("B  U=4 ng=2", kB<2, 4>, 592);
    return 0;
}
