// Microbenchmark: FFMA vs FFMA2 throughput and shared-memory float atomics on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ffma(float* out, float a, float b, int iters) {
    float x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = fmaf(x0, a, b); x1 = fmaf(x1, a, b); x2 = fmaf(x2, a, b); x3 = fmaf(x3, a, b);
            x4 = fmaf(x4, a, b); x5 = fmaf(x5, a, b); x6 = fmaf(x6, a, b); x7 = fmaf(x7, a, b);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}
__global__ void k_ffma2(float* out, float a, float b, int iters) {
    float2 x0 = make_float2(threadIdx.x, 1), x1 = make_float2(2, 3), x2 = make_float2(4, 5), x3 = make_float2(6, 7);
    float2 A = make_float2(a, a), B = make_float2(b, b);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) {
            x0 = __ffma2_rn(x0, A, B); x1 = __ffma2_rn(x1, A, B); x2 = __ffma2_rn(x2, A, B); x3 = __ffma2_rn(x3, A, B);
        }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0.x + x0.y + x1.x + x1.y + x2.x + x2.y + x3.x + x3.y;
}
__global__ void k_dfma(double* out, double a, double b, int iters) {
    double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int j = 0; j < 16; ++j) { x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b); }
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3;
}
__global__ void k_red4(float4* g, int n_nodes, int iters) {
    unsigned h = blockIdx.x * 7919u + threadIdx.x * 104729u;
    for (int i = 0; i < iters; ++i) {
        h = h * 1664525u + 1013904223u;
        atomicAdd(g + (h % n_nodes), make_float4(1.f, 1.f, 1.f, 1.f));
    }
}
int main() {
    float* o; cudaMalloc(&o, 148 * 64 * 1024 * sizeof(double));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    int blocks = 148 * 8, threads = 256, iters = 4096;
    k_ffma<<<blocks, threads>>>(o, 0.999f, 0.001f, 16);
    cudaEventRecord(e0); k_ffma<<<blocks, threads>>>(o, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * blocks * threads * (double)iters * 16 * 8;
    printf("FFMA : %.1f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    k_ffma2<<<blocks, threads>>>(o, 0.999f, 0.001f, 16);
    cudaEventRecord(e0); k_ffma2<<<blocks, threads>>>(o, 0.999f, 0.001f, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("FFMA2: %.1f TFLOP/s (%.3f ms)\n", flops / ms / 1e9, ms);
    k_dfma<<<blocks, threads>>>((double*)o, 0.999, 0.001, 16);
    cudaEventRecord(e0); k_dfma<<<blocks, threads>>>((double*)o, 0.999, 0.001, iters); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("DFMA : %.1f TFLOP/s (%.3f ms)\n", 2.0 * blocks * threads * (double)iters * 16 * 4 / ms / 1e9, ms);
    float4* g; int nn = 64 << 20; cudaMalloc(&g, sizeof(float4) * nn); cudaMemset(g, 0, sizeof(float4) * nn);
    for (int nodes : {1 << 16, 1 << 20, 1 << 24, 64 << 20}) {
        k_red4<<<blocks, threads>>>(g, nodes, 16);
        cudaEventRecord(e0); k_red4<<<blocks, threads>>>(g, nodes, 256); cudaEventRecord(e1); cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("red.v4.f32 random over %d nodes: %.2f G ops/s\n", nodes, (double)blocks * threads * 256 / ms / 1e6);
    }
    printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
