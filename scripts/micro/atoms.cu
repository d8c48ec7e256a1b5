// microbenchmark: shared-memory integer atomic add throughput (spread addresses)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_atoms(int* out, int iters, int spread) {
    __shared__ int s[4096];
    for (int t = threadIdx.x; t < 4096; t += blockDim.x) s[t] = 0;
    __syncthreads();
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    int a0 = 0;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        const int idx = spread ? (x >> 20) & 4095 : (threadIdx.x & 31);
        atomicAdd(&s[idx], 1);
        atomicAdd(&s[(idx + 1024) & 4095], 2);
        atomicAdd(&s[(idx + 2048) & 4095], 3);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[blockIdx.x] = s[0] + a0;
}
__global__ void k_alu(int* out, int iters) {
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x;
    for (int it = 0; it < iters; ++it) { x = x * 1664525u + 1013904223u; x ^= x >> 7; x += 0x9e3779b9u; }
    if (x == 12345) out[0] = x;
}
__global__ void k_red(int* g, int iters, int n) {
    unsigned x = threadIdx.x * 2654435761u + blockIdx.x * 7919u;
    for (int it = 0; it < iters; ++it) {
        x = x * 1664525u + 1013904223u;
        atomicAdd(&g[(x >> 4) % n], 1);
    }
}
int main() {
    int* out; cudaMalloc(&out, 1 << 20);
    int* g; cudaMalloc(&g, 64 << 20);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256, iters = 4096;
    for (int spread = 0; spread < 2; ++spread) {
        k_atoms<<<blocks, threads>>>(out, 16, spread);
        cudaEventRecord(a);
        k_atoms<<<blocks, threads>>>(out, iters, spread);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        double ops = 3.0 * blocks * threads * (double)iters;
        printf("ATOMS spread=%d: %.3f ms, %.1f G lane-atomics/s, %.2f lane-atomics/clk/SM @1.9GHz\n", spread, ms,
               ops / ms / 1e6, ops / (ms * 1e-3) / 148 / 1.9e9);
    }
    cudaEventRecord(a);
    k_alu<<<blocks, threads>>>(out, iters * 4);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("ALU loop ref: %.3f ms\n", ms);
    const int n = 16 << 20;
    k_red<<<blocks, threads>>>(g, 16, n);
    cudaEventRecord(a);
    k_red<<<blocks, threads>>>(g, 1024, n);
    cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    double ops = (double)blocks * threads * 1024;
    printf("RED global spread: %.3f ms, %.1f G atomics/s\n", ms, ops / ms / 1e6);
    return 0;
}
