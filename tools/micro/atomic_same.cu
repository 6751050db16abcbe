// Microbenchmark: throughput of same-address global atomics (with / without return value).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_ret(int *c, int *out, int per_warp) {
    if ((threadIdx.x & 31) == 0) {
        int v = 0;
        for (int i = 0; i < per_warp; i++) v += atomicAdd(c, 1);
        out[blockIdx.x * blockDim.x + threadIdx.x] = v;
    }
}
__global__ void k_red(int *c, int per_warp) {
    if ((threadIdx.x & 31) == 0)
        for (int i = 0; i < per_warp; i++) atomicAdd(c, 1);
}
__global__ void k_spread(int *c, int *out) {  // distinct addresses, with return
    if ((threadIdx.x & 31) == 0) {
        int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
        out[w] = atomicAdd(c + 32 * w, 1);
    }
}
int main() {
    int *c, *out;
    cudaMalloc(&c, 1 << 26);
    cudaMalloc(&out, 1 << 26);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int warps : {1024, 4096, 32768}) {
        int blocks = warps / 8;
        float ms;
        k_ret<<<blocks, 256>>>(c, out, 1);
        cudaEventRecord(a);
        k_ret<<<blocks, 256>>>(c, out, 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("same-address atomicAdd with return: %6d warps x1: %8.2f us (%.2f ns each)\n", warps, ms * 1e3, ms * 1e6 / warps);
        k_red<<<blocks, 256>>>(c, 1);
        cudaEventRecord(a);
        k_red<<<blocks, 256>>>(c, 1);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("same-address RED (no return):       %6d warps x1: %8.2f us (%.2f ns each)\n", warps, ms * 1e3, ms * 1e6 / warps);
        k_spread<<<blocks, 256>>>(c, out);
        cudaEventRecord(a);
        k_spread<<<blocks, 256>>>(c, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        printf("distinct-address atomicAdd w/ ret:  %6d warps x1: %8.2f us\n", warps, ms * 1e3);
    }
    return 0;
}
