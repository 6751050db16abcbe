// Microbenchmark: FFMA vs FFMA2 (fma.rn.f32x2) issue throughput on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
#define ITERS 32768
__device__ __forceinline__ unsigned long long f2(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__global__ void k1(float *out, float s) {
    float a[8];
    for (int i = 0; i < 8; i++) a[i] = threadIdx.x * 0.001f + i;
    for (int it = 0; it < ITERS; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = fmaf(a[i], s, 0.5f);
    float r = 0;
    for (int i = 0; i < 8; i++) r += a[i];
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
__global__ void k2(float *out, float s) {
    unsigned long long a[8];
    float2 sv = make_float2(s, s), hv = make_float2(0.5f, 0.5f);
    unsigned long long ss = *reinterpret_cast<unsigned long long *>(&sv), hh = *reinterpret_cast<unsigned long long *>(&hv);
    for (int i = 0; i < 8; i++) {
        float2 v = make_float2(threadIdx.x * 0.001f + i, i + 0.5f);
        a[i] = *reinterpret_cast<unsigned long long *>(&v);
    }
    for (int it = 0; it < ITERS; it++)
#pragma unroll
        for (int i = 0; i < 8; i++) a[i] = f2(a[i], ss, hh);
    float r = 0;
    for (int i = 0; i < 8; i++) {
        float2 v = *reinterpret_cast<float2 *>(&a[i]);
        r += v.x + v.y;
    }
    out[blockIdx.x * blockDim.x + threadIdx.x] = r;
}
int main() {
    float *o;
    cudaMalloc(&o, 1 << 26);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int blocks = 148 * 8, threads = 256;
    for (int rep = 0; rep < 10; rep++) {
        float ms;
        cudaEventRecord(a);
        k1<<<blocks, threads>>>(o, 0.999f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        double fl = 2.0 * blocks * threads * (double)ITERS * 8;
        printf("FFMA : %.3f ms, %.1f TFLOP/s\n", ms, fl / ms / 1e9);
        cudaEventRecord(a);
        k2<<<blocks, threads>>>(o, 0.999f);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        cudaEventElapsedTime(&ms, a, b);
        fl *= 2;
        printf("FFMA2: %.3f ms, %.1f TFLOP/s\n", ms, fl / ms / 1e9);
    }
    return 0;
}
