// Achievable HBM rate of the fused chain+Adam kernel's access pattern, without its arithmetic:
// read-modify-write of 256-B parameter / m / v rows (+ the 80-B screen-space gradient row,
// zeroed) for a touched list of ~30 % of 1M Gaussians, in the order the preprocess appends it
// (warp-ordered runs, runs in arbitrary order), against a sorted list and a dense stream.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/rowrmw tools/micro/rowrmw.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

constexpr int ROW = 64, G2D = 12;

__global__ void __launch_bounds__(128, 4) rmw(float *p, float *m, float *v, double *g2d, const int *list, int nt) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long k0 = ((long)blockIdx.x * 4 + warp) * 32;
    if (k0 >= nt) return;
    const int g = k0 + lane < nt ? list[k0 + lane] : -1;
    if (g >= 0) {
        double2 *r = reinterpret_cast<double2 *>(g2d) + (long)g * (G2D / 2);
#pragma unroll
        for (int q = 0; q < 5; q++) {
            double2 x = r[q];
            r[q] = make_double2(0.0 * x.x, 0.0 * x.y);
        }
    }
#pragma unroll 1
    for (int j0 = 0; j0 < 16; j0 += 4) {
        float4 P[4], M[4], V[4];
        long off[4];
        int gq[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int kk = lane + 32 * (j0 + q), r = kk >> 4, c4 = kk & 15;
            gq[q] = __shfl_sync(0xffffffffu, g, r);
            off[q] = (long)gq[q] * ROW + 4 * c4;
            if (gq[q] >= 0 && c4 < 15) {
                P[q] = *reinterpret_cast<const float4 *>(p + off[q]);
                M[q] = *reinterpret_cast<const float4 *>(m + off[q]);
                V[q] = *reinterpret_cast<const float4 *>(v + off[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int kk = lane + 32 * (j0 + q), c4 = kk & 15;
            if (gq[q] < 0 || c4 == 15) continue;
            P[q].x += 1e-7f * M[q].x;
            M[q].y += 1e-7f * V[q].y;
            V[q].z += 1e-7f * P[q].z;
            *reinterpret_cast<float4 *>(p + off[q]) = P[q];
            *reinterpret_cast<float4 *>(m + off[q]) = M[q];
            *reinterpret_cast<float4 *>(v + off[q]) = V[q];
        }
    }
}

__global__ void dense(float4 *p, float4 *m, float4 *v, long n4) {
    for (long i = (long)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += (long)gridDim.x * blockDim.x) {
        float4 a = p[i], b = m[i], c = v[i];
        a.x += 1e-7f * b.x;
        b.y += 1e-7f * c.y;
        c.z += 1e-7f * a.z;
        p[i] = a;
        m[i] = b;
        v[i] = c;
    }
}

int main(int argc, char **argv) {
    const int n = 1 << 20;
    const double frac = argc > 1 ? atof(argv[1]) : 0.29;
    std::mt19937 rng(7);
    std::vector<int> ids;
    for (int i = 0; i < n; i++)
        if (std::uniform_real_distribution<double>(0, 1)(rng) < frac) ids.push_back(i);
    const int nt = (int)ids.size();
    // warp-append order: runs of 32 consecutive ids, runs shuffled
    std::vector<int> runs((nt + 31) / 32);
    std::iota(runs.begin(), runs.end(), 0);
    std::shuffle(runs.begin(), runs.end(), rng);
    std::vector<int> app;
    for (int r : runs)
        for (int k = r * 32; k < std::min(nt, r * 32 + 32); k++) app.push_back(ids[k]);
    float *p, *m, *v;
    double *g2d;
    int *l_sorted, *l_app;
    cudaMalloc(&p, (size_t)n * ROW * 4);
    cudaMalloc(&m, (size_t)n * ROW * 4);
    cudaMalloc(&v, (size_t)n * ROW * 4);
    cudaMalloc(&g2d, (size_t)n * G2D * 8);
    cudaMemset(p, 0, (size_t)n * ROW * 4);
    cudaMemset(m, 0, (size_t)n * ROW * 4);
    cudaMemset(v, 0, (size_t)n * ROW * 4);
    cudaMemset(g2d, 0, (size_t)n * G2D * 8);
    cudaMalloc(&l_sorted, nt * 4);
    cudaMalloc(&l_app, nt * 4);
    cudaMemcpy(l_sorted, ids.data(), nt * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(l_app, app.data(), nt * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned blocks = (nt + 127) / 128;
    // bytes moved per row: 3 x 240 read + 3 x 240 written + 80 read + 80 written
    const double row_bytes = 6 * 240.0 + 160.0;
    for (int variant = 0; variant < 3; variant++) {
        for (int rep = 0; rep < 3; rep++) {
            if (variant == 2) dense<<<148 * 8, 256>>>((float4 *)p, (float4 *)m, (float4 *)v, (long)nt * ROW / 4);
            else rmw<<<blocks, 128>>>(p, m, v, g2d, variant ? l_sorted : l_app, nt);
        }
        const int iters = 50;
        cudaEventRecord(a);
        for (int it = 0; it < iters; it++) {
            if (variant == 2) dense<<<148 * 8, 256>>>((float4 *)p, (float4 *)m, (float4 *)v, (long)nt * ROW / 4);
            else rmw<<<blocks, 128>>>(p, m, v, g2d, variant ? l_sorted : l_app, nt);
        }
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms;
        cudaEventElapsedTime(&ms, a, b);
        const double us = 1e3 * ms / iters;
        const double bytes = variant == 2 ? 6.0 * 256 * nt : row_bytes * nt;
        printf("%s rows=%d  %.1f us  %.0f GB/s\n",
               variant == 0 ? "rmw append-order" : variant == 1 ? "rmw sorted      " : "dense same bytes", nt, us,
               bytes / us * 1e-3);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
