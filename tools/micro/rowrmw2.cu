// Layout study for the fused chain+Adam access pattern (no arithmetic): read-modify-write of the
// parameter / m / v rows of a ~27 % touched list of 1M Gaussians (+ the 160-B fixed-point
// screen-space gradient row, zeroed), in the preprocess's warp-run order, for three layouts of
// the Adam state:
//   split   p, m, v in three arrays of 256-B rows (the current layout)
//   mv      p rows + one array of 512-B (m | v) records
//   pmv     one array of 768-B (p | m | v) records
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro/rowrmw2 tools/micro/rowrmw2.cu
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

constexpr int ROW = 64, G2D = 20;

// layout: 0 split, 1 mv, 2 pmv.  Row addresses: p + g*ps, m + g*ms, v + g*vs (floats)
__global__ void __launch_bounds__(128, 4) rmw(float *p, float *m, float *v, long ps, long ms, long vs, long long *g2d,
                                              const int *list, int nt) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const long k0 = ((long)blockIdx.x * 4 + warp) * 32;
    if (k0 >= nt) return;
    const int g = k0 + lane < nt ? list[k0 + lane] : -1;
    if (g >= 0) {
        longlong2 *r = reinterpret_cast<longlong2 *>(g2d) + (long)g * (G2D / 2);
#pragma unroll
        for (int q = 0; q < G2D / 2; q++) {
            longlong2 x = r[q];
            r[q] = make_longlong2(0 * x.x, 0 * x.y);
        }
    }
#pragma unroll 1
    for (int j0 = 0; j0 < 16; j0 += 4) {
        float4 P[4], M[4], V[4];
        long op[4], om[4], ov[4];
        int gq[4];
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int kk = lane + 32 * (j0 + q), r = kk >> 4, c4 = kk & 15;
            gq[q] = __shfl_sync(0xffffffffu, g, r);
            op[q] = (long)gq[q] * ps + 4 * c4;
            om[q] = (long)gq[q] * ms + 4 * c4;
            ov[q] = (long)gq[q] * vs + 4 * c4;
            if (gq[q] >= 0 && c4 < 15) {
                P[q] = *reinterpret_cast<const float4 *>(p + op[q]);
                M[q] = *reinterpret_cast<const float4 *>(m + om[q]);
                V[q] = *reinterpret_cast<const float4 *>(v + ov[q]);
            }
        }
#pragma unroll
        for (int q = 0; q < 4; q++) {
            const int kk = lane + 32 * (j0 + q), c4 = kk & 15;
            if (gq[q] < 0 || c4 == 15) continue;
            P[q].x += 1e-7f * M[q].x;
            M[q].y += 1e-7f * V[q].y;
            V[q].z += 1e-7f * P[q].z;
            *reinterpret_cast<float4 *>(p + op[q]) = P[q];
            *reinterpret_cast<float4 *>(m + om[q]) = M[q];
            *reinterpret_cast<float4 *>(v + ov[q]) = V[q];
        }
    }
}

int main(int argc, char **argv) {
    const int n = 1 << 20;
    const double frac = argc > 1 ? atof(argv[1]) : 0.27;
    std::mt19937 rng(7);
    std::vector<int> ids;
    for (int i = 0; i < n; i++)
        if (std::uniform_real_distribution<double>(0, 1)(rng) < frac) ids.push_back(i);
    const int nt = (int)ids.size();
    std::vector<int> runs((nt + 31) / 32);
    std::iota(runs.begin(), runs.end(), 0);
    std::shuffle(runs.begin(), runs.end(), rng);
    std::vector<int> app;
    for (int r : runs)
        for (int k = r * 32; k < std::min(nt, r * 32 + 32); k++) app.push_back(ids[k]);
    float *buf;
    long long *g2d;
    int *l_app;
    cudaMalloc(&buf, (size_t)n * ROW * 4 * 3);
    cudaMalloc(&g2d, (size_t)n * G2D * 8);
    cudaMemset(buf, 0, (size_t)n * ROW * 4 * 3);
    cudaMemset(g2d, 0, (size_t)n * G2D * 8);
    cudaMalloc(&l_app, nt * 4);
    cudaMemcpy(l_app, app.data(), nt * 4, cudaMemcpyHostToDevice);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const unsigned blocks = (nt + 127) / 128;
    const double row_bytes = 6 * 240.0 + 2 * 160.0;
    const char *names[3] = {"split (p | m | v arrays)", "mv (p rows + m|v records)", "pmv (p|m|v records)"};
    for (int layout = 0; layout < 3; layout++) {
        float *p, *m, *v;
        long ps, ms, vs;
        if (layout == 0) {
            p = buf; m = buf + (size_t)n * ROW; v = buf + 2 * (size_t)n * ROW; ps = ms = vs = ROW;
        } else if (layout == 1) {
            p = buf; m = buf + (size_t)n * ROW; v = m + ROW; ps = ROW; ms = vs = 2 * ROW;
        } else {
            p = buf; m = buf + ROW; v = buf + 2 * ROW; ps = ms = vs = 3 * ROW;
        }
        for (int rep = 0; rep < 3; rep++) rmw<<<blocks, 128>>>(p, m, v, ps, ms, vs, g2d, l_app, nt);
        const int iters = 50;
        cudaEventRecord(a);
        for (int it = 0; it < iters; it++) rmw<<<blocks, 128>>>(p, m, v, ps, ms, vs, g2d, l_app, nt);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms_;
        cudaEventElapsedTime(&ms_, a, b);
        const double us = 1e3 * ms_ / iters;
        printf("%-28s rows=%d  %.1f us  %.0f GB/s\n", names[layout], nt, us, row_bytes * nt / us * 1e-3);
    }
    printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
