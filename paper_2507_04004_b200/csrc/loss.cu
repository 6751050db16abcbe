// loss.cu -- mapping loss (R/losses.py:157-161) and its image gradients (sm_100a).
//
// Photometric term (1-lam) L1 + lam D-SSIM (R/losses.py:89-130): 11-tap Gaussian (sigma 1.5)
// with mirror (triangle-wave) padding and its exact adjoint.  Both are written as position-
// dependent 11-tap correlations: blur(x)(q) = sum_d F[q][d] x(q+d) with
// F[q][d] = sum_t K(t) [refl(q+t) == q+d], and adjoint(g)(p) = sum_d F[p+d][-d] g(p+d); the
// per-axis tables absorb every reflection, so interior and border pixels share one code path.
// One CTA computes a 32x16 output tile for all three channels: halo-10 inputs -> 5 blurred
// moments (halo 5) -> SSIM map + partials -> two adjoint passes -> gradient, all in shared
// memory (one HBM read of rendered+target, one write of the gradient).
//
// Depth term (R/losses.py:133-154) is evaluated only at the view's LiDAR pixels (K-list).
#include "common.cuh"

namespace gs {

constexpr int LW = 32, LH = 16;              // output tile
constexpr int IW = LW + 20, IH = LH + 20;    // input region (halo 10)
constexpr int BW = LW + 10, BH = LH + 10;    // blurred-moment region (halo 5)
constexpr int L_THREADS = 256;
constexpr float C1 = 0.01f * 0.01f, C2 = 0.03f * 0.03f;


__device__ __forceinline__ int reflect_idx(int j, int n) {  // R/losses.py:31-42
    if (n == 1) return 0;
    const int period = 2 * n - 2;
    int a = j < 0 ? -j : j;
    a %= period;
    return a >= n ? period - a : a;
}

// Tables per axis, 22 floats per position: F[q][d+5] (blur) then A[p][d+5] = F[p+d][5-d]
// (adjoint, zero where p+d leaves the axis).  Layout: x axis (w positions) then y axis.
__global__ void loss_tables_kernel(float *tab_x, int w, float *tab_y, int h) {
    // the tables depend only on (w, h): loss_finalize_kernel stamps them valid after first use
    const int *stamp = reinterpret_cast<const int *>(tab_y + 22 * h);
    if (stamp[0] == (w << 16) + h && stamp[1] == ~((w << 16) + h)) return;
    double K[11], s = 0.0;
    for (int i = 0; i < 11; i++) {
        double x = i - 5;
        K[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        s += K[i];
    }
    const int total = w + h;
    for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < total; idx += gridDim.x * blockDim.x) {
        const bool isx = idx < w;
        const int q = isx ? idx : idx - w;
        const int n = isx ? w : h;
        float *F = (isx ? tab_x : tab_y) + 22 * q;
        double acc[11] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
        for (int t = -5; t <= 5; t++) {
            const int r = reflect_idx(q + t, n);
            acc[r - q + 5] += K[t + 5] / s;
        }
        for (int d = 0; d < 11; d++) F[d] = (float)acc[d];
        // adjoint row of position p = q: A[p][d] = F[p+d][-d] (recomputed, no cross-thread read)
        for (int d = -5; d <= 5; d++) {
            const int qq = q + d;
            double a = 0.0;
            if (qq >= 0 && qq < n)
                for (int t = -5; t <= 5; t++)
                    if (reflect_idx(qq + t, n) == q) a += K[t + 5] / s;
            F[11 + d + 5] = (float)a;
        }
    }
}

// normalised 11-tap Gaussian (sigma 1.5), R/losses.py:22-25, as fp32 immediates
__device__ __forceinline__ float kw(int d) {
    constexpr float K[11] = {0.001028380123898387f, 0.0075987582094967365f, 0.036000773310661316f,
                             0.10936068743467331f, 0.21300554275512695f, 0.26601171493530273f,
                             0.21300554275512695f, 0.10936068743467331f, 0.036000773310661316f,
                             0.0075987582094967365f, 0.001028380123898387f};
    return K[d];
}

// INTERIOR: the CTA's whole halo lies >= 10 px inside the image, so every blur / adjoint
// weight is the plain kernel (compile-time immediates); border CTAs read the reflection tables.
struct SsimSmem {
    // region A: inputs (2 x IH x IW), later the SSIM partials (3 x BH x BW)
    // region B: horizontal moments (5 x IH x BW), later the vertical adjoint (3 x LH x BW)
    float A[2 * IH * IW];
    float B[5 * IH * BW];
    float red[2][L_THREADS / 32];
};

template <bool INTERIOR>
__device__ __forceinline__ void ssim_tile(SsimSmem &sm, const gs_frame &f, const gs_view *__restrict__ view,
                                          const float *__restrict__ tab_x, const float *__restrict__ tab_y,
                                          float lam) {
    float *smA = sm.A, *smB = sm.B;
    float(*red)[L_THREADS / 32] = sm.red;
    float(*in_a)[IW] = reinterpret_cast<float(*)[IW]>(smA);
    float(*in_b)[IW] = reinterpret_cast<float(*)[IW]>(smA + IH * IW);
    float(*g)[BH][BW] = reinterpret_cast<float(*)[BH][BW]>(smA);
    float(*hx)[IH][BW] = reinterpret_cast<float(*)[IH][BW]>(smB);
    float(*ry)[LH][BW] = reinterpret_cast<float(*)[LH][BW]>(smB);
    static_assert(3 * BH * BW <= 2 * IH * IW && 3 * LH * BW <= 5 * IH * BW, "smem aliasing");

    const float *__restrict__ target = view->target;
    const int W = f.width, H = f.height;
    const int x0 = blockIdx.x * LW, y0 = blockIdx.y * LH;
    const float inv_n = 1.0f / (3.0f * (float)W * (float)H);
    const int tid = threadIdx.x;
    float l1_acc = 0.0f, s_acc = 0.0f;
    float grad_out[2][3];
    for (int c = 0; c < 3; c++) {
        __syncthreads();
        // 1) inputs on [y0-10, y0+LH+10) x [x0-10, x0+LW+10), zero outside the image
        for (int k = tid; k < IH * IW; k += L_THREADS) {
            const int iy = k / IW, ix = k % IW;
            const int y = y0 - 10 + iy, x = x0 - 10 + ix;
            float a = 0.0f, b = 0.0f;
            if (INTERIOR || (x >= 0 && x < W && y >= 0 && y < H)) {
                const int64_t p = (int64_t)y * W + x;
                a = f.color[3 * p + c];
                b = target[3 * p + c];
            }
            in_a[iy][ix] = a;
            in_b[iy][ix] = b;
        }
        __syncthreads();
        // the two output pixels' own (a, b) are kept in registers: region A is reused below
        float av[2], bv[2];
#pragma unroll
        for (int h = 0; h < 2; h++) {
            av[h] = in_a[(tid >> 5) + 8 * h + 10][(tid & 31) + 10];
            bv[h] = in_b[(tid >> 5) + 8 * h + 10][(tid & 31) + 10];
        }
        // 2) horizontal blur of the 5 moments at columns [x0-5, x0+LW+5)
        for (int k = tid; k < IH * BW; k += L_THREADS) {
            const int iy = k / BW, bx = k % BW;
            const int x = x0 - 5 + bx;
            float m0 = 0.f, m1 = 0.f, m2 = 0.f, m3 = 0.f, m4 = 0.f;
            if (INTERIOR || (x >= 0 && x < W)) {
                const float *F = tab_x + 22 * x;
#pragma unroll
                for (int d = 0; d < 11; d++) {
                    const float wgt = INTERIOR ? kw(d) : F[d];
                    const float a = in_a[iy][bx + d], b = in_b[iy][bx + d];
                    const float wa = wgt * a, wb = wgt * b;
                    m0 += wa;
                    m1 += wb;
                    m2 += wa * a;
                    m3 += wb * b;
                    m4 += wa * b;
                }
            }
            hx[0][iy][bx] = m0;
            hx[1][iy][bx] = m1;
            hx[2][iy][bx] = m2;
            hx[3][iy][bx] = m3;
            hx[4][iy][bx] = m4;
        }
        __syncthreads();
        // 3) vertical blur -> SSIM map and its partials at [y0-5, y0+LH+5) x [x0-5, x0+LW+5)
        for (int k = tid; k < BH * BW; k += L_THREADS) {
            const int by = k / BW, bx = k % BW;
            const int y = y0 - 5 + by, x = x0 - 5 + bx;
            float g0 = 0.f, g1 = 0.f, g2 = 0.f;
            if (INTERIOR || (x >= 0 && x < W && y >= 0 && y < H)) {
                const float *F = tab_y + 22 * y;
                float ua = 0.f, ub = 0.f, uaa = 0.f, ubb = 0.f, uab = 0.f;
#pragma unroll
                for (int d = 0; d < 11; d++) {
                    const float wgt = INTERIOR ? kw(d) : F[d];
                    ua += wgt * hx[0][by + d][bx];
                    ub += wgt * hx[1][by + d][bx];
                    uaa += wgt * hx[2][by + d][bx];
                    ubb += wgt * hx[3][by + d][bx];
                    uab += wgt * hx[4][by + d][bx];
                }
                // R/losses.py:96-113
                const float va = uaa - ua * ua, vb = ubb - ub * ub, vab = uab - ua * ub;
                const float a1 = 2.0f * ua * ub + C1, a2 = 2.0f * vab + C2;
                const float b1 = ua * ua + ub * ub + C1, b2 = va + vb + C2;
                const float rden = 1.0f / (b1 * b2);
                const float S = (a1 * a2) * rden;
                g0 = ((2.0f * ub * a2 - 2.0f * a1 * ub) * rden - S * (2.0f * ua / b1) + S * (2.0f * ua / b2)) * inv_n;
                g1 = (-S / b2) * inv_n;
                g2 = (2.0f * a1 * rden) * inv_n;
                if (by >= 5 && by < 5 + LH && bx >= 5 && bx < 5 + LW) s_acc += S;
            }
            g[0][by][bx] = g0;
            g[1][by][bx] = g1;
            g[2][by][bx] = g2;
        }
        __syncthreads();
        // 4) vertical adjoint at rows [y0, y0+LH): sum_d F[p+d][-d] g(p+d)
        for (int k = tid; k < LH * BW; k += L_THREADS) {
            const int oy = k / BW, bx = k % BW;
            const int y = y0 + oy;
            float r0 = 0.f, r1 = 0.f, r2 = 0.f;
            if (INTERIOR || y < H) {
                const float *A = tab_y + 22 * y + 11;  // zero weights where y+d leaves the image
#pragma unroll
                for (int d = 0; d < 11; d++) {
                    const float wgt = INTERIOR ? kw(d) : A[d];
                    r0 += wgt * g[0][oy + d][bx];
                    r1 += wgt * g[1][oy + d][bx];
                    r2 += wgt * g[2][oy + d][bx];
                }
            }
            ry[0][oy][bx] = r0;
            ry[1][oy][bx] = r1;
            ry[2][oy][bx] = r2;
        }
        __syncthreads();
        // 5) horizontal adjoint + gradient assembly for this channel
#pragma unroll
        for (int h = 0; h < 2; h++) {
            const int ox = tid & 31, oy = (tid >> 5) + 8 * h;
            const int x = x0 + ox, y = y0 + oy;
            float gsum = 0.0f;
            if (INTERIOR || (x < W && y < H)) {
                float A0 = 0.f, A1 = 0.f, A2 = 0.f;
                const float *Aw = tab_x + 22 * x + 11;
#pragma unroll
                for (int d = 0; d < 11; d++) {
                    const float wgt = INTERIOR ? kw(d) : Aw[d];
                    A0 += wgt * ry[0][oy][ox + d];
                    A1 += wgt * ry[1][oy][ox + d];
                    A2 += wgt * ry[2][oy][ox + d];
                }
                const float a = av[h], b = bv[h];
                const float diff = a - b;
                l1_acc += fabsf(diff);
                const float sg = (float)((diff > 0.0f) - (diff < 0.0f));
                // R/losses.py:115-117 and :126-130
                gsum = (1.0f - lam) * (sg * inv_n) + lam * (-0.5f * (A0 + 2.0f * a * A1 + b * A2));
            }
            grad_out[h][c] = gsum;
        }
    }
    // write gradients (and zero the depth/opacity gradient images: the LiDAR kernel follows)
#pragma unroll
    for (int h = 0; h < 2; h++) {
        const int x = x0 + (tid & 31), y = y0 + (tid >> 5) + 8 * h;
        if (x < W && y < H) {
            const int64_t p = (int64_t)y * W + x;
            f.g_color[3 * p] = grad_out[h][0];
            f.g_color[3 * p + 1] = grad_out[h][1];
            f.g_color[3 * p + 2] = grad_out[h][2];
            f.g_depth[p] = 0.0f;
            f.g_opac[p] = 0.0f;
        }
    }
    // block partial sums (deterministic order: warp butterfly, then fixed warp order)
    for (int o = 16; o > 0; o >>= 1) {
        l1_acc += __shfl_xor_sync(0xffffffffu, l1_acc, o);
        s_acc += __shfl_xor_sync(0xffffffffu, s_acc, o);
    }
    if ((tid & 31) == 0) {
        red[0][tid >> 5] = l1_acc;
        red[1][tid >> 5] = s_acc;
    }
    __syncthreads();
    if (tid == 0) {
        double l1 = 0.0, ss = 0.0;
        for (int w = 0; w < L_THREADS / 32; w++) {
            l1 += red[0][w];
            ss += red[1][w];
        }
        const int64_t blk = (int64_t)blockIdx.y * gridDim.x + blockIdx.x;
        f.loss_parts[3 * blk] = l1;
        f.loss_parts[3 * blk + 1] = ss;
        f.loss_parts[3 * blk + 2] = 0.0;
    }
}

// one launch for every tile: interior tiles (halo >= 10 px inside the image) take the
// compile-time-weight path, border tiles the reflection-table path
__global__ void __launch_bounds__(L_THREADS) ssim_l1_kernel(gs_frame f, const gs_view *__restrict__ view,
                                                            const float *__restrict__ tab_x,
                                                            const float *__restrict__ tab_y, float lam) {
    __shared__ SsimSmem sm;
    const int x0 = blockIdx.x * LW, y0 = blockIdx.y * LH;
    if (x0 >= 10 && x0 + LW + 10 <= f.width && y0 >= 10 && y0 + LH + 10 <= f.height)
        ssim_tile<true>(sm, f, view, tab_x, tab_y, lam);
    else
        ssim_tile<false>(sm, f, view, tab_x, tab_y, lam);
}

// depth_ratio_loss on the LiDAR K-list (R/losses.py:133-154), scaled by xi (R/losses.py:161)
__global__ void __launch_bounds__(256) depth_loss_kernel(gs_frame f, const gs_view *__restrict__ view, float xi,
                                                         int64_t part0) {
    __shared__ float red[8];
    const int32_t K = view->lidar_k;
    const int32_t *idx = view->lidar_idx;
    const float *zl = view->lidar_z;
    const float inv_nv = K > 0 ? 1.0f / (float)K : 0.0f;
    float acc = 0.0f;
    for (int k = blockIdx.x * blockDim.x + threadIdx.x; k < K; k += gridDim.x * blockDim.x) {
        const int p = idx[k];
        const float D = f.depth[p], O = f.opacity[p];
        const float so = fmaxf(O, 1e-6f);
        const float r = D / so - zl[k];
        acc += fabsf(r);
        const float s = (float)((r > 0.0f) - (r < 0.0f)) * inv_nv;
        f.g_depth[p] = xi * (s / so);
        f.g_opac[p] = O >= 1e-6f ? xi * (-s * D / (so * so)) : 0.0f;
    }
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        double s = 0.0;
        for (int w = 0; w < 8; w++) s += red[w];
        f.loss_parts[3 * (part0 + blockIdx.x) + 2] = s;
        f.loss_parts[3 * (part0 + blockIdx.x)] = 0.0;
        f.loss_parts[3 * (part0 + blockIdx.x) + 1] = 0.0;
    }
}

__global__ void loss_finalize_kernel(gs_frame f, const gs_view *__restrict__ view, int64_t nparts, float lam,
                                     float xi, float *tab_stamp) {
    __shared__ double r[3][256];
    double a = 0.0, b = 0.0, c = 0.0;
    for (int64_t k = threadIdx.x; k < nparts; k += blockDim.x) {
        a += f.loss_parts[3 * k];
        b += f.loss_parts[3 * k + 1];
        c += f.loss_parts[3 * k + 2];
    }
    r[0][threadIdx.x] = a;
    r[1][threadIdx.x] = b;
    r[2][threadIdx.x] = c;
    __syncthreads();
    if (threadIdx.x == 0) {
        double l1 = 0.0, ss = 0.0, dd = 0.0;
        for (int k = 0; k < 256; k++) {
            l1 += r[0][k];
            ss += r[1][k];
            dd += r[2][k];
        }
        const double n = 3.0 * (double)f.width * (double)f.height;
        const double l1m = l1 / n;
        const double dssim = 0.5 * (1.0 - ss / n);
        const double lc = (1.0 - lam) * l1m + lam * dssim;
        const int32_t K = view->lidar_k;
        const double ld = K > 0 ? dd / (double)K : 0.0;
        f.loss[0] = lc + (double)xi * ld;
        f.loss[1] = lc;
        f.loss[2] = ld;
        f.loss[3] = dssim;
        int *stamp = reinterpret_cast<int *>(tab_stamp);
        stamp[0] = (f.width << 16) + f.height;
        stamp[1] = ~((f.width << 16) + f.height);
    }
}

constexpr int DEPTH_BLOCKS = 64;

// loss_parts holds ssim blocks followed by DEPTH_BLOCKS depth partials; the F tables follow.
int64_t loss_parts_needed(int32_t width, int32_t height) {
    return (int64_t)((width + LW - 1) / LW) * ((height + LH - 1) / LH) + DEPTH_BLOCKS;
}

}  // namespace gs

extern "C" int gs_loss(const gs_frame *f, const gs_view *view, float lam, float xi, void *stream) {
    using namespace gs;
    cudaStream_t st = (cudaStream_t)stream;
    if (f->width <= 0 || f->height <= 0) {
        set_error("gs_loss: empty image");
        return GS_ERR_DIMS;
    }
    const int64_t ssim_blocks = (int64_t)((f->width + LW - 1) / LW) * ((f->height + LH - 1) / LH);
    if (ssim_blocks + DEPTH_BLOCKS > f->loss_blocks) {
        set_error("gs_loss: workspace laid out for a different image size");
        return GS_ERR_WORKSPACE;
    }
    float *tab_x = reinterpret_cast<float *>(f->loss_parts + 3 * f->loss_blocks);
    float *tab_y = tab_x + 22 * f->width;
    loss_tables_kernel<<<(f->width + f->height + 127) / 128, 128, 0, st>>>(tab_x, f->width, tab_y, f->height);
    int rc = check_launch("loss_tables_kernel");
    if (rc) return rc;
    dim3 grid((f->width + LW - 1) / LW, (f->height + LH - 1) / LH);
    ssim_l1_kernel<<<grid, L_THREADS, 0, st>>>(*f, view, tab_x, tab_y, lam);
    if ((rc = check_launch("ssim_l1_kernel"))) return rc;
    depth_loss_kernel<<<DEPTH_BLOCKS, 256, 0, st>>>(*f, view, xi, ssim_blocks);
    if ((rc = check_launch("depth_loss_kernel"))) return rc;
    loss_finalize_kernel<<<1, 256, 0, st>>>(*f, view, ssim_blocks + DEPTH_BLOCKS, lam, xi, tab_y + 22 * f->height);
    return check_launch("loss_finalize_kernel");
}

namespace gs {
void init_loss_attrs() {
    cudaFuncSetAttribute(ssim_l1_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace gs
