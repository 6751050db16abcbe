// loss.cu -- mapping loss (R/losses.py:157-161) and its image gradients (sm_100a).
//
// Photometric term (1-lam) L1 + lam D-SSIM (R/losses.py:89-130): 11-tap Gaussian (sigma 1.5)
// with mirror (triangle-wave) padding and its exact adjoint.  Both are written as position-
// dependent 11-tap correlations: blur(x)(q) = sum_d F[q][d] x(q+d) with
// F[q][d] = sum_t K(t) [refl(q+t) == q+d], and adjoint(g)(p) = sum_d F[p+d][-d] g(p+d); the
// per-axis tables absorb every reflection, so interior and border pixels share one code path.
// Two kernels per view (below): the SSIM map and its partials, then their adjoint.
//
// Depth term (R/losses.py:133-154) is evaluated only at the view's LiDAR pixels (K-list).
#include <algorithm>

#include "common.cuh"

namespace gs {

// Two launches per view, CTA per (64 x 16 output tile, colour channel), 256 threads:
//   ssim_fwd_kernel  inputs on the tile + halo 5 (mirror-padded at the border) -> the four
//                    moments (a, b, aa + bb, ab) blurred vertically over the 74 tile columns,
//                    then horizontally -> SSIM map on the tile only -> its three partial images
//                    (d/d mu_a, d/d (var sum), d/d sigma_ab) to HBM (ssim_g, L2-resident), block
//                    sums of SSIM and |a - b|;
//   ssim_bwd_kernel  the partials on the tile + halo 5 -> vertical, then horizontal adjoint
//                    blur -> gradient of the photometric term.
// Splitting at the SSIM map removes the halo recompute of the fused form (SSIM map and first
// adjoint pass on a (TW+10) x (TH+10) region, forward moments on (TW+20) x (TH+20)): ~125
// instead of ~230 FP32 operations per pixel and channel.  Each pass is register-blocked along
// its blur axis (a thread produces a strip of 4 outputs from one sliding window of
// shared-memory reads), blur-axis-first passes run over columns so that a warp's lanes read
// consecutive words, and the second passes map lanes to rows with an odd float4 row stride
// (conflict-free LDS.128).
constexpr int TW = 64, TH = 16;
constexpr int NR = TH + 10;           // staged rows (halo 5)
constexpr int NC = TW + 10;           // staged columns (halo 5)
constexpr int VS = 4;                 // outputs per vertical strip
constexpr int HS = 4;                 // outputs per horizontal strip
constexpr int RS = NC + 1;            // row stride (float4) of the vertical-pass output (odd)
constexpr int H_THREADS = TH * (TW / HS);    // second-pass strips: one per thread
constexpr int L_THREADS = 320;               // >= the first pass's NC * TH / VS = 296 strips, so
                                             // that neither pass takes a second round (the idle
                                             // warps of a pass wait at its barrier without issuing)
static_assert(H_THREADS == 256 && TH == 16, "second pass: warps 0-7, lanes 0-15 = rows");
static_assert(NC * (TH / VS) <= L_THREADS, "first pass: one strip per thread");
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
    pdl_wait();
    // the tables depend only on (w, h): the loss finalisation stamps them valid after first use
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

// INTERIOR: the CTA's halo lies inside the image, so every blur / adjoint weight is the plain
// kernel (compile-time immediates); border CTAs read their halo mirror-padded (forward) or the
// reflection tables (adjoint).
__device__ __forceinline__ void cp_async4(void *smem, const void *gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)), "l"(gmem));
}
__device__ __forceinline__ void cp_async16_zfill(void *smem, const void *gmem, bool valid) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"((unsigned)__cvta_generic_to_shared(smem)),
                 "l"(gmem), "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// barrier over the first n threads of the CTA (the warps that run the second pass)
__device__ __forceinline__ void named_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

__device__ __forceinline__ float2 pfma(float w, float2 x, float2 acc) { return __ffma2_rn(make_float2(w, w), x, acc); }

template <bool INTERIOR>
__device__ __forceinline__ float wtab(const float *__restrict__ tab, int pos, int d) {
    return INTERIOR ? kw(d) : __ldg(tab + 22 * pos + d);
}

struct SsimFwdSmem {
    float2 in[2][NR][NC];  // (rendered, target) of the channel, halo 5: the tile and the next one
    float4 v[TH][RS];    // vertically blurred moments (a, b, aa + bb, ab)
    float red[2][L_THREADS / 32];
};

struct SsimBwdSmem {
    float4 g[NR][NC];    // SSIM partials (d/d mu_a, d/d (var sum), d/d sigma_ab, -), halo 5
    float4 v[TH][RS];    // their vertical adjoint
};

__device__ __forceinline__ bool ssim_interior(int x0, int y0, int W, int H) {
    return x0 >= 5 && x0 + TW + 5 <= W && y0 >= 5 && y0 + TH + 5 <= H;
}

// ssim_fwd inputs of one tile on [y0-5, y0+TH+5) x [x0-5, x0+TW+5) of channel c, mirror-padded
// (R/losses.py:31-42), issued as cp.async (the caller commits): warp w stages rows w, w + 10, ...,
// lane l columns l, l + 32, l + 64 (their reflected offsets computed once)
template <bool INTERIOR>
__device__ __forceinline__ void ssim_fwd_stage(float2 (*in)[NC], const float *__restrict__ color,
                                               const float *__restrict__ target, int W, int H, int x0, int y0,
                                               int c) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    constexpr int CP = (NC + 31) / 32;
    int xo[CP];
#pragma unroll
    for (int h = 0; h < CP; h++) {
        int x = x0 - 5 + lane + 32 * h;
        if (!INTERIOR) x = reflect_idx(min(x, x0 - 5 + NC - 1), W);
        xo[h] = 3 * x + c;
    }
    for (int iy = warp; iy < NR; iy += L_THREADS / 32) {
        int y = y0 - 5 + iy;
        if (!INTERIOR) y = reflect_idx(y, H);
        const float *crow = color + (int64_t)y * W * 3, *trow = target + (int64_t)y * W * 3;
#pragma unroll
        for (int h = 0; h < CP; h++) {
            const int ix = lane + 32 * h;
            if (ix < NC) {
                cp_async4(&in[iy][ix].x, crow + xo[h]);
                cp_async4(&in[iy][ix].y, trow + xo[h]);
            }
        }
    }
}

// SSIM map and partials of one staged tile; adds the tile's SSIM and |a - b| sums to s_acc, l1_acc
template <bool INTERIOR>
__device__ __forceinline__ void ssim_fwd_tile(SsimFwdSmem &sm, const float2 (*in)[NC], const gs_frame &f, int x0,
                                              int y0, int c, float &s_acc, float &l1_acc) {
    const int W = f.width, H = f.height;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    // 2) vertical blur of the moment pairs (a, b) and (a^2 + b^2, ab) -- the SSIM uses the
    //    variances only as the sum va + vb (R/losses.py:100-104) -- over all NC columns
    for (int it = tid; it < NC * (TH / VS); it += L_THREADS) {
        const int s = it / NC, col = it - s * NC, r0 = s * VS;
        float2 m01[VS], m23[VS];
#pragma unroll
        for (int k = 0; k < VS; k++) m01[k] = m23[k] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int t = 0; t < VS + 10; t++) {
            const float2 ab = in[r0 + t][col];
            const float2 q = make_float2(fmaf(ab.x, ab.x, ab.y * ab.y), ab.x * ab.y);
#pragma unroll
            for (int k = 0; k < VS; k++) {
                const int d = t - k;
                if (d >= 0 && d < 11) {
                    m01[k] = pfma(kw(d), ab, m01[k]);
                    m23[k] = pfma(kw(d), q, m23[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VS; k++) sm.v[r0 + k][col] = make_float4(m01[k].x, m01[k].y, m23[k].x, m23[k].y);
    }
    __syncthreads();
    // 3) horizontal blur -> SSIM map and its partials (R/losses.py:96-113), warps 0-7; lanes
    //    0-15: rows of strip 2w, lanes 16-31: rows of strip 2w + 1
    if (tid < H_THREADS) {
        const int oy = lane & 15, xs = HS * (2 * warp + (lane >> 4));
        float2 u01[HS], u23[HS];
    #pragma unroll
        for (int k = 0; k < HS; k++) u01[k] = u23[k] = make_float2(0.0f, 0.0f);
    #pragma unroll
        for (int t = 0; t < HS + 10; t++) {
            const float4 h = sm.v[oy][xs + t];
            const float2 h01 = make_float2(h.x, h.y), h23 = make_float2(h.z, h.w);
    #pragma unroll
            for (int k = 0; k < HS; k++) {
                const int d = t - k;
                if (d >= 0 && d < 11) {
                    u01[k] = pfma(kw(d), h01, u01[k]);
                    u23[k] = pfma(kw(d), h23, u23[k]);
                }
            }
        }
        const float inv_n = 1.0f / (3.0f * (float)W * (float)H);
        const int y = y0 + oy;
        float4 gk[HS];
    #pragma unroll
        for (int k = 0; k < HS; k++) {
            const int x = x0 + xs + k;
            const float ua = u01[k].x, ub = u01[k].y;
            const float vab = u23[k].y - ua * ub;
            const float a1 = 2.0f * ua * ub + C1, a2 = 2.0f * vab + C2;
            const float uu = ua * ua + ub * ub;
            const float b1 = uu + C1, b2 = (u23[k].x - uu) + C2;  // va + vb + C2
            // b1 >= C1, b2 ~ va + vb + C2 > 0: MUFU reciprocals (no IEEE divide sequences)
            const float rb1 = fast_rcp(b1), rb2 = fast_rcp(b2), rden = rb1 * rb2;
            const float S = (a1 * a2) * rden;
            const float g0 = ((2.0f * ub * a2 - 2.0f * a1 * ub) * rden - S * (2.0f * ua) * rb1 + S * (2.0f * ua) * rb2) * inv_n;
            const float g1 = (-S * rb2) * inv_n;
            const float g2 = (2.0f * a1 * rden) * inv_n;
            gk[k] = make_float4(g0, g1, g2, 0.0f);
            if (INTERIOR || (x < W && y < H)) {
                s_acc += S;
                const float2 ab = in[oy + 5][xs + k + 5];
                l1_acc += fabsf(ab.x - ab.y);
            }
        }
        // the partials leave through shared memory: this thread's lanes run down the rows (the
        // conflict-free layout of the blur), the stores run along them (coalesced 16-B rows)
        named_sync(1, H_THREADS);  // every horizontal window of sm.v has been read
    #pragma unroll
        for (int k = 0; k < HS; k++) sm.v[oy][xs + k] = gk[k];
        named_sync(1, H_THREADS);
        float4 *gout = reinterpret_cast<float4 *>(f.ssim_g) + (int64_t)c * H * W;
    #pragma unroll
        for (int k = 0; k < TH * TW / H_THREADS; k++) {
            const int q = tid + H_THREADS * k, ry = q / TW, rx = q - ry * TW;
            const int gy = y0 + ry, gx = x0 + rx;
            if (INTERIOR || (gx < W && gy < H)) gout[(int64_t)gy * W + gx] = sm.v[ry][rx];
        }
    }
}

template <bool INTERIOR>
__device__ __forceinline__ void ssim_bwd_tile(SsimBwdSmem &sm, const gs_frame &f, const gs_view *__restrict__ view,
                                              const float *__restrict__ tab_x, const float *__restrict__ tab_y,
                                              float lam, int depth_grads_zero) {
    const float *__restrict__ target = view->target;
    const float *__restrict__ color = f.color;
    const int W = f.width, H = f.height;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, c = blockIdx.z;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const float4 *__restrict__ gin = reinterpret_cast<const float4 *>(f.ssim_g) + (int64_t)c * H * W;
    // 1) partials on [y0-5, y0+TH+5) x [x0-5, x0+TW+5); zero outside the image (the adjoint
    //    weights of those positions are zero)
    for (int iy = warp; iy < NR; iy += L_THREADS / 32) {  // warp per row, lanes along it
        const int y = y0 - 5 + iy;
        const bool yin = INTERIOR || (y >= 0 && y < H);
        const float4 *grow = gin + (int64_t)(yin ? y : 0) * W;
#pragma unroll
        for (int h = 0; h < (NC + 31) / 32; h++) {
            const int ix = lane + 32 * h, x = x0 - 5 + ix;
            const bool in = yin && (INTERIOR || (x >= 0 && x < W));
            if (ix < NC) cp_async16_zfill(&sm.g[iy][ix], grow + (in ? x : 0), in);
        }
    }
    // this thread's rendered / target values for the gradient assembly, fetched under the staging
    const bool second = tid < H_THREADS;
    const int oy = lane & 15, xs = HS * (2 * warp + (lane >> 4));
    // the gradient assembly runs along the rows (coalesced): thread tid takes pixels
    // q = tid + H_THREADS k of the tile; their rendered / target values load under the staging
    constexpr int AQ = TH * TW / H_THREADS;
    float av[AQ], bv[AQ];
#pragma unroll
    for (int k = 0; k < AQ; k++) {
        const int q = tid + H_THREADS * k, ry = q / TW, rx = q - ry * TW;
        const int x = x0 + rx, y = y0 + ry;
        av[k] = bv[k] = 0.0f;
        if (second && (INTERIOR || (x < W && y < H))) {
            const int64_t p = (int64_t)y * W + x;
            av[k] = __ldg(color + 3 * p + c);
            bv[k] = __ldg(target + 3 * p + c);
        }
    }
    cp_async_wait_all();
    __syncthreads();
    // 2) vertical adjoint at rows [y0, y0+TH): r(p) = sum_d A[p][d] g(p+d)
    for (int it = tid; it < NC * (TH / VS); it += L_THREADS) {
        const int s = it / NC, col = it - s * NC, r0 = s * VS;
        float2 r01[VS];
        float r2[VS];
#pragma unroll
        for (int k = 0; k < VS; k++) {
            r01[k] = make_float2(0.0f, 0.0f);
            r2[k] = 0.0f;
        }
#pragma unroll
        for (int t = 0; t < VS + 10; t++) {
            const float4 g = sm.g[r0 + t][col];
            const float2 g01 = make_float2(g.x, g.y);
#pragma unroll
            for (int k = 0; k < VS; k++) {
                const int d = t - k;
                if (d >= 0 && d < 11) {
                    const int yp = min(y0 + r0 + k, H - 1);
                    const float w = wtab<INTERIOR>(tab_y + 11, yp, d);
                    r01[k] = pfma(w, g01, r01[k]);
                    r2[k] = fmaf(w, g.z, r2[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VS; k++) sm.v[r0 + k][col] = make_float4(r01[k].x, r01[k].y, r2[k], 0.0f);
    }
    __syncthreads();
    // 3) horizontal adjoint + gradient assembly (R/losses.py:115-117 and :126-130), warps 0-7
    if (!second) return;
    float2 A01[HS];
    float A2[HS];
#pragma unroll
    for (int k = 0; k < HS; k++) {
        A01[k] = make_float2(0.0f, 0.0f);
        A2[k] = 0.0f;
    }
#pragma unroll
    for (int t = 0; t < HS + 10; t++) {
        const float4 rv = sm.v[oy][xs + t];
        const float2 v01 = make_float2(rv.x, rv.y);
#pragma unroll
        for (int k = 0; k < HS; k++) {
            const int d = t - k;
            if (d >= 0 && d < 11) {
                const int xp = min(x0 + xs + k, W - 1);
                const float w = wtab<INTERIOR>(tab_x + 11, xp, d);
                A01[k] = pfma(w, v01, A01[k]);
                A2[k] = fmaf(w, rv.z, A2[k]);
            }
        }
    }
    // transpose through shared memory: every window of sm.v has been read, then each thread
    // leaves its four pixels' adjoints and the assembly picks them up along the rows
    named_sync(1, H_THREADS);
#pragma unroll
    for (int k = 0; k < HS; k++) sm.v[oy][xs + k] = make_float4(A01[k].x, A01[k].y, A2[k], 0.0f);
    named_sync(1, H_THREADS);
    const float inv_n = 1.0f / (3.0f * (float)W * (float)H);
#pragma unroll
    for (int k = 0; k < AQ; k++) {
        const int q = tid + H_THREADS * k, ry = q / TW, rx = q - ry * TW;
        const int x = x0 + rx, y = y0 + ry;
        if (INTERIOR || (x < W && y < H)) {
            const int64_t p = (int64_t)y * W + x;
            const float4 A = sm.v[ry][rx];
            const float a = av[k], b = bv[k];
            const float diff = a - b;
            const float sg = (float)((diff > 0.0f) - (diff < 0.0f));
            f.g_color[3 * p + c] = (1.0f - lam) * (sg * inv_n) + lam * (-0.5f * (A.x + 2.0f * a * A.y + b * A.z));
            // the depth/opacity gradient images start at zero (the LiDAR kernel follows; under
            // GS_LOSS_DEPTH_GRADS_ZERO they already are, and the LiDAR kernel runs alongside)
            if (c == 0 && !depth_grads_zero) {
                f.g_depth[p] = 0.0f;
                f.g_opac[p] = 0.0f;
            }
        }
    }
}

// persistent: CTA k takes tiles k, k + grid, ... (tile = channel-major, then row, then column),
// the next tile's inputs streaming in (cp.async, double buffer) while this one is computed; one
// (|a - b|, SSIM) partial per CTA, summed in a fixed order (deterministic)
__global__ void __launch_bounds__(L_THREADS, 4) ssim_fwd_kernel(gs_frame f, const gs_view *__restrict__ view) {
    pdl_wait();
    extern __shared__ float4 sf_raw[];
    SsimFwdSmem &sm = *reinterpret_cast<SsimFwdSmem *>(sf_raw);
    const int W = f.width, H = f.height;
    const int ntx = (W + TW - 1) / TW, nty = (H + TH - 1) / TH, T = 3 * ntx * nty;
    const float *__restrict__ target = view->target;
    const float *__restrict__ color = f.color;
    auto tile_xy = [&](int t, int &x0, int &y0, int &c) {
        c = t / (ntx * nty);
        const int r = t - c * ntx * nty;
        y0 = (r / ntx) * TH;
        x0 = (r - (r / ntx) * ntx) * TW;
    };
    auto stage = [&](int t, int buf) {
        int x0, y0, c;
        tile_xy(t, x0, y0, c);
        if (ssim_interior(x0, y0, W, H)) ssim_fwd_stage<true>(sm.in[buf], color, target, W, H, x0, y0, c);
        else ssim_fwd_stage<false>(sm.in[buf], color, target, W, H, x0, y0, c);
    };
    float s_acc = 0.0f, l1_acc = 0.0f;
    int t = blockIdx.x, buf = 0;
    if (t < T) stage(t, 0);
    cp_async_commit();
    for (; t < T; t += gridDim.x, buf ^= 1) {
        if (t + (int)gridDim.x < T) stage(t + gridDim.x, buf ^ 1);
        cp_async_commit();
        cp_async_wait_1();  // this tile's inputs have landed (the next tile's stay in flight)
        __syncthreads();
        int x0, y0, c;
        tile_xy(t, x0, y0, c);
        if (ssim_interior(x0, y0, W, H)) ssim_fwd_tile<true>(sm, sm.in[buf], f, x0, y0, c, s_acc, l1_acc);
        else ssim_fwd_tile<false>(sm, sm.in[buf], f, x0, y0, c, s_acc, l1_acc);
        __syncthreads();  // the input buffer and the moments are free for the tile after next
    }
    // CTA partial sums (deterministic order: warp butterfly, then fixed warp order)
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        l1_acc += __shfl_xor_sync(0xffffffffu, l1_acc, o);
        s_acc += __shfl_xor_sync(0xffffffffu, s_acc, o);
    }
    if (lane == 0) {
        sm.red[0][warp] = l1_acc;
        sm.red[1][warp] = s_acc;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l1 = 0.0, ss = 0.0;
        for (int w = 0; w < L_THREADS / 32; w++) {
            l1 += sm.red[0][w];
            ss += sm.red[1][w];
        }
        f.loss_parts[3 * blockIdx.x] = l1;
        f.loss_parts[3 * blockIdx.x + 1] = ss;
        f.loss_parts[3 * blockIdx.x + 2] = 0.0;
    }
}

#ifndef SB_MINB
#define SB_MINB 3
#endif
__global__ void __launch_bounds__(L_THREADS, SB_MINB) ssim_bwd_kernel(gs_frame f, const gs_view *__restrict__ view,
                                                                const float *__restrict__ tab_x,
                                                                const float *__restrict__ tab_y, float lam,
                                                                int depth_grads_zero) {
    pdl_wait();
    // let the LiDAR kernel launch into the SMs this grid's last wave leaves idle (it waits for
    // this grid's completion itself before it reads the partials, or before anything when the
    // g_depth / g_opac clearing below is on)
    asm volatile("griddepcontrol.launch_dependents;");
    extern __shared__ float4 sb_raw[];
    SsimBwdSmem &sm = *reinterpret_cast<SsimBwdSmem *>(sb_raw);
    if (ssim_interior(blockIdx.x * TW, blockIdx.y * TH, f.width, f.height))
        ssim_bwd_tile<true>(sm, f, view, tab_x, tab_y, lam, depth_grads_zero);
    else
        ssim_bwd_tile<false>(sm, f, view, tab_x, tab_y, lam, depth_grads_zero);
}

// depth_ratio_loss on the LiDAR K-list (R/losses.py:133-154), scaled by xi (R/losses.py:161)
// (defined below)
template <int NT>
__device__ __forceinline__ void finalize_body(const gs_frame &f, const gs_view *__restrict__ view, int64_t first,
                                              int64_t nparts, float lam, float xi, float *tab_stamp, int accumulate);

// depth_ratio_loss on the LiDAR K-list, then -- in the last block to finish, found by a ticket
// (threadfence reduction) -- the mapping loss from all block partials: no separate finalize launch
__global__ void __launch_bounds__(256) depth_loss_kernel(gs_frame f, const gs_view *__restrict__ view, float lam,
                                                         float xi, int64_t part0, float *tab_stamp, int accumulate,
                                                         int overlap) {
    // overlap (GS_LOSS_DEPTH_GRADS_ZERO): the depth term reads only the forward's images, which
    // were complete before the SSIM grid started; it waits for that grid before the partials
    if (!overlap) pdl_wait();
    __shared__ double red[3][8];
    __shared__ int s_last;
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
    // this block's share of the SSIM-kernel partials (part0 triples), one per thread: the last
    // block then sums gridDim.x triples instead of part0 + gridDim.x (one memory round trip).
    // They come from ssim_fwd, complete before the SSIM adjoint released this grid, so the
    // pre-reduction runs before the wait for the adjoint below.
    double l1 = 0.0, ss = 0.0;
    const int64_t per = (part0 + gridDim.x - 1) / gridDim.x;
    for (int64_t i = blockIdx.x * per + threadIdx.x; i < min(part0, (int64_t)(blockIdx.x + 1) * per); i += blockDim.x) {
        l1 += f.loss_parts[3 * i];
        ss += f.loss_parts[3 * i + 1];
    }
    double dsum = acc;
    for (int o = 16; o > 0; o >>= 1) {
        dsum += __shfl_xor_sync(0xffffffffu, dsum, o);
        l1 += __shfl_xor_sync(0xffffffffu, l1, o);
        ss += __shfl_xor_sync(0xffffffffu, ss, o);
    }
    if ((threadIdx.x & 31) == 0) {
        red[0][threadIdx.x >> 5] = l1;
        red[1][threadIdx.x >> 5] = ss;
        red[2][threadIdx.x >> 5] = dsum;
    }
    __syncthreads();
    if (overlap) pdl_wait();  // the adjoint grid is done before this grid completes (render_bwd follows)
    if (threadIdx.x == 0) {
        double a = 0.0, b = 0.0, d = 0.0;
        for (int w = 0; w < 8; w++) {
            a += red[0][w];
            b += red[1][w];
            d += red[2][w];
        }
        f.loss_parts[3 * (part0 + blockIdx.x)] = a;
        f.loss_parts[3 * (part0 + blockIdx.x) + 1] = b;
        f.loss_parts[3 * (part0 + blockIdx.x) + 2] = d;
        __threadfence();
        s_last = atomicAdd(&f.counters[GS_CNT_LOSS_TICKET], 1) == (int)gridDim.x - 1;
    }
    __syncthreads();
    if (s_last) {
        __threadfence();
        finalize_body<256>(f, view, part0, gridDim.x, lam, xi, tab_stamp, accumulate);
        if (threadIdx.x == 0) f.counters[GS_CNT_LOSS_TICKET] = 0;
    }
}


// mapping_loss from the block partials (R/losses.py:157-161), by NT threads: coalesced over the
// flat (nparts x 3) array, then a fixed-order shuffle tree -- deterministic
template <int NT>
__device__ __forceinline__ void finalize_body(const gs_frame &f, const gs_view *__restrict__ view, int64_t first,
                                              int64_t nparts, float lam, float xi, float *tab_stamp, int accumulate) {
    const double *parts = f.loss_parts + 3 * first;
    static_assert(NT % 3 == 1, "component bookkeeping: thread t keeps component (t + j) % 3 in acc[j]");
    __shared__ double r[3][NT / 32];
    const int64_t total = 3 * nparts;
    double acc[3] = {0.0, 0.0, 0.0};
    const int64_t stride = NT * 3;  // element e is component e % 3, and 3 NT % 3 == 0
    const int comp0 = threadIdx.x % 3;
#pragma unroll 4
    for (int64_t e = threadIdx.x; e < total; e += stride) {
        acc[0] += parts[e];
        if (e + NT < total) acc[1] += parts[e + NT];
        if (e + 2 * NT < total) acc[2] += parts[e + 2 * NT];
    }
    double comp[3];
#pragma unroll
    for (int j = 0; j < 3; j++) comp[(comp0 + j) % 3] = acc[j];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int q = 0; q < 3; q++) {
        double v = comp[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane == 0) r[q][warp] = v;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double l1 = 0.0, ss = 0.0, dd = 0.0;
        for (int k = 0; k < NT / 32; k++) {
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
        // running sum of the engine's losses; an iteration whose binning overflowed its entry
        // capacity is a no-op (rendered nothing, no gradient, no Adam step) and is re-run by the
        // engine after re-laying out the workspace, so it is not counted here
        if (accumulate && !f.counters[GS_CNT_OVERFLOW]) f.loss[4] += lc + (double)xi * ld;
        if (accumulate) {  // per-iteration ring: the host reads iteration i's loss at slot i % RING
            const long long pos = (long long)f.loss[6];
            f.loss[8 + pos % GS_LOSS_RING] = lc + (double)xi * ld;
            // the binning counters of this iteration (final here) for the host's lagged capacity
            // check, read back off the compute stream
            int32_t *snap = reinterpret_cast<int32_t *>(f.loss + 8 + GS_LOSS_RING) + 8 * (pos % GS_LOSS_RING);
            for (int q = 0; q < 8; q++) snap[q] = f.counters[q];
            f.loss[6] = (double)(pos + 1);
        }
        int *stamp = reinterpret_cast<int *>(tab_stamp);
        stamp[0] = (f.width << 16) + f.height;
        stamp[1] = ~((f.width << 16) + f.height);
    }
}

#ifndef DEPTH_BLOCKS_N
#define DEPTH_BLOCKS_N 148  // one per SM: short gather chains per thread
#endif
constexpr int DEPTH_BLOCKS = DEPTH_BLOCKS_N;

// loss_parts holds ssim blocks followed by DEPTH_BLOCKS depth partials; the F tables follow.
int64_t loss_parts_needed(int32_t width, int32_t height) {
    return 3 * (int64_t)((width + TW - 1) / TW) * ((height + TH - 1) / TH) + DEPTH_BLOCKS;
}

}  // namespace gs

extern "C" int gs_loss(const gs_frame *f, const gs_view *view, float lam, float xi, void *stream) {
    return gs_loss_ex(f, view, lam, xi, 0, stream);
}

extern "C" int gs_loss_ex(const gs_frame *f, const gs_view *view, float lam, float xi, int32_t flags, void *stream) {
    using namespace gs;
    if (flags & ~(GS_LOSS_TABLES_READY | GS_LOSS_ACCUMULATE | GS_LOSS_DEPTH_GRADS_ZERO)) {
        set_error("gs_loss_ex: unknown flags");
        return GS_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (f->width <= 0 || f->height <= 0) {
        set_error("gs_loss: empty image");
        return GS_ERR_DIMS;
    }
    const int64_t ssim_blocks = 3 * (int64_t)((f->width + TW - 1) / TW) * ((f->height + TH - 1) / TH);
    if (ssim_blocks + DEPTH_BLOCKS > f->loss_blocks) {
        set_error("gs_loss: workspace laid out for a different image size");
        return GS_ERR_WORKSPACE;
    }
    float *tab_x = reinterpret_cast<float *>(f->loss_parts + 3 * f->loss_blocks);
    float *tab_y = tab_x + 22 * f->width;
    int rc;
    if (!(flags & GS_LOSS_TABLES_READY)) {
        launch_pdl(loss_tables_kernel, (f->width + f->height + 127) / 128, 128, 0, st, tab_x, f->width, tab_y,
                   f->height);
        if ((rc = check_launch("loss_tables_kernel"))) return rc;
    }
    dim3 grid((f->width + TW - 1) / TW, (f->height + TH - 1) / TH, 3);
    const int dz = (flags & GS_LOSS_DEPTH_GRADS_ZERO) ? 1 : 0;
    const int fwd_ctas = (int)std::min<int64_t>(ssim_blocks, 4 * 148);
    launch_pdl(ssim_fwd_kernel, fwd_ctas, L_THREADS, sizeof(SsimFwdSmem), st, *f, view);
    if ((rc = check_launch("ssim_fwd_kernel"))) return rc;
    launch_pdl(ssim_bwd_kernel, grid, L_THREADS, sizeof(SsimBwdSmem), st, *f, view, tab_x, tab_y, lam, dz);
    if ((rc = check_launch("ssim_bwd_kernel"))) return rc;
    launch_pdl(depth_loss_kernel, DEPTH_BLOCKS, 256, 0, st, *f, view, lam, xi, (int64_t)fwd_ctas, tab_y + 22 * f->height,
               (flags & GS_LOSS_ACCUMULATE) ? 1 : 0, dz);
    return check_launch("depth_loss_kernel");
}

namespace gs {
void init_loss_attrs() {
    cudaFuncSetAttribute(ssim_fwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimFwdSmem));
    cudaFuncSetAttribute(ssim_fwd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(ssim_bwd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(SsimBwdSmem));
    cudaFuncSetAttribute(ssim_bwd_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace gs
