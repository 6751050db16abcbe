// loss.cu -- mapping loss (R/losses.py:157-161) and its image gradients (sm_100a).
//
// Photometric term (1-lam) L1 + lam D-SSIM (R/losses.py:89-130): 11-tap Gaussian (sigma 1.5)
// with mirror (triangle-wave) padding and its exact adjoint.  Both are written as position-
// dependent 11-tap correlations: blur(x)(q) = sum_d F[q][d] x(q+d) with
// F[q][d] = sum_t K(t) [refl(q+t) == q+d], and adjoint(g)(p) = sum_d F[p+d][-d] g(p+d); the
// per-axis tables absorb every reflection, so interior and border pixels share one code path.
// One CTA computes a 32x16 output tile of one channel: halo-10 inputs -> 4 blurred moments (a, b, aa + bb, ab)
// (halo 5) -> SSIM map + partials -> two adjoint passes -> gradient, all in shared memory (one
// HBM read of rendered+target, one write of the gradient).
//
// Depth term (R/losses.py:133-154) is evaluated only at the view's LiDAR pixels (K-list).
#include "common.cuh"

namespace gs {

// One CTA per (32 x 16 output tile, colour channel).  Every pass is register-blocked along its
// blur axis (a thread produces a strip of outputs from one sliding window of shared-memory
// reads); row strides are odd so that a warp reading one column per lane (or one row per lane)
// hits 32 distinct banks.  40 KB of shared memory and <= 64 registers give 4 CTAs (32 warps)
// per SM: the passes are separated by barriers, so it is the other CTAs that keep the SM busy.
constexpr int TW = 32, TH = 16;
constexpr int NIR = TH + 20;          // input rows (halo 10)
constexpr int HXC = TW + 10;          // horizontal-moment columns (strips of 6 / 3)
constexpr int HXS = HXC + 1;          // their row stride (odd)
constexpr int NIC = HXC + 12;         // input row stride in float2 (even: 16-B aligned rows for pairwise
                                      // LDS.128; >= HXC + 10); columns >= TW + 20 are never read
constexpr int GR = TH + 10;           // SSIM-map rows (halo 5)
constexpr int GW = TW + 10;           // SSIM-map columns
constexpr int GC = GW + 1;            // SSIM-map / vertical-adjoint row stride (odd)
constexpr int HS = 2;                 // horizontal adjoint: strips of 2 columns, one per thread
constexpr int L_THREADS = 256;
static_assert(TH * (TW / HS) == L_THREADS, "one horizontal-adjoint strip per thread");
static_assert(HXC % 6 == 0 && HXC % 3 == 0, "horizontal strips");
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

// Item it of `groups` groups of `len` (>= 32) elements, in warp-aligned order: the first 32
// elements of every group (one warp each), then the remaining len - 32 of every group.
__device__ __forceinline__ void split32(int it, int groups, int len, int &group, int &elem) {
    if (it < 32 * groups) {
        group = it >> 5;
        elem = it & 31;
    } else {
        const int j = it - 32 * groups, rest = len - 32;
        group = j / rest;
        elem = 32 + j % rest;
    }
}

// INTERIOR: the CTA's whole halo lies >= 10 px inside the image, so every blur / adjoint
// weight is the plain kernel (compile-time immediates); border CTAs read the reflection tables.
// The moments travel in pairs -- (a, b) and (a^2 + b^2, ab) through the blurs, (dS/dua, dS/dsig)
// through the adjoint -- so every tap of every pass is one paired FMA (sm_100 FFMA2) per pair.
struct SsimSmem {
    union {
        float2 in[NIR][NIC];  // (rendered, target) of the channel
        float4 g[GR][GC];     // SSIM partials (d/d mu_a, d/d (var sum), d/d sigma_ab, -)
    } u1;
    union {
        float4 hx[NIR][HXS];  // horizontal moments (a, b, aa + bb, ab)
        float4 ry[TH][GC];    // vertical adjoint of the three partial images
    } u2;
    float red[2][L_THREADS / 32];
};

__device__ __forceinline__ float2 pfma(float w, float2 x, float2 acc) { return __ffma2_rn(make_float2(w, w), x, acc); }

template <bool INTERIOR>
__device__ __forceinline__ float wtab(const float *__restrict__ tab, int pos, int d) {
    return INTERIOR ? kw(d) : __ldg(tab + 22 * pos + d);
}

template <bool INTERIOR>
__device__ __forceinline__ void ssim_tile(SsimSmem &sm, const gs_frame &f, const gs_view *__restrict__ view,
                                          const float *__restrict__ tab_x, const float *__restrict__ tab_y,
                                          float lam, int depth_grads_zero) {
    const float *__restrict__ target = view->target;
    const float *__restrict__ color = f.color;
    const int W = f.width, H = f.height;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH, c = blockIdx.z;
    const float inv_n = 1.0f / (3.0f * (float)W * (float)H);
    const int tid = threadIdx.x;
    // The forward blurs of every tile are plain 11-tap convolutions (compile-time weights): a
    // border tile loads its halo mirror-padded (R/losses.py:31-42, triangle wave), which is what
    // the reflection of the blur amounts to.  Only the adjoint passes of border tiles need the
    // per-position tables (the reflection folds several taps onto one pixel).
    constexpr int HB = 6;
    constexpr int VS = 5, NVS = (GR + VS - 1) / VS;
    constexpr int AS = 4, NAS = TH / AS;
    // 1) inputs on [y0-10, y0+TH+10) x [x0-10, x0+TW+10) of channel c, mirror-padded: warp w
    //    stages rows w, w + 8, ... (the TW + 20 = 52 columns in two lane passes), every load in
    //    flight before the first store, no index division (columns >= TW + 20 are never read)
    {
        constexpr int NW = L_THREADS / 32, RPW = (NIR + NW - 1) / NW, CP = (TW + 20 + 31) / 32;
        const int warp = tid >> 5, lane = tid & 31;
        float va[RPW][CP], vb[RPW][CP];
#pragma unroll
        for (int j = 0; j < RPW; j++) {
            const int iy = warp + NW * j;
            int y = y0 - 10 + iy;
            if (!INTERIOR) y = reflect_idx(min(y, y0 - 10 + NIR - 1), H);
#pragma unroll
            for (int h = 0; h < CP; h++) {
                const int ix = lane + 32 * h;
                int x = x0 - 10 + ix;
                if (!INTERIOR) x = reflect_idx(x, W);
                va[j][h] = vb[j][h] = 0.0f;
                if (iy < NIR && ix < TW + 20) {
                    const int64_t p = (int64_t)y * W + x;
                    va[j][h] = __ldg(color + 3 * p + c);
                    vb[j][h] = __ldg(target + 3 * p + c);
                }
            }
        }
#pragma unroll
        for (int j = 0; j < RPW; j++) {
            const int iy = warp + NW * j;
#pragma unroll
            for (int h = 0; h < CP; h++) {
                const int ix = lane + 32 * h;
                if (iy < NIR && ix < TW + 20) sm.u1.in[iy][ix] = make_float2(va[j][h], vb[j][h]);
            }
        }
    }
    __syncthreads();
    // 2) horizontal blur of the 4 moments (a, b, aa + bb, ab) -- SSIM uses the variances only as
    //    the sum va + vb (R/losses.py:100-104), so blur(aa) + blur(bb) is one blur; hx column j
    //    <-> x = x0-5+j
    for (int it = tid; it < NIR * (HXC / HB); it += L_THREADS) {
        // warp-aligned items: rows 0..31 of a strip per warp, then the last NIR - 32 rows of every
        // strip (odd row stride: a warp's 32 rows hit distinct banks)
        int iy, c0;
        split32(it, HXC / HB, NIR, c0, iy);
        c0 *= HB;
        float2 m01[HB], m23[HB];
#pragma unroll
        for (int k = 0; k < HB; k++) m01[k] = m23[k] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int t2 = 0; t2 < (HB + 10) / 2; t2++) {  // two input columns per 16-B load
            const float4 in2 = *reinterpret_cast<const float4 *>(&sm.u1.in[iy][c0 + 2 * t2]);
#pragma unroll
            for (int h = 0; h < 2; h++) {
                const int t = 2 * t2 + h;
                const float2 ab = h ? make_float2(in2.z, in2.w) : make_float2(in2.x, in2.y);
                const float2 q = make_float2(fmaf(ab.x, ab.x, ab.y * ab.y), ab.x * ab.y);
#pragma unroll
                for (int k = 0; k < HB; k++) {
                    const int d = t - k;
                    if (d >= 0 && d < 11) {
                        m01[k] = pfma(kw(d), ab, m01[k]);
                        m23[k] = pfma(kw(d), q, m23[k]);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < HB; k++) sm.u2.hx[iy][c0 + k] = make_float4(m01[k].x, m01[k].y, m23[k].x, m23[k].y);
    }
    __syncthreads();
    // 3) vertical blur -> SSIM map and its partials (R/losses.py:96-113); g row gy <-> y0-5+gy
    float s_acc = 0.0f;
    float2 g01v[VS];
    float g2v[VS];
    for (int it = tid; it < GW * NVS; it += L_THREADS) {
        int gx, gy0;  // warp-aligned items: 32 consecutive columns of one strip per warp
        split32(it, NVS, GW, gy0, gx);
        gy0 *= VS;
        const int x = x0 - 5 + gx;
        float2 u01[VS], u23[VS];
#pragma unroll
        for (int k = 0; k < VS; k++) u01[k] = u23[k] = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int r = 0; r < VS + 10; r++) {
            if (gy0 + r < NIR) {
                const float4 h = sm.u2.hx[gy0 + r][gx];
                const float2 h01 = make_float2(h.x, h.y), h23 = make_float2(h.z, h.w);
#pragma unroll
                for (int k = 0; k < VS; k++) {
                    const int d = r - k;
                    if (d >= 0 && d < 11) {
                        u01[k] = pfma(kw(d), h01, u01[k]);
                        u23[k] = pfma(kw(d), h23, u23[k]);
                    }
                }
            }
        }
#pragma unroll
        for (int k = 0; k < VS; k++) {
            const int gy = gy0 + k, y = y0 - 5 + gy;
            float g0 = 0.f, g1 = 0.f, g2 = 0.f;
            if (gy < GR && (INTERIOR || (x >= 0 && x < W && y >= 0 && y < H))) {
                const float ua = u01[k].x, ub = u01[k].y;
                const float vab = u23[k].y - ua * ub;
                const float a1 = 2.0f * ua * ub + C1, a2 = 2.0f * vab + C2;
                const float uu = ua * ua + ub * ub;
                const float b1 = uu + C1, b2 = (u23[k].x - uu) + C2;  // va + vb + C2
                // b1 >= C1, b2 ~ va + vb + C2 > 0: MUFU reciprocals (no IEEE divide sequences)
                const float rb1 = fast_rcp(b1), rb2 = fast_rcp(b2), rden = rb1 * rb2;
                const float S = (a1 * a2) * rden;
                g0 = ((2.0f * ub * a2 - 2.0f * a1 * ub) * rden - S * (2.0f * ua) * rb1 + S * (2.0f * ua) * rb2) * inv_n;
                g1 = (-S * rb2) * inv_n;
                g2 = (2.0f * a1 * rden) * inv_n;
                if (gy >= 5 && gy < 5 + TH && gx >= 5 && gx < 5 + TW) s_acc += S;
            }
            g01v[k] = make_float2(g0, g1);
            g2v[k] = g2;
        }
#pragma unroll
        for (int k = 0; k < VS; k++)
            if (gy0 + k < GR) sm.u1.g[gy0 + k][gx] = make_float4(g01v[k].x, g01v[k].y, g2v[k], 0.0f);
    }
    __syncthreads();
    // 4) vertical adjoint at rows [y0, y0+TH): r(p) = sum_d A[p][d] g(p+d) (zero weights where
    //    p+d leaves the image)
    for (int it = tid; it < GW * NAS; it += L_THREADS) {
        int gx, oy0;
        split32(it, NAS, GW, oy0, gx);
        oy0 *= AS;
        float2 r01[AS];
        float r2[AS];
#pragma unroll
        for (int k = 0; k < AS; k++) {
            r01[k] = make_float2(0.0f, 0.0f);
            r2[k] = 0.0f;
        }
#pragma unroll
        for (int r = 0; r < AS + 10; r++) {
            const float4 hg = sm.u1.g[oy0 + r][gx];
            const float2 h01 = make_float2(hg.x, hg.y);
            const float h2 = hg.z;
#pragma unroll
            for (int k = 0; k < AS; k++) {
                const int d = r - k;
                if (d >= 0 && d < 11) {
                    const int yp = min(y0 + oy0 + k, H - 1);
                    const float w = wtab<INTERIOR>(tab_y + 11, yp, d);
                    r01[k] = pfma(w, h01, r01[k]);
                    r2[k] = fmaf(w, h2, r2[k]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < AS; k++) {
            const bool ok = INTERIOR || y0 + oy0 + k < H;
            sm.u2.ry[oy0 + k][gx] = ok ? make_float4(r01[k].x, r01[k].y, r2[k], 0.0f) : make_float4(0.f, 0.f, 0.f, 0.f);
        }
    }
    __syncthreads();
    // 5) horizontal adjoint + gradient assembly (R/losses.py:115-117 and :126-130); a warp
    //    covers 16 rows x 2 strips
    float l1_acc = 0.0f;
    {
        // lanes 0-15: strip w, lanes 16-31: strip w + 8
        const int oy = tid & 15, ox0 = HS * ((tid >> 5) + 8 * ((tid >> 4) & 1));
        float2 A01[HS];
        float A2[HS];
#pragma unroll
        for (int k = 0; k < HS; k++) {
            A01[k] = make_float2(0.0f, 0.0f);
            A2[k] = 0.0f;
        }
#pragma unroll
        for (int t = 0; t < HS + 10; t++) {
            const float4 rv = sm.u2.ry[oy][ox0 + t];
            const float2 v01 = make_float2(rv.x, rv.y);
            const float v2 = rv.z;
#pragma unroll
            for (int k = 0; k < HS; k++) {
                const int d = t - k;
                if (d >= 0 && d < 11) {
                    const int xp = min(x0 + ox0 + k, W - 1);
                    const float w = wtab<INTERIOR>(tab_x + 11, xp, d);
                    A01[k] = pfma(w, v01, A01[k]);
                    A2[k] = fmaf(w, v2, A2[k]);
                }
            }
        }
        const int y = y0 + oy;
#pragma unroll
        for (int k = 0; k < HS; k++) {
            const int x = x0 + ox0 + k;
            if (INTERIOR || (x < W && y < H)) {
                const int64_t p = (int64_t)y * W + x;
                const float a = __ldg(color + 3 * p + c), b = __ldg(target + 3 * p + c);
                const float diff = a - b;
                l1_acc += fabsf(diff);
                const float sg = (float)((diff > 0.0f) - (diff < 0.0f));
                f.g_color[3 * p + c] =
                    (1.0f - lam) * (sg * inv_n) + lam * (-0.5f * (A01[k].x + 2.0f * a * A01[k].y + b * A2[k]));
                // the depth/opacity gradient images start at zero (the LiDAR kernel follows; under
                // GS_LOSS_DEPTH_GRADS_ZERO they already are, and the LiDAR kernel runs alongside)
                if (c == 0 && !depth_grads_zero) {
                    f.g_depth[p] = 0.0f;
                    f.g_opac[p] = 0.0f;
                }
            }
        }
    }
    // block partial sums (deterministic order: warp butterfly, then fixed warp order)
    for (int o = 16; o > 0; o >>= 1) {
        l1_acc += __shfl_xor_sync(0xffffffffu, l1_acc, o);
        s_acc += __shfl_xor_sync(0xffffffffu, s_acc, o);
    }
    if ((tid & 31) == 0) {
        sm.red[0][tid >> 5] = l1_acc;
        sm.red[1][tid >> 5] = s_acc;
    }
    __syncthreads();
    if (tid == 0) {
        double l1 = 0.0, ss = 0.0;
        for (int w = 0; w < L_THREADS / 32; w++) {
            l1 += sm.red[0][w];
            ss += sm.red[1][w];
        }
        const int64_t blk = ((int64_t)blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
        f.loss_parts[3 * blk] = l1;
        f.loss_parts[3 * blk + 1] = ss;
        f.loss_parts[3 * blk + 2] = 0.0;
    }
}

// one launch for every (tile, channel): interior tiles (halo >= 10 px inside the image) take
// the compile-time-weight path, border tiles the reflection-table path
__global__ void __launch_bounds__(L_THREADS, 4) ssim_l1_kernel(gs_frame f, const gs_view *__restrict__ view,
                                                               const float *__restrict__ tab_x,
                                                               const float *__restrict__ tab_y, float lam,
                                                               int depth_grads_zero) {
    pdl_wait();
    // let the LiDAR kernel launch into the SMs this grid's last wave leaves idle (it waits for
    // this grid's completion itself before it reads the partials, or before anything when the
    // g_depth / g_opac clearing below is on)
    asm volatile("griddepcontrol.launch_dependents;");
    __shared__ SsimSmem sm;
    const int x0 = blockIdx.x * TW, y0 = blockIdx.y * TH;
    if (x0 >= 10 && x0 + TW + 10 <= f.width && y0 >= 10 && y0 + TH + 10 <= f.height)
        ssim_tile<true>(sm, f, view, tab_x, tab_y, lam, depth_grads_zero);
    else
        ssim_tile<false>(sm, f, view, tab_x, tab_y, lam, depth_grads_zero);
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
    if (overlap) pdl_wait();
    // this block's share of the SSIM-kernel partials (part0 triples), one per thread: the last
    // block then sums gridDim.x triples instead of part0 + gridDim.x (one memory round trip)
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
            f.loss[6] = (double)(pos + 1);
        }
        int *stamp = reinterpret_cast<int *>(tab_stamp);
        stamp[0] = (f.width << 16) + f.height;
        stamp[1] = ~((f.width << 16) + f.height);
    }
}

constexpr int DEPTH_BLOCKS = 64;

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
    launch_pdl(ssim_l1_kernel, grid, L_THREADS, 0, st, *f, view, tab_x, tab_y, lam, dz);
    if ((rc = check_launch("ssim_l1_kernel"))) return rc;
    launch_pdl(depth_loss_kernel, DEPTH_BLOCKS, 256, 0, st, *f, view, lam, xi, ssim_blocks, tab_y + 22 * f->height,
               (flags & GS_LOSS_ACCUMULATE) ? 1 : 0, dz);
    return check_launch("depth_loss_kernel");
}

namespace gs {
void init_loss_attrs() {
    cudaFuncSetAttribute(ssim_l1_kernel, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace gs
