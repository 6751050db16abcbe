// adam.cu -- chain rule to Gaussian attributes fused with the sparse Adam step (sm_100a).
//
// R/rasterizer.py:559-644 (_chain_to_attributes, attribute part) and R/rasterizer.py:707-725
// (sparse_adam_step: per-Gaussian step counter, eps 1e-15, untouched rows untouched).
// Work runs over the compacted touched list.  Each warp owns 32 touched Gaussians: their
// 256-B parameter rows are staged in shared memory with coalesced float4 loads, every lane
// computes its Gaussian's 59 gradients into shared memory, then the warp streams the Adam
// update over the 32 rows (params, m, v) with coalesced float4 traffic.  Nothing but the
// updated rows is written: the parameter-gradient rows never reach HBM on the 1-GPU path.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"

namespace gs {

constexpr int CA_WARPS = 4;
constexpr int CA_THREADS = CA_WARPS * 32;
constexpr int RP = 65;  // padded smem row
#ifndef CA_BATCH
#define CA_BATCH 4  // float4 per lane and array in flight in the fused Adam stream
#endif
static_assert(16 % CA_BATCH == 0, "the Adam stream's rounds tile the warp's 16 float4 per lane");
#ifndef CA_MINB
#define CA_MINB 4  // CTAs per SM the register budget is fitted to (16 warps)
#endif

// dR/dq of the normalised quaternion (R/rasterizer.py:490-499), contracted with gR
template <typename T>
__device__ __forceinline__ void quat_grad(const float q0[4], const T gR[9], float out[4]) {
    const T a = q0[0], b = q0[1], c = q0[2], d = q0[3];
    const T rn = (T)1 / gs_sqrt(a * a + b * b + c * c + d * d);
    const T w = a * rn, x = b * rn, y = c * rn, z = d * rn;
    const T zero = 0, two = 2;
    const T dw[9] = {zero, -z, y, z, zero, -x, -y, x, zero};
    const T dx[9] = {zero, y, z, y, -two * x, -w, z, w, -two * x};
    const T dy[9] = {-two * y, x, w, x, zero, z, -w, z, -two * y};
    const T dz[9] = {-two * z, -w, x, w, -two * z, y, x, y, zero};
    T a0 = 0, a1 = 0, a2 = 0, a3 = 0;
#pragma unroll
    for (int k = 0; k < 9; k++) {
        a0 += gR[k] * dw[k];
        a1 += gR[k] * dx[k];
        a2 += gR[k] * dy[k];
        a3 += gR[k] * dz[k];
    }
    const T gq[4] = {two * a0, two * a1, two * a2, two * a3};
    const T qh[4] = {w, x, y, z};
    const T dot = gq[0] * qh[0] + gq[1] * qh[1] + gq[2] * qh[2] + gq[3] * qh[3];
#pragma unroll
    for (int k = 0; k < 4; k++) out[k] = (float)((gq[k] - qh[k] * dot) * rn);
}

// gradient of the scalar loss w.r.t. one parameter row (59 columns written to G; every write
// happens after the last read of p, so G may alias p).  POSE: also this Gaussian's terms of the
// 6-dof pose gradient (rho, theta) on the left tangent of T_cw (R/rasterizer.py:646-657).
template <bool POSE>
__device__ __forceinline__ void chain_row(const float *p, const double *g, const gs_camera &cam, float *G,
                                          double *pose6) {
    // geometric chain in FP64: for Gaussians just past the 0.01 m near plane, J ~ fx/z ~ 1e5 and
    // the products below lose several fp32 digits; B200's FP64 pipe makes this nearly free here
    using D = double;
    const float *Rcf = cam.rot_cw;
    D Rc[9];
#pragma unroll
    for (int k = 0; k < 9; k++) Rc[k] = Rcf[k];
    const D fx = cam.fx, fy = cam.fy;
    ProjectedT<D> pr;
    project_full<D>(p, cam, pr);
    const D z = pr.mu[2];
    // conic -> 2x2 covariance gradient (R/rasterizer.py:583-592)
    const D ca = pr.ca, cb = pr.cb, cc = pr.cc;
    const D ga = g[2], gb = 0.5 * (D)g[3], gc = g[4];
    const D t00 = ca * ga + cb * gb, t01 = ca * gb + cb * gc, t10 = cb * ga + cc * gb, t11 = cb * gb + cc * gc;
    const D gv00 = -(t00 * ca + t01 * cb), gv01 = -(t00 * cb + t01 * cc);
    const D gv10 = -(t10 * ca + t11 * cb), gv11 = -(t10 * cb + t11 * cc);
    // cov2d = M S M^T (R/rasterizer.py:595-597)
    D tmp[6];
#pragma unroll
    for (int b = 0; b < 3; b++) {
        tmp[b] = gv00 * pr.M[b] + gv01 * pr.M[3 + b];
        tmp[3 + b] = gv10 * pr.M[b] + gv11 * pr.M[3 + b];
    }
    D gS[9], gM[6], gJ[6];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) gS[3 * a + b] = pr.M[a] * tmp[b] + pr.M[3 + a] * tmp[3 + b];
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            gM[3 * a + b] = 2.0 * (tmp[3 * a] * pr.S[b] + tmp[3 * a + 1] * pr.S[3 + b] + tmp[3 * a + 2] * pr.S[6 + b]);
#pragma unroll
    for (int a = 0; a < 2; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            gJ[3 * a + b] = gM[3 * a] * Rc[3 * b] + gM[3 * a + 1] * Rc[3 * b + 1] + gM[3 * a + 2] * Rc[3 * b + 2];
    // J and mean2d depend on the camera-frame mean (R/rasterizer.py:600-611)
    const D iz = 1.0 / z, iz2 = iz * iz, iz3 = iz2 * iz;
    D gx = gJ[2] * (-fx * iz2);
    D gy = gJ[5] * (-fy * iz2);
    D gz = gJ[0] * (-fx * iz2) + gJ[4] * (-fy * iz2) + gJ[2] * (2.0 * fx * pr.mu[0] * iz3) +
           gJ[5] * (2.0 * fy * pr.mu[1] * iz3);
    gx += (D)g[0] * fx * iz;
    gy += (D)g[1] * fy * iz;
    gz += -(D)g[0] * fx * pr.mu[0] * iz2 - (D)g[1] * fy * pr.mu[1] * iz2;
    gz += (D)g[9];
    float gpos[3];
#pragma unroll
    for (int c = 0; c < 3; c++) gpos[c] = (float)(gx * Rc[c] + gy * Rc[3 + c] + gz * Rc[6 + c]);
    // Sigma = (R S)(R S)^T (R/rasterizer.py:613-626)
    D gN[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++)
            gN[3 * a + b] = 2.0 * (gS[3 * a] * pr.R[b] + gS[3 * a + 1] * pr.R[3 + b] + gS[3 * a + 2] * pr.R[6 + b]) * pr.s[b];
    float gls[3];
#pragma unroll
    for (int j = 0; j < 3; j++)
        gls[j] = (float)((pr.R[j] * gN[j] + pr.R[3 + j] * gN[3 + j] + pr.R[6 + j] * gN[6 + j]) * pr.s[j]);
    D gR[9];
#pragma unroll
    for (int a = 0; a < 3; a++)
#pragma unroll
        for (int b = 0; b < 3; b++) gR[3 * a + b] = gN[3 * a + b] * pr.s[b];
    float gq[4];
    quat_grad<D>(p + 6, gR, gq);
    // opacity logit (R/rasterizer.py:629-630)
    const float o = 1.0f / (1.0f + expf(-p[10]));
    const float g_opl = (float)g[5] * o * (1.0f - o);
    // SH colour incl. the view-direction dependence (R/rasterizer.py:633-644)
    const float u0 = p[0] - cam.center[0], u1 = p[1] - cam.center[1], u2 = p[2] - cam.center[2];
    float un = sqrtf(u0 * u0 + u1 * u1 + u2 * u2);
    if (un < 1e-12f) un = 1.0f;
    const float run = 1.0f / un;
    const float d0 = u0 * run, d1 = u1 * run, d2 = u2 * run;
    float bs[16];
    sh_basis(d0, d1, d2, bs);
    float gcol[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < 15; k++) acc += bs[k + 1] * p[14 + 3 * k + c];
        const float pre = bs[0] * p[11 + c] + acc + 0.5f;
        gcol[c] = pre > 0.0f ? (float)g[6 + c] : 0.0f;
    }
    float sk[16];
    sk[0] = p[11] * gcol[0] + p[12] * gcol[1] + p[13] * gcol[2];
#pragma unroll
    for (int k = 0; k < 15; k++) sk[k + 1] = p[14 + 3 * k] * gcol[0] + p[15 + 3 * k] * gcol[1] + p[16 + 3 * k] * gcol[2];
    float gd[3];
    sh_basis_vjp(d0, d1, d2, sk, gd);
    const float dot = gd[0] * d0 + gd[1] * d1 + gd[2] * d2;
    const float gu[3] = {(gd[0] - d0 * dot) * run, (gd[1] - d1 * dot) * run, (gd[2] - d2 * dot) * run};
    if (POSE) {
        // translation: g_mu_cam + R_cw gu (the camera centre moves with rho, :656); rotation:
        // mu_cam x g_mu_cam + the covariance path through M = J R_cw: X = (J^T gM) R_cw^T,
        // theta += (X21 - X12, X02 - X20, X10 - X01) (:648-655)
        const D gmu[3] = {gx, gy, gz};
#pragma unroll
        for (int r = 0; r < 3; r++) pose6[r] = gmu[r] + (Rc[3 * r] * gu[0] + Rc[3 * r + 1] * gu[1] + Rc[3 * r + 2] * gu[2]);
        pose6[3] = pr.mu[1] * gz - pr.mu[2] * gy;
        pose6[4] = pr.mu[2] * gx - pr.mu[0] * gz;
        pose6[5] = pr.mu[0] * gy - pr.mu[1] * gx;
        D grc[9];
#pragma unroll
        for (int a = 0; a < 3; a++)
#pragma unroll
            for (int b = 0; b < 3; b++) grc[3 * a + b] = pr.J[a] * gM[b] + pr.J[3 + a] * gM[3 + b];
        auto X = [&](int a, int k) {
            return grc[3 * a] * Rc[3 * k] + grc[3 * a + 1] * Rc[3 * k + 1] + grc[3 * a + 2] * Rc[3 * k + 2];
        };
        pose6[3] += X(2, 1) - X(1, 2);
        pose6[4] += X(0, 2) - X(2, 0);
        pose6[5] += X(1, 0) - X(0, 1);
    }
    // every read of p is done: G may alias p from here on
#pragma unroll
    for (int c = 0; c < 3; c++) G[11 + c] = bs[0] * gcol[c];
#pragma unroll
    for (int k = 0; k < 15; k++)
#pragma unroll
        for (int c = 0; c < 3; c++) G[14 + 3 * k + c] = bs[k + 1] * gcol[c];
    G[0] = gpos[0] + gu[0];
    G[1] = gpos[1] + gu[1];
    G[2] = gpos[2] + gu[2];
#pragma unroll
    for (int j = 0; j < 3; j++) G[3 + j] = gls[j];
#pragma unroll
    for (int k = 0; k < 4; k++) G[6 + k] = gq[k];
    G[10] = g_opl;
}

// mode 0: fused Adam on params/m/v/t.  mode 1: grads[row] += G, touched_accum[row] = 1.
// mode 2: compact gradient rows + bias corrections for adam_list_kernel.  mode 3: nothing but the
// pose gradient (tracking).  POSE: pose6 (FP64, 6) += the pose gradient of the touched Gaussians.
template <bool POSE>
__global__ void __launch_bounds__(CA_THREADS, CA_MINB) chain_kernel(gs_frame f, float *__restrict__ params,
                                                           float *__restrict__ am, float *__restrict__ av,
                                                           int32_t *__restrict__ at, const gs_view *__restrict__ view,
                                                           const float *__restrict__ lr_cols, int mode,
                                                           float *__restrict__ grads, uint8_t *__restrict__ touched_accum,
                                                           double *__restrict__ pose_out, int part, int nparts) {
    pdl_wait();
    // one 32 x 65 staging tile per warp: parameter rows in, gradient rows out (in place)
    __shared__ float srow[CA_WARPS][32][RP];
    __shared__ float sbc[CA_WARPS][32][2];
    float(*sgr)[32][RP] = srow;
    __shared__ gs_camera scam;
    if (threadIdx.x == 0) scam = view->cam;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t ntt = f.counters[GS_CNT_OVERFLOW] ? 0 : f.counters[GS_CNT_TOUCHED];
    // without the forward's clear (GS_FWD_CLEAR_G2D) the engine keeps each row zero for the next
    // view by clearing it once read
    const bool clear_rows = mode != 2 && f.counters[GS_CNT_LAZY] && !f.counters[GS_CNT_FWD_CLEARED];
    // touched-list chunk `part` of `nparts` (warp-aligned bounds)
    // (no 64-bit divide -- a long subroutine -- on the common single-chunk path)
    const int64_t kb = nparts == 1 ? 0 : (ntt * part / nparts) & ~(int64_t)31;
    const int64_t nt = part == nparts - 1 ? ntt : ((ntt * (part + 1) / nparts) & ~(int64_t)31);
    const int64_t k0 = kb + ((int64_t)blockIdx.x * CA_WARPS + warp) * 32;
    if (k0 >= nt) return;
    const int64_t k = k0 + lane;
    const int g = k < nt ? f.touched_list[k] : -1;

    // stage the 32 parameter rows (coalesced: 16 lanes x float4 = one row)
#pragma unroll 4
    for (int j = 0; j < 16; j++) {
        const int kk = lane + 32 * j, r = kk >> 4, c4 = kk & 15;
        const int gg = __shfl_sync(0xffffffffu, g, r);
        if (gg >= 0) {
            const float4 val = *reinterpret_cast<const float4 *>(params + (int64_t)gg * GS_ROW + 4 * c4);
            srow[warp][r][4 * c4] = val.x;
            srow[warp][r][4 * c4 + 1] = val.y;
            srow[warp][r][4 * c4 + 2] = val.z;
            srow[warp][r][4 * c4 + 3] = val.w;
        }
    }
    __syncwarp();
    double pose6[6] = {0, 0, 0, 0, 0, 0};
    if (g >= 0) {
        // the fixed-point screen-space gradient row (GS_G2D_FIELDS (hi, lo) pairs, render.cu)
        const longlong2 *g2 = reinterpret_cast<const longlong2 *>(f.g2d) + k * (GS_G2D / 2);  // row = touched slot
        double gv[GS_G2D_FIELDS];
#pragma unroll
        for (int q = 0; q < GS_G2D_FIELDS; q++) {
            const longlong2 w = g2[q];
            gv[q] = fx_value(w.x, w.y);
        }
        if (clear_rows)
#pragma unroll
            for (int q = 0; q < GS_G2D_FIELDS; q++) const_cast<longlong2 *>(g2)[q] = make_longlong2(0, 0);
        chain_row<POSE>(srow[warp][lane], gv, scam, sgr[warp][lane], pose6);
        for (int q = GS_NPARAM; q < RP; q++) sgr[warp][lane][q] = 0.0f;
        if (mode == 0 || mode == 2) {
            const int tn = at[g] + 1;
            at[g] = tn;
            // reciprocal bias corrections 1/(1-b1^t), 1/(1-b2^t) (per-Gaussian t, R/rasterizer.py:714-722)
            const float bc1 = (float)(1.0 / (1.0 - pow(0.9, (double)tn))),
                        bc2 = (float)(1.0 / (1.0 - pow(0.999, (double)tn)));
            sbc[warp][lane][0] = bc1;
            sbc[warp][lane][1] = bc2;
            if (mode == 2) reinterpret_cast<float2 *>(f.bias_corr)[k] = make_float2(bc1, bc2);
        } else if (mode == 1) {
            touched_accum[g] = 1;
        }
    }
    if (POSE) {
        // per Gaussian to fixed point, integer warp sums, one pair of integer atomics per
        // component and warp: the sum does not depend on the (atomic-built) touched-list order
#pragma unroll
        for (int q = 0; q < 6; q++) {
            long long hi, lo;
            fx_split(pose6[q], hi, lo);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                hi += __shfl_xor_sync(0xffffffffu, hi, o);
                lo += __shfl_xor_sync(0xffffffffu, lo, o);
            }
            if (lane == 0) {
                atomicAdd(reinterpret_cast<unsigned long long *>(f.pose_acc) + 2 * q, (unsigned long long)hi);
                atomicAdd(reinterpret_cast<unsigned long long *>(f.pose_acc) + 2 * q + 1, (unsigned long long)lo);
            }
        }
        if (mode == 3) return;
    }
    __syncwarp();
    if (mode == 2) {  // gradient rows in touched-list order, streamed by adam_list_kernel
#pragma unroll 4
        for (int j = 0; j < 16; j++) {
            const int kk = lane + 32 * j, r = kk >> 4, c4 = kk & 15;
            if (k0 + r >= nt) continue;
            const float *G = &sgr[warp][r][4 * c4];
            reinterpret_cast<float4 *>(f.grad_rows)[(k0 + r) * (GS_ROW / 4) + c4] = make_float4(G[0], G[1], G[2], G[3]);
        }
        return;
    }
    if (mode == 0) {
        // the warp's 32 rows streamed in batches of CA_BATCH float4 per lane and array: every load
        // of a batch is in flight before the first use, so the update keeps HBM busy even at the
        // chain's low occupancy.  Parameters are re-read from global (staged a
        // moment ago: L2 hits); the smem tile holds G.
#pragma unroll 1
        for (int j0 = 0; j0 < 16; j0 += CA_BATCH) {
            float4 P[CA_BATCH], M4[CA_BATCH], V4[CA_BATCH];
            int64_t off[CA_BATCH];
            int gq[CA_BATCH];
#pragma unroll
            for (int q = 0; q < CA_BATCH; q++) {
                const int kk = lane + 32 * (j0 + q), r = kk >> 4, c4 = kk & 15;
                gq[q] = __shfl_sync(0xffffffffu, g, r);
                off[q] = (int64_t)gq[q] * GS_ROW + 4 * c4;
                if (gq[q] >= 0 && c4 < 15) {  // columns 60-63: padding, untouched
                    P[q] = *reinterpret_cast<const float4 *>(params + off[q]);
                    M4[q] = *reinterpret_cast<const float4 *>(am + off[q]);
                    V4[q] = *reinterpret_cast<const float4 *>(av + off[q]);
                }
            }
#pragma unroll
            for (int q = 0; q < CA_BATCH; q++) {
                const int kk = lane + 32 * (j0 + q), r = kk >> 4, c4 = kk & 15;
                if (gq[q] < 0 || c4 == 15) continue;
                const float *G = &sgr[warp][r][4 * c4];
                const float bc1 = sbc[warp][r][0], bc2 = sbc[warp][r][1];
                const float4 lr = __ldg(reinterpret_cast<const float4 *>(lr_cols) + c4);
                float4 m4 = M4[q], v4 = V4[q], p4;
#ifdef CA_SCALAR_ADAM
                p4.x = adam_one(P[q].x, m4.x, v4.x, G[0], lr.x, bc1, bc2);
                p4.y = adam_one(P[q].y, m4.y, v4.y, G[1], lr.y, bc1, bc2);
                p4.z = adam_one(P[q].z, m4.z, v4.z, G[2], lr.z, bc1, bc2);
                p4.w = c4 == 14 ? P[q].w : adam_one(P[q].w, m4.w, v4.w, G[3], lr.w, bc1, bc2);  // col 59: padding
#else
                adam_two(P[q].x, P[q].y, m4.x, m4.y, v4.x, v4.y, G[0], G[1], lr.x, lr.y, bc1, bc2, p4.x, p4.y);
                adam_two(P[q].z, P[q].w, m4.z, m4.w, v4.z, v4.w, G[2], G[3], lr.z, lr.w, bc1, bc2, p4.z, p4.w);
                if (c4 == 14) p4.w = P[q].w;  // col 59: padding
#endif
                if (c4 == 14) {
                    m4.w = M4[q].w;
                    v4.w = V4[q].w;
                }
                *reinterpret_cast<float4 *>(am + off[q]) = m4;
                *reinterpret_cast<float4 *>(av + off[q]) = v4;
                *reinterpret_cast<float4 *>(params + off[q]) = p4;
            }
        }
        return;
    }
#pragma unroll 2
    for (int j = 0; j < 16; j++) {
        const int kk = lane + 32 * j, r = kk >> 4, c4 = kk & 15;
        const int gg = __shfl_sync(0xffffffffu, g, r);
        if (gg < 0) continue;
        const int64_t off = (int64_t)gg * GS_ROW + 4 * c4;
        const float *G = &sgr[warp][r][4 * c4];
        {
            float4 acc = *reinterpret_cast<const float4 *>(grads + off);
            acc.x += G[0];
            acc.y += G[1];
            acc.z += G[2];
            acc.w += G[3];
            *reinterpret_cast<float4 *>(grads + off) = acc;
        }
    }
}

// sparse Adam streamed over the touched list: 16 threads per 256-B row, gradient rows and
// bias corrections produced by chain_kernel (mode 2) in the same order
__global__ void __launch_bounds__(256) adam_list_kernel(gs_frame f, float *__restrict__ params,
                                                        float *__restrict__ am, float *__restrict__ av,
                                                        const float *__restrict__ lr_cols, int part, int nparts) {
    pdl_wait();
    const int64_t ntt = f.counters[GS_CNT_OVERFLOW] ? 0 : f.counters[GS_CNT_TOUCHED];
    const int64_t kb = nparts == 1 ? 0 : (ntt * part / nparts) & ~(int64_t)31;
    const int64_t nt = part == nparts - 1 ? ntt : ((ntt * (part + 1) / nparts) & ~(int64_t)31);
    for (int64_t idx = kb * 16 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < nt * 16;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t k = idx >> 4;
        const int c4 = (int)(idx & 15);
        if (c4 == 15) continue;  // columns 60-63: padding
        const int64_t g = f.touched_list[k];
        if (c4 < GS_G2D / 2 && f.counters[GS_CNT_LAZY] && !f.counters[GS_CNT_FWD_CLEARED])
            reinterpret_cast<longlong2 *>(f.g2d)[k * (GS_G2D / 2) + c4] = make_longlong2(0, 0);
        const float2 bc = reinterpret_cast<const float2 *>(f.bias_corr)[k];
        const float4 G = reinterpret_cast<const float4 *>(f.grad_rows)[k * (GS_ROW / 4) + c4];
        const int64_t off = g * GS_ROW + 4 * c4;
        const float4 P = *reinterpret_cast<const float4 *>(params + off);
        float4 m4 = *reinterpret_cast<const float4 *>(am + off);
        float4 v4 = *reinterpret_cast<const float4 *>(av + off);
        const float4 lr = __ldg(reinterpret_cast<const float4 *>(lr_cols) + c4);
        float4 p4;
        p4.x = adam_one(P.x, m4.x, v4.x, G.x, lr.x, bc.x, bc.y);
        p4.y = adam_one(P.y, m4.y, v4.y, G.y, lr.y, bc.x, bc.y);
        p4.z = adam_one(P.z, m4.z, v4.z, G.z, lr.z, bc.x, bc.y);
        p4.w = c4 == 14 ? P.w : adam_one(P.w, m4.w, v4.w, G.w, lr.w, bc.x, bc.y);  // column 59: padding
        *reinterpret_cast<float4 *>(am + off) = m4;
        *reinterpret_cast<float4 *>(av + off) = v4;
        *reinterpret_cast<float4 *>(params + off) = p4;
    }
}

// dense sparse-Adam over a touched mask (multi-view / multi-GPU batches)
__global__ void adam_kernel(float *__restrict__ params, float *__restrict__ am, float *__restrict__ av,
                            int32_t *__restrict__ at, const float *__restrict__ grads,
                            const uint8_t *__restrict__ touched, int64_t n, const float *__restrict__ lr_cols) {
    pdl_wait();
    const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= n * 16) return;
    const int64_t row = idx >> 4;
    const int c4 = (int)(idx & 15);
    if (!touched[row]) return;
    const int tn = at[row] + 1;
    const float bc1 = (float)(1.0 / (1.0 - pow(0.9, (double)tn))), bc2 = (float)(1.0 / (1.0 - pow(0.999, (double)tn)));
    const int64_t off = row * GS_ROW + 4 * c4;
    float4 p4 = *reinterpret_cast<const float4 *>(params + off);
    float4 m4 = *reinterpret_cast<const float4 *>(am + off);
    float4 v4 = *reinterpret_cast<const float4 *>(av + off);
    const float4 g4 = *reinterpret_cast<const float4 *>(grads + off);
    const float4 lr = *reinterpret_cast<const float4 *>(lr_cols + 4 * c4);
    const float4 old = p4;
    p4.x = adam_one(p4.x, m4.x, v4.x, g4.x, lr.x, bc1, bc2);
    p4.y = adam_one(p4.y, m4.y, v4.y, g4.y, lr.y, bc1, bc2);
    p4.z = adam_one(p4.z, m4.z, v4.z, g4.z, lr.z, bc1, bc2);
    p4.w = adam_one(p4.w, m4.w, v4.w, g4.w, lr.w, bc1, bc2);
    if (c4 == 14) p4.w = old.w;
    if (c4 == 15) p4 = old;
    *reinterpret_cast<float4 *>(am + off) = m4;
    *reinterpret_cast<float4 *>(av + off) = v4;
    *reinterpret_cast<float4 *>(params + off) = p4;
}

// ---------------------------------------------------------------------------------------------
// Batch reduction (multi-view / multi-GPU): the touched union compacted in id
// order (identical on every rank, no host-side nonzero), the union's gradient rows gathered
// into a packed buffer for the collective, and Adam applied straight from the packed rows.

constexpr int CF_CHUNK = 1024;  // flags per compaction block

__global__ void __launch_bounds__(CF_CHUNK) compact_count_kernel(const uint8_t *__restrict__ flags, int64_t n,
                                                                 int32_t *chunk_cnt) {
    pdl_wait();
    __shared__ int s_w[CF_CHUNK / 32];
    const int64_t i = (int64_t)blockIdx.x * CF_CHUNK + threadIdx.x;
    const unsigned m = __ballot_sync(0xffffffffu, i < n && flags[i]);
    if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = __popc(m);
    __syncthreads();
    if (threadIdx.x < 32) {
        int v = s_w[threadIdx.x];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = v;
    }
}

__global__ void __launch_bounds__(CF_CHUNK) compact_write_kernel(const uint8_t *__restrict__ flags, int64_t n,
                                                                 const int32_t *__restrict__ chunk_cnt, int32_t *idx,
                                                                 int32_t *count) {
    pdl_wait();
    __shared__ int s_w[CF_CHUNK / 32];
    __shared__ int s_base;
    // this block's offset: the counts of the blocks before it (summed by the whole block)
    int acc = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += CF_CHUNK) acc += chunk_cnt[c];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (lane == 0) s_w[warp] = acc;
    __syncthreads();
    if (threadIdx.x == 0) {
        int b = 0;
        for (int w = 0; w < CF_CHUNK / 32; w++) b += s_w[w];
        s_base = b;
    }
    __syncthreads();
    const int64_t i = (int64_t)blockIdx.x * CF_CHUNK + threadIdx.x;
    const bool hit = i < n && flags[i];
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s_w[warp] = __popc(m);
    __syncthreads();
    int before = s_base;
    for (int w = 0; w < warp; w++) before += s_w[w];
    if (hit) idx[before + __popc(m & ((1u << lane) - 1u))] = (int32_t)i;
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        int tot = s_base;
        for (int w = 0; w < CF_CHUNK / 32; w++) tot += s_w[w];
        *count = tot;
    }
}

// packed[i, 0:60] = rows[idx[i], 0:60] for i < min(*count, cap): 15 float4 per row
__global__ void gather_rows_kernel(const float *__restrict__ rows, const int32_t *__restrict__ idx,
                                   const int32_t *__restrict__ count, int64_t cap, float *__restrict__ packed) {
    pdl_wait();
    const int64_t nr = min((int64_t)*count, cap);
    for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < nr * 15; q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q / 15;
        const int c4 = (int)(q - i * 15);
        reinterpret_cast<float4 *>(packed)[i * 15 + c4] =
            reinterpret_cast<const float4 *>(rows)[(int64_t)idx[i] * (GS_ROW / 4) + c4];
    }
}

// Sparse Adam over rows idx[first .. first + num) (clipped to *count): 16 threads per row; the
// gradient row is packed[i] (60 floats) or, without a packed buffer, grads[idx[i]]; the
// consumed gradient row and touched flag are cleared for the next batch.
__global__ void adam_packed_kernel(float *__restrict__ params, float *__restrict__ am, float *__restrict__ av,
                                   int32_t *__restrict__ at, const float *__restrict__ packed,
                                   const int32_t *__restrict__ idx, const int32_t *__restrict__ count, int64_t first,
                                   int64_t num, const float *__restrict__ lr_cols, float *__restrict__ grads,
                                   uint8_t *__restrict__ touched) {
    pdl_wait();
    const int64_t end = min(first + num, (int64_t)*count);
    for (int64_t q = first * 16 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < end * 16;
         q += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = q >> 4;
        const int c4 = (int)(q & 15);
        const int64_t row = idx[i];
        const int tn = at[row] + 1;  // read by the row's 16 lanes before its lane 15 writes it
        __syncwarp(0xffffu << (threadIdx.x & 16u));  // (the 16 lanes of a row share every loop trip)
        const float bc1 = (float)(1.0 / (1.0 - pow(0.9, (double)tn))), bc2 = (float)(1.0 / (1.0 - pow(0.999, (double)tn)));
        if (c4 == 15) {  // columns 60-63: padding; this lane bumps the step and clears the flag
            at[row] = tn;
            if (touched) touched[row] = 0;
            continue;
        }
        const int64_t off = row * GS_ROW + 4 * c4;
        const float4 g4 = packed ? reinterpret_cast<const float4 *>(packed)[i * 15 + c4]
                                 : *reinterpret_cast<const float4 *>(grads + off);
        if (grads) *reinterpret_cast<float4 *>(grads + off) = make_float4(0.f, 0.f, 0.f, 0.f);
        const float4 P = *reinterpret_cast<const float4 *>(params + off);
        float4 m4 = *reinterpret_cast<const float4 *>(am + off);
        float4 v4 = *reinterpret_cast<const float4 *>(av + off);
        const float4 lr = __ldg(reinterpret_cast<const float4 *>(lr_cols) + c4);
        float4 p4;
        p4.x = adam_one(P.x, m4.x, v4.x, g4.x, lr.x, bc1, bc2);
        p4.y = adam_one(P.y, m4.y, v4.y, g4.y, lr.y, bc1, bc2);
        p4.z = adam_one(P.z, m4.z, v4.z, g4.z, lr.z, bc1, bc2);
        if (c4 == 14) {  // column 59: padding
            p4.w = P.w;
        } else {
            p4.w = adam_one(P.w, m4.w, v4.w, g4.w, lr.w, bc1, bc2);
        }
        *reinterpret_cast<float4 *>(am + off) = m4;
        *reinterpret_cast<float4 *>(av + off) = v4;
        *reinterpret_cast<float4 *>(params + off) = p4;
    }
}

// the pose gradient from its fixed-point accumulators (gs_chain_pose)
// the pose gradient from its fixed-point accumulators, which are then cleared for the next
// gs_chain_pose (self-resetting: no memset node in a captured tracking iteration; workspaces
// start zero-filled)
__global__ void pose_finish_kernel(int64_t *__restrict__ acc, double *pose) {
    pdl_wait();
    const int q = threadIdx.x;
    if (q < 6) {
        pose[q] = fx_value(acc[2 * q], acc[2 * q + 1]);
        acc[2 * q] = 0;
        acc[2 * q + 1] = 0;
    }
}

// step counters advance after the update kernel has read them (no intra-kernel race)
__global__ void adam_step_kernel(int32_t *__restrict__ at, const uint8_t *__restrict__ touched, int64_t n) {
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && touched[i]) at[i] += 1;
}

}  // namespace gs

using namespace gs;

static int launch_chain(const gs_frame *f, float *params, float *m, float *v, int32_t *t, const gs_view *view,
                        const float *lr, int mode, float *grads, uint8_t *acc, void *stream, double *pose = nullptr,
                        int part = 0, int nparts = 1) {
    if (f->n == 0) return GS_OK;
    const int64_t warps = (f->n / nparts + 63) / 32;  // a chunk's upper bound (touched <= n)
    const unsigned blocks = (unsigned)((warps + CA_WARPS - 1) / CA_WARPS);
    if (pose)
        launch_pdl(chain_kernel<true>, blocks, CA_THREADS, 0, (cudaStream_t)stream, *f, params, m, v, t, view, lr, mode, grads,
                                                                            acc, pose, part, nparts);
    else
        launch_pdl(chain_kernel<false>, blocks, CA_THREADS, 0, (cudaStream_t)stream, *f, params, m, v, t, view, lr, mode, grads,
                                                                             acc, nullptr, part, nparts);
    return check_launch("chain_kernel");
}

extern "C" int gs_chain_adam(const gs_frame *f, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                             const gs_view *view, const float *lr_cols, void *stream) {
    if (!params || !adam_m || !adam_v || !adam_t || !view || !lr_cols) {
        set_error("gs_chain_adam: null argument");
        return GS_ERR_ARG;
    }
    // fused: the chain rule (FP64 geometry) hands each warp's 32 gradient rows to the Adam update
    // through shared memory, so gradient rows never reach HBM.  GSLIC_SPLIT_ADAM=1 selects the
    // split form (compact gradient rows + a streaming adam_list_kernel) for comparison.
    static const bool split = [] {
        const char *e = getenv("GSLIC_SPLIT_ADAM");
        return e && e[0] == '1';
    }();
    int rc = launch_chain(f, params, adam_m, adam_v, adam_t, view, lr_cols, split ? 2 : 0, nullptr, nullptr, stream);
    if (rc || !split) return rc;
    if (f->n == 0) return GS_OK;
    launch_pdl(adam_list_kernel, 8 * 148, 256, 0, (cudaStream_t)stream, *f, params, adam_m, adam_v, lr_cols, 0, 1);
    return check_launch("adam_list_kernel");
}

extern "C" int gs_chain_adam_part(const gs_frame *f, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                                  const gs_view *view, const float *lr_cols, int32_t stage, int32_t part,
                                  int32_t nparts, void *stream) {
    if (!params || !adam_m || !adam_v || !adam_t || !view || !lr_cols || nparts < 1 || part < 0 || part >= nparts ||
        (stage != 0 && stage != 1)) {
        set_error("gs_chain_adam_part: bad arguments");
        return GS_ERR_ARG;
    }
    if (f->n == 0) return GS_OK;
    if (stage == 0)  // chain rule of the chunk: compact gradient rows + bias corrections, t bumped
        return launch_chain(f, params, adam_m, adam_v, adam_t, view, lr_cols, 2, nullptr, nullptr, stream, nullptr,
                            part, nparts);
    launch_pdl(adam_list_kernel, 4 * 148, 256, 0, (cudaStream_t)stream, *f, params, adam_m, adam_v, lr_cols, part, nparts);
    return check_launch("adam_list_kernel");
}

extern "C" int gs_chain(const gs_frame *f, const float *params, float *grads, uint8_t *touched_accum,
                        const gs_view *view, void *stream) {
    if (!params || !grads || !touched_accum || !view) {
        set_error("gs_chain: null argument");
        return GS_ERR_ARG;
    }
    return launch_chain(f, const_cast<float *>(params), nullptr, nullptr, nullptr, view, nullptr, 1, grads,
                        touched_accum, stream);
}

extern "C" int gs_chain_pose(const gs_frame *f, const float *params, float *grads, uint8_t *touched_accum,
                             const gs_view *view, double *pose, void *stream) {
    if (!params || !view || !pose || (!grads) != (!touched_accum)) {
        set_error("gs_chain_pose: null argument (grads and touched_accum are both set or both NULL)");
        return GS_ERR_ARG;
    }
    // (pose_acc is zero here: pose_finish_kernel clears it after every use)
    int rc = launch_chain(f, const_cast<float *>(params), nullptr, nullptr, nullptr, view, nullptr, grads ? 1 : 3,
                          grads, touched_accum, stream, pose);
    if (rc) return rc;
    launch_pdl(pose_finish_kernel, 1, 32, 0, (cudaStream_t)stream, f->pose_acc, pose);
    return check_launch("pose_finish_kernel");
}

extern "C" int gs_adam(float *params, float *adam_m, float *adam_v, int32_t *adam_t, const float *grads,
                       const uint8_t *touched, int64_t n, const float *lr_cols, void *stream) {
    if (n == 0) return GS_OK;
    const int64_t work = n * 16;
    launch_pdl(adam_kernel, (unsigned)((work + 255) / 256), 256, 0, (cudaStream_t)stream, params, adam_m, adam_v, adam_t, grads,
                                                                                   touched, n, lr_cols);
    int rc = check_launch("adam_kernel");
    if (rc) return rc;
    launch_pdl(adam_step_kernel, (unsigned)((n + 255) / 256), 256, 0, (cudaStream_t)stream, adam_t, touched, n);
    return check_launch("adam_step_kernel");
}

extern "C" int gs_compact_flags(const uint8_t *flags, int64_t n, int32_t *idx, int32_t *count, int32_t *scratch,
                                void *stream) {
    if (n < 0 || (n > 0 && (!flags || !idx || !count || !scratch))) {
        set_error("gs_compact_flags: bad arguments");
        return GS_ERR_ARG;
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (n == 0) {
        cudaMemsetAsync(count, 0, sizeof(int32_t), st);
        return check_launch("gs_compact_flags");
    }
    const unsigned chunks = (unsigned)((n + CF_CHUNK - 1) / CF_CHUNK);
    launch_pdl(compact_count_kernel, chunks, CF_CHUNK, 0, st, flags, n, scratch);
    int rc = check_launch("compact_count_kernel");
    if (rc) return rc;
    launch_pdl(compact_write_kernel, chunks, CF_CHUNK, 0, st, flags, n, (const int32_t *)scratch, idx, count);
    return check_launch("compact_write_kernel");
}

extern "C" int gs_gather_rows(const float *rows, const int32_t *idx, const int32_t *count, int64_t cap, float *packed,
                              void *stream) {
    if (!rows || !idx || !count || !packed || cap < 0) {
        set_error("gs_gather_rows: bad arguments");
        return GS_ERR_ARG;
    }
    if (cap == 0) return GS_OK;
    launch_pdl(gather_rows_kernel, 4 * 148, 256, 0, (cudaStream_t)stream, rows, idx, count, cap, packed);
    return check_launch("gather_rows_kernel");
}

extern "C" int gs_adam_packed(float *params, float *adam_m, float *adam_v, int32_t *adam_t, const float *packed,
                              const int32_t *idx, const int32_t *count, int64_t first, int64_t num,
                              const float *lr_cols, float *grads, uint8_t *touched, void *stream) {
    if (!params || !adam_m || !adam_v || !adam_t || !idx || !count || !lr_cols || (!packed && !grads) || first < 0 ||
        num < 0) {
        set_error("gs_adam_packed: bad arguments");
        return GS_ERR_ARG;
    }
    if (num == 0) return GS_OK;
    const int64_t work = num * 16;
    const unsigned blocks = (unsigned)std::min<int64_t>((work + 255) / 256, 16 * 148);
    launch_pdl(adam_packed_kernel, blocks, 256, 0, (cudaStream_t)stream, params, adam_m, adam_v, adam_t, packed, idx,
               count, first, num, lr_cols, grads, touched);
    return check_launch("adam_packed_kernel");
}

namespace gs {
void init_chain_attrs() {
    // static shared memory only (33 KB per 4-warp CTA); nothing to opt in
    cudaFuncSetAttribute(chain_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(chain_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace gs
