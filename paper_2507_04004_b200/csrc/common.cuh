// common.cuh -- shared device helpers for the sm_100a map-optimisation kernels.
#pragma once
#include <utility>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/gslic.h"

#define GS_WARP 32
#define GS_NEAR_CLIP 0.01f     // R/gaussians.py:34
#define GS_DILATION 0.3f       // R/gaussians.py:33
#define GS_ALPHA_CLAMP 0.99f   // R/gaussians.py:35
#define GS_EARLY_STOP_T 1e-4f  // R/rasterizer.py:43
#define GS_LOG2E 1.4426950408889634f

// counters beyond the public GS_CNT_* slots: per-pass tile tickets for the lookback kernels
#define GS_CNT_TICKET0 8

namespace gs {

// huge records (depth order): 8 ints each (id, depth bits, slot), then their ids, then their keys
constexpr int HREC = 8;
constexpr int HIDS = HREC * GS_HUGE_CAP;
constexpr int HKEYS = HIDS + GS_HUGE_CAP;  // int offset of the uint64 key array (8-B aligned)
constexpr int HSTAGE = HKEYS + 2 * GS_HUGE_CAP;  // unsorted keys staged by big_cull_kernel

// ---------------------------------------------------------------------------
// error plumbing (thread-local, no global mutable state shared across threads)
void set_error(const char *fmt, ...);
int check_launch(const char *what);

// Single MUFU instructions without the IEEE rounding / range fix-up sequences (~1-2 ulp,
// subnormal inputs and results flush to zero).  Used where the operands are known to be normal
// and an ulp is far below the path's tolerance (blend alpha, SSIM map, Adam denominator).
__device__ __forceinline__ float fast_ex2(float x) {
    float y;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_rcp(float x) {
    float y;
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}
__device__ __forceinline__ float fast_sqrt(float x) {
    float y;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
    return y;
}

// Programmatic dependent launch: every kernel of the library is launched with programmatic
// stream serialisation and waits for its predecessor's completion (and memory flush) as its
// first action, so its launch and block scheduling overlap the predecessor's tail instead of
// following it.  Outside a PDL launch griddepcontrol.wait returns at once.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t stream,
                              Args &&...args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// SH constants, R/gaussians.py:24-30
__device__ __constant__ static const float SH_C0 = 0.28209479177387814f;
__device__ __constant__ static const float SH_C1 = 0.4886025119029199f;

struct Sh {
    static constexpr float C2_0 = 1.0925484305920792f, C2_1 = -1.0925484305920792f, C2_2 = 0.31539156525252005f,
                           C2_3 = -1.0925484305920792f, C2_4 = 0.5462742152960396f;
    static constexpr float C3_0 = -0.5900435899266435f, C3_1 = 2.890611442640554f, C3_2 = -0.4570457994644658f,
                           C3_3 = 0.3731763325901154f, C3_4 = -0.4570457994644658f, C3_5 = 1.445305721320277f,
                           C3_6 = -0.5900435899266435f;
};

// real SH basis, degrees 0..3 (R/gaussians.py:51-74)
__device__ __forceinline__ void sh_basis(float x, float y, float z, float b[16]) {
    float xx = x * x, yy = y * y, zz = z * z, xy = x * y, yz = y * z, xz = x * z;
    b[0] = 0.28209479177387814f;
    b[1] = -0.4886025119029199f * y;
    b[2] = 0.4886025119029199f * z;
    b[3] = -0.4886025119029199f * x;
    b[4] = Sh::C2_0 * xy;
    b[5] = Sh::C2_1 * yz;
    b[6] = Sh::C2_2 * (2.0f * zz - xx - yy);
    b[7] = Sh::C2_3 * xz;
    b[8] = Sh::C2_4 * (xx - yy);
    b[9] = Sh::C3_0 * y * (3.0f * xx - yy);
    b[10] = Sh::C3_1 * xy * z;
    b[11] = Sh::C3_2 * y * (4.0f * zz - xx - yy);
    b[12] = Sh::C3_3 * z * (2.0f * zz - 3.0f * xx - 3.0f * yy);
    b[13] = Sh::C3_4 * x * (4.0f * zz - xx - yy);
    b[14] = Sh::C3_5 * z * (xx - yy);
    b[15] = Sh::C3_6 * x * (xx - 3.0f * yy);
}

// d basis / d dir  (R/gaussians.py:77-99), returns gdir = sum_k dB_k/dd * s_k
__device__ __forceinline__ void sh_basis_vjp(float x, float y, float z, const float s[16], float g[3]) {
    float gx = -0.4886025119029199f * s[3], gy = -0.4886025119029199f * s[1], gz = 0.4886025119029199f * s[2];
    gx += Sh::C2_0 * y * s[4];
    gy += Sh::C2_0 * x * s[4];
    gy += Sh::C2_1 * z * s[5];
    gz += Sh::C2_1 * y * s[5];
    gx += Sh::C2_2 * (-2.0f * x) * s[6];
    gy += Sh::C2_2 * (-2.0f * y) * s[6];
    gz += Sh::C2_2 * (4.0f * z) * s[6];
    gx += Sh::C2_3 * z * s[7];
    gz += Sh::C2_3 * x * s[7];
    gx += Sh::C2_4 * (2.0f * x) * s[8];
    gy += Sh::C2_4 * (-2.0f * y) * s[8];
    gx += Sh::C3_0 * (6.0f * x * y) * s[9];
    gy += Sh::C3_0 * (3.0f * x * x - 3.0f * y * y) * s[9];
    gx += Sh::C3_1 * (y * z) * s[10];
    gy += Sh::C3_1 * (x * z) * s[10];
    gz += Sh::C3_1 * (x * y) * s[10];
    gx += Sh::C3_2 * (-2.0f * x * y) * s[11];
    gy += Sh::C3_2 * (4.0f * z * z - x * x - 3.0f * y * y) * s[11];
    gz += Sh::C3_2 * (8.0f * y * z) * s[11];
    gx += Sh::C3_3 * (-6.0f * x * z) * s[12];
    gy += Sh::C3_3 * (-6.0f * y * z) * s[12];
    gz += Sh::C3_3 * (6.0f * z * z - 3.0f * x * x - 3.0f * y * y) * s[12];
    gx += Sh::C3_4 * (4.0f * z * z - 3.0f * x * x - y * y) * s[13];
    gy += Sh::C3_4 * (-2.0f * x * y) * s[13];
    gz += Sh::C3_4 * (8.0f * x * z) * s[13];
    gx += Sh::C3_5 * (2.0f * x * z) * s[14];
    gy += Sh::C3_5 * (-2.0f * y * z) * s[14];
    gz += Sh::C3_5 * (x * x - y * y) * s[14];
    gx += Sh::C3_6 * (3.0f * x * x - 3.0f * y * y) * s[15];
    gy += Sh::C3_6 * (-6.0f * x * y) * s[15];
    g[0] = gx;
    g[1] = gy;
    g[2] = gz;
}

// ---------------------------------------------------------------------------
// projection (R/gaussians.py:156-215)

// T = float on the forward path; T = double in the chain rule, whose Jacobian products are
// ill-conditioned for Gaussians just beyond the 0.01 m near plane (fx/z ~ 1e5)
template <typename T>
struct ProjectedT {
    T mu[3];
    T J[6];   // 2x3
    T M[6];   // J R_cw
    T R[9];   // rotation of the Gaussian (normalised quaternion)
    T s[3];   // exp(log_scale)
    T S[9];   // world covariance
    T c00, c01, c11;  // dilated 2x2 covariance
    T det;
    T mx, my;
    T ca, cb, cc;  // conic
    bool valid;
};
using Projected = ProjectedT<float>;

__device__ __forceinline__ float gs_sqrt(float x) { return sqrtf(x); }
__device__ __forceinline__ double gs_sqrt(double x) { return sqrt(x); }
__device__ __forceinline__ float gs_exp(float x) { return expf(x); }
__device__ __forceinline__ double gs_exp(double x) { return exp(x); }

template <typename T>
__device__ __forceinline__ void quat_rot(const float q[4], T R[9]) {
    const T q0 = q[0], q1 = q[1], q2 = q[2], q3 = q[3];
    const T rn = (T)1 / gs_sqrt(q0 * q0 + q1 * q1 + q2 * q2 + q3 * q3);  // one divide, four products
    const T w = q0 * rn, x = q1 * rn, y = q2 * rn, z = q3 * rn;
    const T one = 1, two = 2;
    R[0] = one - two * (y * y + z * z); R[1] = two * (x * y - w * z); R[2] = two * (x * z + w * y);
    R[3] = two * (x * y + w * z); R[4] = one - two * (x * x + z * z); R[5] = two * (y * z - w * x);
    R[6] = two * (x * z - w * y); R[7] = two * (y * z + w * x); R[8] = one - two * (x * x + y * y);
}

// p: pos[3], log_scale[3], quat[4] (the first 10 columns of a parameter row)
template <typename T>
__device__ __forceinline__ void project_full(const float *p, const gs_camera &cam, ProjectedT<T> &o) {
    const float *Rc = cam.rot_cw;
    for (int r = 0; r < 3; r++)
        o.mu[r] = ((T)p[0] * (T)Rc[3 * r] + (T)p[1] * (T)Rc[3 * r + 1] + (T)p[2] * (T)Rc[3 * r + 2]) + (T)cam.trans_cw[r];
    const T z = o.mu[2];
    bool v = z > (T)GS_NEAR_CLIP;
    const T zs = v ? z : (T)1;
    const T iz = (T)1 / zs;
    const T fx = cam.fx, fy = cam.fy;
    o.mx = fx * o.mu[0] * iz + (T)cam.cx;
    o.my = fy * o.mu[1] * iz + (T)cam.cy;
    o.J[0] = fx * iz; o.J[1] = 0; o.J[2] = -fx * o.mu[0] * iz * iz;
    o.J[3] = 0; o.J[4] = fy * iz; o.J[5] = -fy * o.mu[1] * iz * iz;
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 3; c++)
            o.M[3 * r + c] = o.J[3 * r] * (T)Rc[c] + o.J[3 * r + 1] * (T)Rc[3 + c] + o.J[3 * r + 2] * (T)Rc[6 + c];
    quat_rot<T>(p + 6, o.R);
    // scales from the fp32 exponential (~2 ulp): no cancellation downstream, unlike mu_cam
    o.s[0] = (T)expf(p[3]); o.s[1] = (T)expf(p[4]); o.s[2] = (T)expf(p[5]);
    const T s2[3] = {o.s[0] * o.s[0], o.s[1] * o.s[1], o.s[2] * o.s[2]};
    for (int a = 0; a < 3; a++)
        for (int b = a; b < 3; b++) {
            const T val = o.R[3 * a] * s2[0] * o.R[3 * b] + o.R[3 * a + 1] * s2[1] * o.R[3 * b + 1] +
                          o.R[3 * a + 2] * s2[2] * o.R[3 * b + 2];
            o.S[3 * a + b] = val;
            o.S[3 * b + a] = val;
        }
    T MS[6];
    for (int r = 0; r < 2; r++)
        for (int c = 0; c < 3; c++) MS[3 * r + c] = o.M[3 * r] * o.S[c] + o.M[3 * r + 1] * o.S[3 + c] + o.M[3 * r + 2] * o.S[6 + c];
    o.c00 = MS[0] * o.M[0] + MS[1] * o.M[1] + MS[2] * o.M[2] + (T)GS_DILATION;
    o.c01 = MS[0] * o.M[3] + MS[1] * o.M[4] + MS[2] * o.M[5];
    o.c11 = MS[3] * o.M[3] + MS[4] * o.M[4] + MS[5] * o.M[5] + (T)GS_DILATION;
    o.det = o.c00 * o.c11 - o.c01 * o.c01;
    v = v && (o.det > (T)1e-12f) && isfinite(o.det);
    o.valid = v;
    const T idet = (T)1 / (v ? o.det : (T)1);
    o.ca = o.c11 * idet;
    o.cb = -o.c01 * idet;
    o.cc = o.c00 * idet;
}

// ---------------------------------------------------------------------------
// binning decision path: strict IEEE fp32 (no contraction) so that the CPU fp32 restatement
// (oracle/gs_oracle.c f32_rect / f32_tile_min_q) reproduces every decision bit for bit.

__device__ __forceinline__ float det_logf(float x) {  // x >= 1, see DESIGN.md
    uint32_t u = __float_as_uint(x);
    int e = (int)((u >> 23) & 0xffu) - 127;
    float m = __uint_as_float((u & 0x7fffffu) | 0x3f800000u);
    if (m > 1.41421353816986083984375f) {
        m = __fmul_rn(m, 0.5f);
        e += 1;
    }
    float s = __fdiv_rn(__fsub_rn(m, 1.0f), __fadd_rn(m, 1.0f));
    float s2 = __fmul_rn(s, s);
    float p = __fmaf_rn(s2, 0.111111111938953399658203125f, 0.14285714924335479736328125f);
    p = __fmaf_rn(p, s2, 0.20000000298023223876953125f);
    p = __fmaf_rn(p, s2, 0.3333333432674407958984375f);
    p = __fmaf_rn(p, s2, 1.0f);
    float lm = __fmul_rn(__fmul_rn(2.0f, s), p);
    return __fmaf_rn((float)e, 0.693147182464599609375f, lm);
}

// influence radius + tile rectangle (R/rasterizer.py:84-102, 183-194).  Returns false when the
// Gaussian has no candidate tile.
__device__ __forceinline__ bool tile_rect(float c00, float c01, float c11, float o, float mx, float my, int width,
                                          int height, int tiles_x, int tiles_y, int4 &rect, float &qcut,
                                          float &radius) {
    float half_tr = __fmul_rn(0.5f, __fadd_rn(c00, c11));
    float df = __fsub_rn(c00, c11);
    float dd = __fadd_rn(__fmul_rn(0.25f, __fmul_rn(df, df)), __fmul_rn(c01, c01));
    float lam = __fadd_rn(half_tr, __fsqrt_rn(dd > 0.0f ? dd : 0.0f));
    if (!(o > (float)(1.0 / 255.0))) return false;
    float L = det_logf(__fmul_rn(255.0f, o));
    float r = __fadd_rn(__fsqrt_rn(__fmul_rn(__fmul_rn(2.0f, L), lam)), 1e-6f);
    radius = r;
    if (!(r > 0.0f)) return false;
    if ((__fadd_rn(mx, r) < 0.0f) || (__fsub_rn(mx, r) > (float)(width - 1)) || (__fadd_rn(my, r) < 0.0f) ||
        (__fsub_rn(my, r) > (float)(height - 1)))
        return false;
    float f;
    f = floorf(__fmul_rn(__fsub_rn(mx, r), 0.0625f));
    rect.x = f < 0.0f ? 0 : (f > (float)(tiles_x - 1) ? tiles_x - 1 : (int)f);
    f = floorf(__fmul_rn(__fadd_rn(mx, r), 0.0625f));
    rect.y = f < 0.0f ? 0 : (f > (float)(tiles_x - 1) ? tiles_x - 1 : (int)f);
    f = floorf(__fmul_rn(__fsub_rn(my, r), 0.0625f));
    rect.z = f < 0.0f ? 0 : (f > (float)(tiles_y - 1) ? tiles_y - 1 : (int)f);
    f = floorf(__fmul_rn(__fadd_rn(my, r), 0.0625f));
    rect.w = f < 0.0f ? 0 : (f > (float)(tiles_y - 1) ? tiles_y - 1 : (int)f);
    qcut = __fmul_rn(2.0f, L);
    return true;
}

// q at integer pixel column xc on row offset dy (R/rasterizer.py:143-144, strict order)
__device__ __forceinline__ float quad_q(float ca, float cb, float cc, float dx, float dy) {
    return __fadd_rn(__fadd_rn(__fmul_rn(__fmul_rn(ca, dx), dx), __fmul_rn(__fmul_rn(__fmul_rn(2.0f, cb), dx), dy)),
                     __fmul_rn(__fmul_rn(cc, dy), dy));
}

// Exact cull of one (Gaussian, tile) pair (R/rasterizer.py:125-166): keep iff the minimum of
// the quadratic over the tile's integer pixel grid is <= qcut (= 2 ln(255 o), the q-domain
// form of o e^{-q/2} >= 1/255).  "min <= qcut" == "some evaluated q <= qcut", so rows are
// scanned outward from the mean row and the scan stops at the first hit.  A conservative
// continuous lower bound rejects clearly-outside tiles without the scan.
// the two per-row candidates of R/rasterizer.py:134-146 for one pixel row; true if either
// evaluates to q <= qcut
__device__ __forceinline__ bool row_hits(float mx, float my, float ca, float cb, float cc, float qcut, int x0, int x1,
                                         int py) {
    const float dy = __fsub_rn((float)py, my);
    float xsr = __fsub_rn(mx, __fdiv_rn(__fmul_rn(cb, dy), ca));
    const float lo = (float)(x0 - 1), hi = (float)(x1 + 1);
    if (!(xsr >= lo)) xsr = lo;
    if (xsr > hi) xsr = hi;
    const int xf = (int)floorf(xsr);
#pragma unroll
    for (int j = 0; j < 2; j++) {
        int xc = xf + j;
        xc = xc < x0 ? x0 : (xc > x1 ? x1 : xc);
        const float dx = __fsub_rn((float)xc, mx);
        if (quad_q(ca, cb, cc, dx, dy) <= qcut) return true;
    }
    return false;
}

__device__ __forceinline__ bool tile_keep(float mx, float my, float ca, float cb, float cc, float qcut, int x0,
                                          int x1, int y0, int y1) {
    // 1) the row nearest the mean first: most kept tiles are decided by its two candidates
    int r0 = (int)floorf(my + 0.5f);
    r0 = r0 < y0 ? y0 : (r0 > y1 ? y1 : r0);
    if (row_hits(mx, my, ca, cb, cc, qcut, x0, x1, r0)) return true;
    // 2) conservative continuous lower bound over [x0,x1]x[y0,y1] rejects clearly-outside
    //    tiles (margin >> the fp32 evaluation error of q, so no kept tile is ever rejected)
    const float ax0 = (float)x0 - mx, ax1 = (float)x1 - mx, ay0 = (float)y0 - my, ay1 = (float)y1 - my;
    if (!(ax0 <= 0.0f && ax1 >= 0.0f && ay0 <= 0.0f && ay1 >= 0.0f)) {
        float qc = 3.0e38f;
        const float ys[2] = {ay0, ay1}, xs[2] = {ax0, ax1};
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const float y = ys[k];
            const float dx = fminf(fmaxf(-cb * y / ca, ax0), ax1);
            qc = fminf(qc, ca * dx * dx + 2.0f * cb * dx * y + cc * y * y);
            const float x = xs[k];
            const float dy = fminf(fmaxf(-cb * x / cc, ay0), ay1);
            qc = fminf(qc, ca * x * x + 2.0f * cb * x * dy + cc * dy * dy);
        }
        const float scale = ca * fmaxf(ax0 * ax0, ax1 * ax1) + cc * fmaxf(ay0 * ay0, ay1 * ay1);
        if (qc - 1e-5f * scale - 1e-6f > qcut) return false;
    }
    // 3) the remaining rows, outward from r0 (r0-1, r0+1, r0-2, ...)
    for (int k = 1, up = r0 + 1, dn = r0 - 1; k < y1 - y0 + 1; k++) {
        int py;
        if ((k & 1) == 1) py = (dn >= y0) ? dn-- : up++;
        else py = (up <= y1) ? up++ : dn--;
        if (row_hits(mx, my, ca, cb, cc, qcut, x0, x1, py)) return true;
    }
    return false;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// ---------------------------------------------------------------------------
// 2D splat records (GS_SPLAT floats per Gaussian, gslic.h).  The blend evaluates the quadratic
// in the factored form q = a (dx + beta dy)^2 + gamma dy^2 (beta = b / a, gamma = det / a =
// 1 / c00'), whose three coefficients are rounded to fp32 from FP64 and stay well conditioned for
// needle-shaped footprints: rounding (a, b, c) themselves perturbs det(conic) by
// ~6e-8 * a c / det, up to 5e-3 for Gaussians just past the near plane, which moved their
// position gradients by 2e-3.  The binning keeps the reference's
// (a, b, c) in the strict-IEEE decision path of the fp32 oracle restatement.
struct SplatCull {
    float mx, my, ca, cb, cc, qcut;
};

__device__ __forceinline__ SplatCull splat_cull(const float *splat2d, int64_t g) {
    const float4 A = reinterpret_cast<const float4 *>(splat2d)[GS_SPLAT / 4 * g];
    const float4 B = reinterpret_cast<const float4 *>(splat2d)[GS_SPLAT / 4 * g + 1];
    const float2 D = reinterpret_cast<const float2 *>(splat2d)[GS_SPLAT / 2 * g + 6];
    return SplatCull{A.x, A.y, A.z, D.x, D.y, B.w};
}

__device__ __forceinline__ float splat_depth(const float *splat2d, int64_t g) { return splat2d[GS_SPLAT * g + 6]; }

// The touched-list slot of a touched Gaussian (float 14 of its record, as int bits): its
// screen-space gradient row in the g2d array.  g2d rows are indexed by slot, not by Gaussian, so
// the rows the backward accumulates into and the chain rule reads and clears form one dense
// block of nt rows (46 MB at the benchmark's 286k touched) instead of 160-B rows scattered over
// the n-row array: every line of the block is fully used and it stays L2-resident.
__device__ __forceinline__ void splat_set_slot(float *splat2d, int64_t g, int slot) {
    splat2d[GS_SPLAT * g + 14] = __int_as_float(slot);
}
__device__ __forceinline__ int splat_slot(const float *splat2d, int64_t g) {
    return __float_as_int(__ldg(splat2d + GS_SPLAT * g + 14));
}

// stores a record: A = (mx, my, a, beta), B = (gamma, opacity, depth, qcut), C = (r, g, b,
// 1 - opacity) (colour written separately when c == nullptr), D = (b, c, touched slot, 0)
// Per-Gaussian binning record: one aligned 32-B sector (the preprocess writes it whole, so no
// partial-sector write reaches HBM): tile rectangle (x0, x1, y0, y1), the keep bits of a small
// rectangle (candidate order) or the bitmap base of a large one, and the kept-tile count (< 0:
// -(1 + huge slot); the large-footprint cull's countdown while it runs).  gs_frame.rect points
// at the array (gs_frame.keep_bits / kept are unused).
struct __align__(32) BinRec {
    int4 rect;
    unsigned long long bits;
    int kept;
    int pad_;
};
__device__ __forceinline__ BinRec *bin_rec(const gs_frame &f) { return reinterpret_cast<BinRec *>(f.rect); }
__device__ __forceinline__ void bin_store(const gs_frame &f, int64_t i, int4 rect, unsigned long long bits, int kept) {
    int4 *p = reinterpret_cast<int4 *>(bin_rec(f) + i);
    p[0] = rect;
    p[1] = make_int4((int)(uint32_t)bits, (int)(uint32_t)(bits >> 32), kept, 0);
}

__device__ __forceinline__ void splat_store(float *splat2d, int64_t g, float mx, float my, double ca, double cb,
                                            double cc, float op, float z, float qcut) {
    float4 *s = reinterpret_cast<float4 *>(splat2d) + GS_SPLAT / 4 * g;
    const bool ok = ca > 0.0;
    const double beta = ok ? cb / ca : 0.0, gamma = ok ? (ca * cc - cb * cb) / ca : 0.0;
    s[0] = make_float4(mx, my, (float)ca, (float)beta);
    s[1] = make_float4((float)gamma, op, z, qcut);
    s[3] = make_float4((float)cb, (float)cc, 0.0f, 0.0f);
}

// ---------------------------------------------------------------------------
// Sparse Adam (R/rasterizer.py:707-725), shared by the fused chain + Adam and the packed updates

// One Adam element (R/rasterizer.py:715-725): m, v moments, bias-corrected step
// lr * (m / bc1) / (sqrt(v / bc2) + 1e-15).  rbc1 = 1/bc1, rbc2 = 1/bc2 are per-row constants.
// The square root and the reciprocal are single MUFU instructions (sqrt.approx / rcp.approx,
// ~1 ulp; the denominator is >= 1e-15, never subnormal): with IEEE sqrtf and __frcp_rn
// (Newton steps + fix-up paths) the 59 updates per row were a third of the fused chain+Adam
// kernel's instructions.
__device__ __forceinline__ float adam_one(float p, float &m, float &v, float g, float lr, float rbc1, float rbc2) {
    m = 0.9f * m + 0.1f * g;
    v = 0.999f * v + 0.001f * g * g;
    const float den = fast_sqrt(v * rbc2) + 1e-15f;
    return p - (lr * (m * rbc1)) * fast_rcp(den);
}

// Two Adam elements with paired fp32 instructions (FFMA2 / FMUL2 / FADD2): the operations and
// their order of adam_one as compiled (m = fma(0.9, m, 0.1 g), v = fma(0.999, v, (0.001 g) g),
// p - (lr (m rbc1)) rcp(den) as one fused multiply-add), so the results are the same bits.
__device__ __forceinline__ void adam_two(float p0, float p1, float &m0, float &m1, float &v0, float &v1, float g0,
                                         float g1, float lr0, float lr1, float rbc1, float rbc2, float &o0,
                                         float &o1) {
    const float2 g = make_float2(g0, g1);
    const float2 m = __ffma2_rn(make_float2(0.9f, 0.9f), make_float2(m0, m1), __fmul2_rn(g, make_float2(0.1f, 0.1f)));
    const float2 gg = __fmul2_rn(__fmul2_rn(g, make_float2(0.001f, 0.001f)), g);
    const float2 v = __ffma2_rn(make_float2(0.999f, 0.999f), make_float2(v0, v1), gg);
    const float2 vr = __fmul2_rn(v, make_float2(rbc2, rbc2));
    const float2 den = __fadd2_rn(make_float2(fast_sqrt(vr.x), fast_sqrt(vr.y)), make_float2(1e-15f, 1e-15f));
    const float2 nstep = __fmul2_rn(make_float2(-lr0, -lr1), __fmul2_rn(m, make_float2(rbc1, rbc1)));
    const float2 o = __ffma2_rn(nstep, make_float2(fast_rcp(den.x), fast_rcp(den.y)), make_float2(p0, p1));
    m0 = m.x;
    m1 = m.y;
    v0 = v.x;
    v1 = v.y;
    o0 = o.x;
    o1 = o.y;
}

// ---------------------------------------------------------------------------
// Deterministic accumulation.  Screen-space gradient rows (and the pose gradient) are sums of
// per-tile (per-Gaussian) partials in an order the scheduler picks.  Each partial is split
// exactly into two 64-bit fixed-point words, hi in units of 2^-24 and lo in units of 2^-64, and
// added with integer atomics: integer addition is associative, so the sums -- and everything
// computed from them -- are bit-identical run to run (the reference pins this,
// T/test_rasterizer.py:153-162, T/test_mapper.py:399-410).  Range |x| < 2^38 per partial and
// 2^39 per sum (hi); lo holds < 2^40 per partial, so 2^23 partials fit; bits below 2^-64 are
// truncated (deterministically).
constexpr double FX_HI_SCALE = 16777216.0;             // 2^24
constexpr double FX_LO_SCALE = 1099511627776.0;        // 2^40
constexpr double FX_HI_UNIT = 1.0 / 16777216.0;        // 2^-24
constexpr double FX_LO_UNIT = 5.421010862427522e-20;   // 2^-64

__device__ __forceinline__ void fx_split(double x, long long &hi, long long &lo) {
    double d = x * FX_HI_SCALE;
    d = fmin(fmax(d, -4.0e18), 4.0e18);  // saturate (never reached by a finite gradient of this path)
    const double h = trunc(d);
    hi = (long long)h;
    lo = (long long)trunc((d - h) * FX_LO_SCALE);  // d - h is exact
}

__device__ __forceinline__ void fx_atomic_add(long long *dst, double x) {
    long long hi, lo;
    fx_split(x, hi, lo);
    if (hi) atomicAdd(reinterpret_cast<unsigned long long *>(dst), (unsigned long long)hi);
    if (lo) atomicAdd(reinterpret_cast<unsigned long long *>(dst) + 1, (unsigned long long)lo);
}

__device__ __forceinline__ double fx_value(long long hi, long long lo) {
    return (double)hi * FX_HI_UNIT + (double)lo * FX_LO_UNIT;
}

// Exact cull of every candidate tile of a Gaussian's rectangle (ty-major, then tx, as
// R/rasterizer.py:113-122 enumerates them).  Returns the kept count; bit c of `bits` is the
// result for candidate c < 64 (the emit pass recomputes candidates >= 64).
__device__ __forceinline__ int cull_rect(float mx, float my, float ca, float cb, float cc, float qcut, int4 r,
                                         int width, int height, uint64_t &bits) {
    int count = 0, c = 0;
    bits = 0ull;
    for (int ty = r.z; ty <= r.w; ty++) {
        const int y0 = ty * GS_TILE, y1 = min(y0 + GS_TILE - 1, height - 1);
        for (int tx = r.x; tx <= r.y; tx++, c++) {
            const int x0 = tx * GS_TILE, x1 = min(x0 + GS_TILE - 1, width - 1);
            if (tile_keep(mx, my, ca, cb, cc, qcut, x0, x1, y0, y1)) {
                count++;
                if (c < 64) bits |= 1ull << c;
            }
        }
    }
    return count;
}

// c / n for 0 <= c < 2^16 and 1 <= n <= 2^16 from rn = 1/n (fp32): (c + 0.5) / n lies >= 0.5 / n
// from every integer, far beyond the ~1e-7 relative error of the product, so the floor is exact
// (an integer divide by a runtime value is a ~20-instruction subroutine)
__device__ __forceinline__ int small_div(int c, float rn) { return (int)(((float)c + 0.5f) * rn); }

// Per-tile bucket counts (tile_scratch[0..T)) and smallest keys of one Gaussian's kept
// candidates (cull bits of cull_rect, ncand <= GS_SMALL_CAND); fire-and-forget reductions.
__device__ __forceinline__ void count_kept_tiles(int32_t *cnt, unsigned long long *minkey, unsigned long long key, int4 r,
                                                 uint64_t bits, int tiles_x) {
    const int nx = r.y - r.x + 1;
    const float rnx = __frcp_rn((float)nx);
    while (bits) {
        const int c = __ffsll((long long)bits) - 1;
        bits &= bits - 1ull;
        const int dy = small_div(c, rnx), t = (r.z + dy) * tiles_x + r.x + c - dy * nx;
        atomicAdd(&cnt[t], 1);
        atomicMin(&minkey[t], key);  // smallest bucketed key of the tile (lazy lists)
    }
}

// Append flagged ids to a list with one atomic per warp (all 32 lanes must call).
__device__ __forceinline__ int warp_append(bool flag, int32_t id, int32_t *counter, int32_t *list) {
    const unsigned m = __ballot_sync(0xffffffffu, flag);
    if (!m) return -1;
    const unsigned lane = threadIdx.x & 31u;
    const int leader = __ffs(m) - 1;
    int base = 0;
    if ((int)lane == leader) base = atomicAdd(counter, __popc(m));
    base = __shfl_sync(0xffffffffu, base, leader);
    const int at = base + __popc(m & ((1u << lane) - 1u));
    if (flag) list[at] = id;
    return flag ? at : -1;
}

// warp_append onto the touched list, recording each appended Gaussian's slot in its splat record
__device__ __forceinline__ void touched_append(const gs_frame &f, bool flag, int32_t g) {
    const int at = warp_append(flag, g, &f.counters[GS_CNT_TOUCHED], f.touched_list);
    if (at >= 0) splat_set_slot(f.splat2d, g, at);
}

}  // namespace gs
