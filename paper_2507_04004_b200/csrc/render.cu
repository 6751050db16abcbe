// render.cu -- front-to-back blend and its adjoint (sm_100a).
//
// Forward: R/rasterizer.py:226-293 (_forward_kernel).  One CTA per 16x16 tile, one thread
// per pixel; the tile's depth-ordered entries are staged 256 at a time in shared memory.
// Reference semantics: no per-pixel alpha < 1/255 skip, alpha clamped at 0.99, the entry that
// drives T below 1e-4 is included and counted in n_contrib.
//
// Backward: R/rasterizer.py:296-435 (_backward_kernel + _reduce_entries).  Per pixel the
// blend is replayed back to front from the final transmittance (T_before = T_after/(1-alpha)),
// accumulating suffix sums instead of the reference's checkpointed prefix replay (same
// dL/dalpha formula, R/rasterizer.py:392-404).  Two pixels per thread; per entry their
// contributions are summed in registers, reduced across the warp with a transposed butterfly
// (10 fields in 12 shuffles), merged across the 4 warps with shared-memory atomics, and added
// to the per-Gaussian FP64 gradient rows once per tile.
#include "common.cuh"

namespace gs {

constexpr int RT = 256;  // threads per tile CTA = pixels per tile
constexpr float NEG_HALF_LOG2E = -0.5f * GS_LOG2E;

__device__ __forceinline__ float quad(float ca, float cb, float cc, float dx, float dy) {
    return ca * dx * dx + 2.0f * cb * dx * dy + cc * dy * dy;
}

// alpha = min(o e^{-q/2}, 0.99) (R/rasterizer.py:270-272) and 1 - alpha.  1 - alpha is formed
// with one rounding (FMA) and is exactly 0.01 on the clamp, so the transmittance product does
// not pick up the cancellation of 1 - 0.99f.  (omo = 1 - o is carried in the splat record for
// the higher-accuracy variant 1 - o e = (1 - e) + (1 - o) e.)
__device__ __forceinline__ void alpha_oma(float op, float omo, float q, float &araw, float &alpha, float &oma) {
    (void)omo;
    const float e = exp2f(-0.5f * GS_LOG2E * q);
    araw = op * e;
    if (araw > GS_ALPHA_CLAMP) {
        alpha = GS_ALPHA_CLAMP;
        oma = 0.01f;
    } else {
        alpha = araw;
        oma = fmaf(-op, e, 1.0f);
    }
}

__global__ void __launch_bounds__(RT) render_fwd_kernel(gs_frame f, int early_stop) {
    __shared__ float4 s_a[RT];  // mx my ca cb
    __shared__ float4 s_b[RT];  // cc opacity depth -
    __shared__ float4 s_c[RT];  // r g b -
    const int tile = blockIdx.x;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int px = tx * GS_TILE + (threadIdx.x & 15), py = ty * GS_TILE + (threadIdx.x >> 4);
    const bool inside = px < f.width && py < f.height;
    const int start = f.tile_offsets[tile], stop = f.tile_offsets[tile + 1];
    const float fx = (float)px, fy = (float)py;
    // opacity is accumulated as sum(w) (== 1 - T exactly in real arithmetic): 1 - T in fp32
    // cancels for nearly transparent pixels, and the depth loss divides by it
    float T = 1.0f, c0 = 0.0f, c1 = 0.0f, c2 = 0.0f, dsum = 0.0f, osum = 0.0f;
    int cnt = 0;
    bool done = !inside;
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    for (int b = start; b < stop; b += RT) {
        if (__syncthreads_count(done) == RT) break;
        const int e = b + threadIdx.x;
        if (e < stop) {
            const int g = f.entry_splat[e];
            s_a[threadIdx.x] = __ldg(sp + 3 * g);
            s_b[threadIdx.x] = __ldg(sp + 3 * g + 1);
            s_c[threadIdx.x] = __ldg(sp + 3 * g + 2);
        }
        __syncthreads();
        if (!done) {
            const int nb = min(RT, stop - b);
            for (int j = 0; j < nb; j++) {
                const float4 A = s_a[j], B = s_b[j], C = s_c[j];
                const float dx = fx - A.x, dy = fy - A.y;
                float araw, alpha, oma;
                alpha_oma(B.y, C.w, quad(A.z, A.w, B.x, dx, dy), araw, alpha, oma);
                const float w = alpha * T;
                c0 += C.x * w;
                c1 += C.y * w;
                c2 += C.z * w;
                dsum += B.z * w;
                osum += w;
                T *= oma;
                if (early_stop && T < GS_EARLY_STOP_T) {
                    done = true;
                    cnt = b - start + j + 1;
                    break;
                }
            }
            if (!done) cnt = b - start + nb;
        }
    }
    if (inside) {
        const int64_t p = (int64_t)py * f.width + px;
        f.color[3 * p] = c0;
        f.color[3 * p + 1] = c1;
        f.color[3 * p + 2] = c2;
        f.depth[p] = dsum;
        f.opacity[p] = osum;
        f.trans[p] = T;
        f.n_contrib[p] = cnt;
    }
}

// Transposed butterfly over 10 fields in 12 shuffles: on return, an even lane L holds the warp
// sum of field reduce10_field(L) (or -1: nothing to store; field 2 is held by 4 lanes, only one
// stores it).  Stages: xor 16 splits the fields 5/5, xor 8 splits 2/2 and sums the fifth
// everywhere, xor 4 splits 1/1 (+ the fifth), xor 2 separates the fifth, xor 1 completes.
__device__ __forceinline__ float reduce10(const float v[10]) {
    const unsigned lane = threadIdx.x & 31u;
    const bool h = lane & 16u, b3 = lane & 8u, b2 = lane & 4u, b1 = lane & 2u;
    float u[5];
#pragma unroll
    for (int k = 0; k < 5; k++) {
        const float send = h ? v[k] : v[k + 5];
        const float keep = h ? v[k + 5] : v[k];
        u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float w[3];
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const float send = b3 ? u[k] : u[k + 3];
        const float keep = b3 ? u[k + 3] : u[k];
        w[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
    w[2] = u[2] + __shfl_xor_sync(0xffffffffu, u[2], 8);
    float z0, z1;
    {
        const float send = b2 ? w[0] : w[1];
        const float keep = b2 ? w[1] : w[0];
        z0 = keep + __shfl_xor_sync(0xffffffffu, send, 4);
        z1 = w[2] + __shfl_xor_sync(0xffffffffu, w[2], 4);
    }
    const float send = b1 ? z0 : z1;
    const float keep = b1 ? z1 : z0;
    const float y = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    return y + __shfl_xor_sync(0xffffffffu, y, 1);
}

__device__ __forceinline__ int reduce10_field(unsigned lane) {
    if (lane & 1u) return -1;
    const int h5 = (lane & 16u) ? 5 : 0;
    if (!(lane & 2u)) return h5 + ((lane & 8u) ? 3 : 0) + ((lane & 4u) ? 1 : 0);
    return (lane & 12u) ? -1 : h5 + 2;
}

// One pixel's contribution to the 10 screen-space gradient fields of an entry, back-to-front
// replay step (R/rasterizer.py:365-410): undoes the entry's 1 - alpha on T, accumulates into v
// and advances the suffix sums S.
struct BwdPixel {
    float fx, fy, T, gc0, gc1, gc2, gd, go, S0, S1, S2, Sd, So;
    int cnt;
};

__device__ __forceinline__ void bwd_step(BwdPixel &p, const float4 &A, const float4 &B, const float4 &C, float v[10]) {
    const float dx = p.fx - A.x, dy = p.fy - A.y;
    const float ca = A.z, cb = A.w, cc = B.x, op = B.y, dep = B.z;
    const float e = exp2f(NEG_HALF_LOG2E * quad(ca, cb, cc, dx, dy));
    const float araw = op * e;
    const bool clamped = araw > GS_ALPHA_CLAMP;
    const float alpha = clamped ? GS_ALPHA_CLAMP : araw;
    const float om = clamped ? 0.01f : fmaf(-op, e, 1.0f);
    const float rom = __frcp_rn(om);
    const float Tb = p.T * rom;
    const float w = alpha * Tb;
    v[6] += w * p.gc0;
    v[7] += w * p.gc1;
    v[8] += w * p.gc2;
    v[9] += w * p.gd;
    const float dl = Tb * (C.x * p.gc0 + C.y * p.gc1 + C.z * p.gc2 + dep * p.gd + p.go) -
                     (p.S0 * p.gc0 + p.S1 * p.gc1 + p.S2 * p.gc2 + p.Sd * p.gd + p.So * p.go) * rom;
    if (!clamped) {  // no alpha-chain gradient on the 0.99 clamp (R/rasterizer.py:399-404)
        const float gq = dl * (-0.5f * alpha);
        v[5] += dl * e;  // d alpha / d opacity = e
        v[2] += gq * dx * dx;
        v[3] += gq * 2.0f * dx * dy;
        v[4] += gq * dy * dy;
        v[0] += gq * (-2.0f * (ca * dx + cb * dy));
        v[1] += gq * (-2.0f * (cb * dx + cc * dy));
    }
    p.S0 += C.x * w;
    p.S1 += C.y * w;
    p.S2 += C.z * w;
    p.Sd += dep * w;
    p.So += w;
    p.T = Tb;
}

// 128 threads per 16x16 tile, two pixels per thread (rows y and y + 8): the two pixels'
// contributions are summed in registers before the warp reduction.
constexpr int BT = 128;

__global__ void __launch_bounds__(BT) render_bwd_kernel(gs_frame f) {
    __shared__ float4 s_a[RT];
    __shared__ float4 s_b[RT];
    __shared__ float4 s_c[RT];
    __shared__ int s_g[RT];
    __shared__ float s_acc[RT][10];
    __shared__ int s_max;
    const int tile = blockIdx.x;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int start = f.tile_offsets[tile], stop = f.tile_offsets[tile + 1];
    if (stop == start) return;
    const unsigned lane = threadIdx.x & 31u;
    const int fld = reduce10_field(lane);
    BwdPixel px[2];
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 2; k++) {
        BwdPixel &p = px[k];
        const int x = tx * GS_TILE + (threadIdx.x & 15), y = ty * GS_TILE + (threadIdx.x >> 4) + 8 * k;
        p.fx = (float)x;
        p.fy = (float)y;
        p.T = 1.0f;
        p.gc0 = p.gc1 = p.gc2 = p.gd = p.go = 0.0f;
        p.S0 = p.S1 = p.S2 = p.Sd = p.So = 0.0f;
        p.cnt = 0;
        if (x < f.width && y < f.height) {
            const int64_t q = (int64_t)y * f.width + x;
            p.T = f.trans[q];
            p.cnt = f.n_contrib[q];
            p.gc0 = f.g_color[3 * q];
            p.gc1 = f.g_color[3 * q + 1];
            p.gc2 = f.g_color[3 * q + 2];
            p.gd = f.g_depth[q];
            p.go = f.g_opac[q];
        }
    }
    atomicMax(&s_max, max(px[0].cnt, px[1].cnt));
    __syncthreads();
    const int max_cnt = s_max;
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    for (int b_end = start + max_cnt; b_end > start; b_end -= RT) {
        const int b0 = max(start, b_end - RT);
        const int nb = b_end - b0;
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += BT) {
            const int g = f.entry_splat[b0 + i];
            s_g[i] = g;
            s_a[i] = __ldg(sp + 3 * g);
            s_b[i] = __ldg(sp + 3 * g + 1);
            s_c[i] = __ldg(sp + 3 * g + 2);
#pragma unroll
            for (int k = 0; k < 10; k++) s_acc[i][k] = 0.0f;
        }
        __syncthreads();
        for (int j = nb - 1; j >= 0; j--) {
            const int le = b0 + j - start;
            const bool c0 = le < px[0].cnt, c1 = le < px[1].cnt;
            if (!__any_sync(0xffffffffu, c0 || c1)) continue;
            const float4 A = s_a[j], B = s_b[j], C = s_c[j];
            float v[10];
#pragma unroll
            for (int k = 0; k < 10; k++) v[k] = 0.0f;
            if (c0) bwd_step(px[0], A, B, C, v);
            if (c1) bwd_step(px[1], A, B, C, v);
            const float sum = reduce10(v);
            if (fld >= 0 && sum != 0.0f) atomicAdd(&s_acc[j][fld], sum);
        }
        __syncthreads();
        for (int i = threadIdx.x; i < nb; i += BT) {
            // cross-tile accumulation in FP64: a large Gaussian collects thousands of per-tile
            // partial sums of mixed sign (near-plane splats cover every tile of the image)
            const float *a = s_acc[i];
            double *dst = f.g2d + (int64_t)s_g[i] * GS_G2D;
#pragma unroll
            for (int k = 0; k < 10; k++)
                if (a[k] != 0.0f) atomicAdd(dst + k, (double)a[k]);
        }
    }
}

// zero the g2d rows of the touched Gaussians (12 doubles = 6 double2 per row)
__global__ void zero_g2d_kernel(gs_frame f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    if (i >= 6 * nt) return;
    const int64_t g = f.touched_list[i / 6];
    reinterpret_cast<double2 *>(f.g2d)[g * (GS_G2D / 2) + i % 6] = make_double2(0.0, 0.0);
}

}  // namespace gs

using namespace gs;

extern "C" int gs_render_fwd(const gs_frame *f, int32_t early_stop, void *stream) {
    const int T = f->tiles_x * f->tiles_y;
    if (T == 0) return GS_OK;
    render_fwd_kernel<<<T, RT, 0, (cudaStream_t)stream>>>(*f, early_stop);
    return check_launch("render_fwd_kernel");
}

extern "C" int gs_render_bwd(const gs_frame *f, void *stream) {
    const int T = f->tiles_x * f->tiles_y;
    if (T == 0) return GS_OK;
    if (f->n > 0) {  // each backward starts from zero gradients (backward_2d is a pure function)
        zero_g2d_kernel<<<(unsigned)((f->n * 6 + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*f);
        int rc = check_launch("zero_g2d_kernel");
        if (rc) return rc;
    }
    render_bwd_kernel<<<T, BT, 0, (cudaStream_t)stream>>>(*f);
    return check_launch("render_bwd_kernel");
}
