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
// dL/dalpha formula, R/rasterizer.py:392-404).  Per entry, the 256 pixel contributions are
// reduced with a transposed warp butterfly (10 fields in 16 shuffles), merged across warps
// with shared-memory atomics, and added to the per-Gaussian gradient rows with one vector
// atomic per 4 floats.
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

// transposed butterfly: on return lane l holds the warp sum of field (l >> 1) (fields >= 10 are 0)
__device__ __forceinline__ float warp_sum16(float v[16]) {
    const unsigned lane = threadIdx.x & 31u;
#pragma unroll
    for (int k = 0; k < 8; k++) {
        const bool hi = lane & 16u;
        const float send = hi ? v[k] : v[k + 8];
        const float keep = hi ? v[k + 8] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
#pragma unroll
    for (int k = 0; k < 4; k++) {
        const bool hi = lane & 8u;
        const float send = hi ? v[k] : v[k + 4];
        const float keep = hi ? v[k + 4] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 8);
    }
#pragma unroll
    for (int k = 0; k < 2; k++) {
        const bool hi = lane & 4u;
        const float send = hi ? v[k] : v[k + 2];
        const float keep = hi ? v[k + 2] : v[k];
        v[k] = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    }
    {
        const bool hi = lane & 2u;
        const float send = hi ? v[0] : v[1];
        const float keep = hi ? v[1] : v[0];
        v[0] = keep + __shfl_xor_sync(0xffffffffu, send, 2);
    }
    return v[0] + __shfl_xor_sync(0xffffffffu, v[0], 1);
}

__global__ void __launch_bounds__(RT) render_bwd_kernel(gs_frame f) {
    __shared__ float4 s_a[RT];
    __shared__ float4 s_b[RT];
    __shared__ float4 s_c[RT];
    __shared__ int s_g[RT];
    __shared__ float s_acc[RT][GS_G2D];
    __shared__ int s_max;
    const int tile = blockIdx.x;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int px = tx * GS_TILE + (threadIdx.x & 15), py = ty * GS_TILE + (threadIdx.x >> 4);
    const bool inside = px < f.width && py < f.height;
    const int start = f.tile_offsets[tile], stop = f.tile_offsets[tile + 1];
    if (stop == start) return;
    const unsigned lane = threadIdx.x & 31u;
    const float fx = (float)px, fy = (float)py;
    float T = 1.0f, gc0 = 0.f, gc1 = 0.f, gc2 = 0.f, gd = 0.f, go = 0.f;
    int cnt = 0;
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    if (inside) {
        const int64_t p = (int64_t)py * f.width + px;
        T = f.trans[p];
        cnt = f.n_contrib[p];
        gc0 = f.g_color[3 * p];
        gc1 = f.g_color[3 * p + 1];
        gc2 = f.g_color[3 * p + 2];
        gd = f.g_depth[p];
        go = f.g_opac[p];
        atomicMax(&s_max, cnt);
    }
    __syncthreads();
    const int max_cnt = s_max;
    float S0 = 0.f, S1 = 0.f, S2 = 0.f, Sd = 0.f, So = 0.f;
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    for (int b_end = start + max_cnt; b_end > start; b_end -= RT) {
        const int b0 = max(start, b_end - RT);
        const int nb = b_end - b0;
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            const int g = f.entry_splat[b0 + threadIdx.x];
            s_g[threadIdx.x] = g;
            s_a[threadIdx.x] = __ldg(sp + 3 * g);
            s_b[threadIdx.x] = __ldg(sp + 3 * g + 1);
            s_c[threadIdx.x] = __ldg(sp + 3 * g + 2);
#pragma unroll
            for (int k = 0; k < GS_G2D; k++) s_acc[threadIdx.x][k] = 0.0f;
        }
        __syncthreads();
        for (int j = nb - 1; j >= 0; j--) {
            const int le = b0 + j - start;
            const bool contrib = le < cnt;
            if (!__any_sync(0xffffffffu, contrib)) continue;
            float v[16];
#pragma unroll
            for (int k = 0; k < 16; k++) v[k] = 0.0f;
            if (contrib) {
                const float4 A = s_a[j], B = s_b[j], C = s_c[j];
                const float dx = fx - A.x, dy = fy - A.y;
                const float ca = A.z, cb = A.w, cc = B.x, op = B.y, dep = B.z;
                float araw, alpha, om;
                alpha_oma(op, C.w, quad(ca, cb, cc, dx, dy), araw, alpha, om);
                const float Tb = T / om;
                const float w = alpha * Tb;
                v[6] = w * gc0;
                v[7] = w * gc1;
                v[8] = w * gc2;
                v[9] = w * gd;
                const float dl = Tb * (C.x * gc0 + C.y * gc1 + C.z * gc2 + dep * gd + go) -
                                 (S0 * gc0 + S1 * gc1 + S2 * gc2 + Sd * gd + So * go) / om;
                if (araw <= GS_ALPHA_CLAMP) {
                    const float gq = dl * (-0.5f * alpha);
                    v[5] = dl * (alpha / op);
                    v[2] = gq * dx * dx;
                    v[3] = gq * 2.0f * dx * dy;
                    v[4] = gq * dy * dy;
                    v[0] = gq * (-2.0f * (ca * dx + cb * dy));
                    v[1] = gq * (-2.0f * (cb * dx + cc * dy));
                }
                S0 += C.x * w;
                S1 += C.y * w;
                S2 += C.z * w;
                Sd += dep * w;
                So += w;
                T = Tb;
            }
            const float sum = warp_sum16(v);
            const unsigned fld = lane >> 1;
            if (!(lane & 1u) && fld < 10u && sum != 0.0f) atomicAdd(&s_acc[j][fld], sum);
        }
        __syncthreads();
        if ((int)threadIdx.x < nb) {
            // cross-tile accumulation in FP64: a large Gaussian collects thousands of per-tile
            // partial sums of mixed sign (near-plane splats cover every tile of the image)
            const float *a = s_acc[threadIdx.x];
            double *dst = f.g2d + (int64_t)s_g[threadIdx.x] * GS_G2D;
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
    render_bwd_kernel<<<T, RT, 0, (cudaStream_t)stream>>>(*f);
    return check_launch("render_bwd_kernel");
}
