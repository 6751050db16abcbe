// preprocess.cu -- projection / EWA covariance / SH colour / tile rectangle (sm_100a).
//
// R/gaussians.py:180-215 (project), R/rasterizer.py:445-452 (sigmoid, camera->Gaussian view
// directions, eval_sh R/gaussians.py:102-111), R/rasterizer.py:84-102 + 183-194 (influence
// radius and tile rectangle).  One thread per Gaussian; each warp stages its 32 parameter
// rows (256 B each) through shared memory with coalesced float4 loads, skipping the SH
// columns of Gaussians behind the near plane.
#include "common.cuh"

namespace gs {

constexpr int PP_WARPS = 4;
constexpr int PP_THREADS = PP_WARPS * 32;
constexpr int ROWP = 65;  // padded smem row (conflict-free per-lane column reads)

__global__ void __launch_bounds__(PP_THREADS) preprocess_kernel(gs_frame f, const float *__restrict__ params,
                                                                const gs_view *__restrict__ view) {
    __shared__ float srow[PP_WARPS][32][ROWP];
    __shared__ gs_camera scam;
    if (threadIdx.x == 0) scam = view->cam;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t base = ((int64_t)blockIdx.x * PP_WARPS + warp) * 32;
    const int64_t i = base + lane;
    const int64_t n = f.n;
    const gs_camera &cam = scam;

    // 1) own row's first float4 (pos) -> near-plane test (R/gaussians.py:188-191)
    bool near_ok = false;
    if (i < n) {
        float4 p0 = __ldg(reinterpret_cast<const float4 *>(params + i * GS_ROW));
        float z = (p0.x * cam.rot_cw[6] + p0.y * cam.rot_cw[7] + p0.z * cam.rot_cw[8]) + cam.trans_cw[2];
        near_ok = z > GS_NEAR_CLIP;
        srow[warp][lane][0] = p0.x;
        srow[warp][lane][1] = p0.y;
        srow[warp][lane][2] = p0.z;
        srow[warp][lane][3] = p0.w;
    }
    const unsigned need = __ballot_sync(0xffffffffu, near_ok);
    // 2) cooperative, coalesced load of the remaining 15 float4 of every needed row
#pragma unroll
    for (int j = 0; j < 15; j++) {
        int k = lane + 32 * j;       // 0..479
        int r = k / 15, c4 = 1 + k % 15;
        if ((need >> r) & 1u) {
            float4 v = __ldg(reinterpret_cast<const float4 *>(params + (base + r) * GS_ROW + 4 * c4));
            srow[warp][r][4 * c4 + 0] = v.x;
            srow[warp][r][4 * c4 + 1] = v.y;
            srow[warp][r][4 * c4 + 2] = v.z;
            srow[warp][r][4 * c4 + 3] = v.w;
        }
    }
    __syncwarp();
    if (i >= n) return;
    const float *p = srow[warp][lane];
    f.touched[i] = 0;
    float4 *s2 = reinterpret_cast<float4 *>(f.splat2d) + 3 * i;
    float4 *cv = reinterpret_cast<float4 *>(f.cov2d) + i;
    int4 *rc = reinterpret_cast<int4 *>(f.rect) + i;
    const uint64_t inactive_key = (0xffffffffull << 32) | (uint64_t)i;
    if (!near_ok) {
        float z = (p[0] * cam.rot_cw[6] + p[1] * cam.rot_cw[7] + p[2] * cam.rot_cw[8]) + cam.trans_cw[2];
        s2[0] = make_float4(0.f, 0.f, 0.f, 0.f);
        s2[1] = make_float4(0.f, 0.f, z, 0.f);
        s2[2] = make_float4(0.f, 0.f, 0.f, 0.f);
        *cv = make_float4(0.f, 0.f, 0.f, -1.f);
        *rc = make_int4(0, -1, 0, -1);
        f.valid[i] = 0;
        f.keys_a[i] = inactive_key;
        return;
    }
    Projected pr;
    project_full(p, cam, pr);
    float op = 1.0f / (1.0f + expf(-p[10]));
    // view direction camera->Gaussian (R/rasterizer.py:447-451) and SH colour
    float u0 = p[0] - cam.center[0], u1 = p[1] - cam.center[1], u2 = p[2] - cam.center[2];
    float un = sqrtf(u0 * u0 + u1 * u1 + u2 * u2);
    if (un < 1e-12f) un = 1.0f;
    float b[16];
    sh_basis(u0 / un, u1 / un, u2 / un, b);
    float col[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        float acc = 0.0f;
#pragma unroll
        for (int k = 0; k < 15; k++) acc += b[k + 1] * p[14 + 3 * k + c];
        float pre = b[0] * p[11 + c] + acc + 0.5f;
        col[c] = pre > 0.0f ? pre : 0.0f;
    }
    int4 rect = make_int4(0, -1, 0, -1);
    float qcut = 0.0f, radius = -1.0f;
    bool active = pr.valid && tile_rect(pr.c00, pr.c01, pr.c11, op, pr.mx, pr.my, f.width, f.height, f.tiles_x,
                                         f.tiles_y, rect, qcut, radius);
    if (!active) rect = make_int4(0, -1, 0, -1);
    s2[0] = make_float4(pr.mx, pr.my, pr.ca, pr.cb);
    s2[1] = make_float4(pr.cc, op, pr.mu[2], qcut);
    s2[2] = make_float4(col[0], col[1], col[2], 0.0f);
    *cv = make_float4(pr.c00, pr.c01, pr.c11, radius);
    *rc = rect;
    f.valid[i] = pr.valid ? 1 : 0;
    f.keys_a[i] = active ? (((uint64_t)__float_as_uint(pr.mu[2]) << 32) | (uint64_t)i) : inactive_key;
}

// gs_project: full projection records for the project() API (R/gaussians.py:180-215)
__global__ void project_kernel(const float *__restrict__ params, int64_t n, const gs_camera *__restrict__ camp,
                               float *mu_cam, float *mean2d, float *cov2d, float *conic, float *depth,
                               uint8_t *valid, float *jproj, float *mmat, float *cov3d) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    gs_camera cam = *camp;
    float p[10];
#pragma unroll
    for (int k = 0; k < 10; k++) p[k] = params[i * GS_ROW + k];
    Projected pr;
    project_full(p, cam, pr);
    if (mu_cam)
        for (int k = 0; k < 3; k++) mu_cam[3 * i + k] = pr.mu[k];
    if (mean2d) {
        mean2d[2 * i] = pr.mx;
        mean2d[2 * i + 1] = pr.my;
    }
    if (cov2d) {
        cov2d[4 * i] = pr.c00;
        cov2d[4 * i + 1] = pr.c01;
        cov2d[4 * i + 2] = pr.c01;
        cov2d[4 * i + 3] = pr.c11;
    }
    if (conic) {
        conic[3 * i] = pr.ca;
        conic[3 * i + 1] = pr.cb;
        conic[3 * i + 2] = pr.cc;
    }
    if (depth) depth[i] = pr.mu[2];
    if (valid) valid[i] = pr.valid;
    if (jproj)
        for (int k = 0; k < 6; k++) jproj[6 * i + k] = pr.J[k];
    if (mmat)
        for (int k = 0; k < 6; k++) mmat[6 * i + k] = pr.M[k];
    if (cov3d)
        for (int k = 0; k < 9; k++) cov3d[9 * i + k] = pr.S[k];
}

__global__ void eval_sh_kernel(const float *__restrict__ sh_low, const float *__restrict__ sh_high,
                               const float *__restrict__ dirs, int64_t n, float *colors, float *preclamp) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    float b[16];
    sh_basis(dirs[3 * i], dirs[3 * i + 1], dirs[3 * i + 2], b);
    for (int c = 0; c < 3; c++) {
        float acc = 0.0f;
        for (int k = 0; k < 15; k++) acc += b[k + 1] * sh_high[45 * i + 3 * k + c];
        float pre = b[0] * sh_low[3 * i + c] + acc + 0.5f;
        if (preclamp) preclamp[3 * i + c] = pre;
        if (colors) colors[3 * i + c] = pre > 0.0f ? pre : 0.0f;
    }
}

// stand-alone cull_tiles(): pack caller-provided 2D splats into the frame
__global__ void pack_kernel(gs_frame f, const float *__restrict__ mean2d, const float *__restrict__ conic,
                            const float *__restrict__ cov2d3, const float *__restrict__ opac,
                            const float *__restrict__ depth, const uint8_t *__restrict__ valid,
                            const float *__restrict__ colors) {
    int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= f.n) return;
    float mx = mean2d[2 * i], my = mean2d[2 * i + 1];
    float c00 = cov2d3[3 * i], c01 = cov2d3[3 * i + 1], c11 = cov2d3[3 * i + 2];
    float o = opac[i];
    int4 rect = make_int4(0, -1, 0, -1);
    float qcut = 0.f, radius = -1.f;
    bool v = valid[i] != 0;
    bool active = v && tile_rect(c00, c01, c11, o, mx, my, f.width, f.height, f.tiles_x, f.tiles_y, rect, qcut, radius);
    if (!active) rect = make_int4(0, -1, 0, -1);
    float4 *s2 = reinterpret_cast<float4 *>(f.splat2d) + 3 * i;
    s2[0] = make_float4(mx, my, conic[3 * i], conic[3 * i + 1]);
    s2[1] = make_float4(conic[3 * i + 2], o, depth[i], qcut);
    s2[2] = colors ? make_float4(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2], 0.f) : make_float4(0.f, 0.f, 0.f, 0.f);
    reinterpret_cast<float4 *>(f.cov2d)[i] = make_float4(c00, c01, c11, radius);
    reinterpret_cast<int4 *>(f.rect)[i] = rect;
    f.valid[i] = v;
    f.touched[i] = 0;
    f.keys_a[i] = active ? (((uint64_t)__float_as_uint(depth[i]) << 32) | (uint64_t)i) : ((0xffffffffull << 32) | (uint64_t)i);
}

__global__ void lidar_compact_kernel(const float *__restrict__ sparse, int64_t npx, int32_t *idx, float *z,
                                     int32_t *k_out) {
    // ordered compaction (single block, so the K-list keeps pixel order like np.flatnonzero)
    __shared__ int32_t s_base;
    __shared__ int32_t s_warp[32];
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int64_t off = 0; off < npx; off += blockDim.x) {
        int64_t p = off + threadIdx.x;
        float v = p < npx ? sparse[p] : 0.0f;
        bool hit = v > 0.0f;
        unsigned m = __ballot_sync(0xffffffffu, hit);
        if (lane == 0) s_warp[warp] = __popc(m);
        __syncthreads();
        int before = 0, total = 0;
        for (int w = 0; w < nwarps; w++) {
            if (w < warp) before += s_warp[w];
            total += s_warp[w];
        }
        int pos = s_base + before + __popc(m & ((1u << lane) - 1u));
        if (hit) {
            idx[pos] = (int32_t)p;
            z[pos] = v;
        }
        __syncthreads();
        if (threadIdx.x == 0) s_base += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) *k_out = s_base;
}

}  // namespace gs

using namespace gs;

extern "C" int gs_preprocess(const gs_frame *f, const float *params, const gs_view *view, void *stream) {
    if (!f || !params || !view) {
        set_error("gs_preprocess: null argument");
        return GS_ERR_ARG;
    }
    if (f->n == 0) return GS_OK;
    int64_t warps = (f->n + 31) / 32;
    int blocks = (int)((warps + PP_WARPS - 1) / PP_WARPS);
    preprocess_kernel<<<blocks, PP_THREADS, 0, (cudaStream_t)stream>>>(*f, params, view);
    return check_launch("preprocess_kernel");
}

extern "C" int gs_project(const float *params, int64_t n, const gs_camera *cam, float *mu_cam, float *mean2d,
                          float *cov2d, float *conic, float *depth, uint8_t *valid, float *jproj, float *mmat,
                          float *cov3d, void *stream) {
    if (n == 0) return GS_OK;
    project_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(
        params, n, cam, mu_cam, mean2d, cov2d, conic, depth, valid, jproj, mmat, cov3d);
    return check_launch("project_kernel");
}

extern "C" int gs_eval_sh(const float *sh_low, const float *sh_high, const float *dirs, int64_t n, float *colors,
                          float *preclamp, void *stream) {
    if (n == 0) return GS_OK;
    eval_sh_kernel<<<(unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(sh_low, sh_high, dirs, n, colors,
                                                                                   preclamp);
    return check_launch("eval_sh_kernel");
}

extern "C" int gs_pack_splats(const gs_frame *f, const float *mean2d, const float *conic, const float *cov2d3,
                              const float *opacity, const float *depth, const uint8_t *valid, const float *colors,
                              void *stream) {
    if (f->n == 0) return GS_OK;
    pack_kernel<<<(unsigned)((f->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*f, mean2d, conic, cov2d3, opacity,
                                                                                   depth, valid, colors);
    return check_launch("pack_kernel");
}

extern "C" int gs_lidar_compact(const float *sparse_depth, int32_t width, int32_t height, int32_t *idx, float *z,
                                int32_t *k_out, void *stream) {
    lidar_compact_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(sparse_depth, (int64_t)width * height, idx, z, k_out);
    return check_launch("lidar_compact_kernel");
}
