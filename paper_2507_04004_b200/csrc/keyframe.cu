// keyframe.cu -- keyframe preparation on the device (sm_100a).
//
// The inputs of the hot path, built where they are consumed instead of on the host per keyframe:
//   gs_project_points  R/mapper.py:69-81 project_points, fused with bilinear_color (:84-98) and
//                      expand_map's opacity test (:218-230): thread per LiDAR point, FP64
//                      projection of the fp32 point (np.round = round-half-even = rint);
//   gs_zbuffer         R/mapper.py:101-107 zbuffer_project: nearest point per pixel by an atomicMin
//                      on the fp32 depth bits (positive floats order as their bit patterns), then
//                      0 where empty -- the dense sparse-depth map gs_lidar_compact turns into the
//                      LiDAR K-list;
//   gs_init_rows       R/gaussians.py:227-248 init_from_points: parameter rows of new Gaussians.
// All three are streaming, HBM-bound passes (12-28 B per point, 4-8 B per pixel).
#include "common.cuh"

namespace gs {

struct PointProj {
    double u, v, z;
    int ui, vi;
    bool inside;
};

__device__ __forceinline__ PointProj project_point(const float *__restrict__ p, const gs_camera &cam) {
    PointProj o;
    double pc[3];
#pragma unroll
    for (int r = 0; r < 3; r++)
        pc[r] = ((double)p[0] * cam.rot_cw[3 * r] + (double)p[1] * cam.rot_cw[3 * r + 1] +
                 (double)p[2] * cam.rot_cw[3 * r + 2]) + (double)cam.trans_cw[r];
    o.z = pc[2];
    const bool front = o.z > (double)GS_NEAR_CLIP;
    const double zs = front ? o.z : 1.0;
    o.u = (double)cam.fx * pc[0] / zs + (double)cam.cx;
    o.v = (double)cam.fy * pc[1] / zs + (double)cam.cy;
    const double ur = rint(o.u), vr = rint(o.v);  // pixel centres sit at integer coordinates
    o.inside = front && ur >= 0.0 && ur < (double)cam.width && vr >= 0.0 && vr < (double)cam.height;
    o.ui = o.inside ? (int)ur : (int)fmax(fmin(ur, 2147483647.0), -2147483648.0);
    o.vi = o.inside ? (int)vr : (int)fmax(fmin(vr, 2147483647.0), -2147483648.0);
    return o;
}

__global__ void project_points_kernel(const float *__restrict__ points, int64_t m, const gs_camera *__restrict__ camp,
                                      const float *__restrict__ image, const float *__restrict__ opacity, float tau,
                                      float *u, float *v, int32_t *ui, int32_t *vi, float *z, uint8_t *flags,
                                      float *colors) {
    pdl_wait();
    __shared__ gs_camera cam;
    if (threadIdx.x == 0) cam = *camp;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const PointProj o = project_point(points + 3 * i, cam);
        if (u) u[i] = (float)o.u;
        if (v) v[i] = (float)o.v;
        if (ui) ui[i] = o.ui;
        if (vi) vi[i] = o.vi;
        if (z) z[i] = (float)o.z;
        const int w = cam.width, h = cam.height;
        if (flags) {
            // expand_map (R/mapper.py:222-225): fresh = inside and the rendered opacity < tau
            const bool fresh = opacity && o.inside && opacity[(int64_t)o.vi * w + o.ui] < tau;
            flags[i] = (uint8_t)((o.inside ? 1 : 0) | (fresh ? 2 : 0));
        }
        if (colors && image) {  // bilinear_color (R/mapper.py:84-98)
            const double x = fmin(fmax(o.u, 0.0), (double)(w - 1)), y = fmin(fmax(o.v, 0.0), (double)(h - 1));
            const int x0 = w > 1 ? min(max((int)floor(x), 0), w - 2) : 0;
            const int y0 = h > 1 ? min(max((int)floor(y), 0), h - 2) : 0;
            const double fx = x - x0, fy = y - y0;
            const int x1 = min(x0 + 1, w - 1), y1 = min(y0 + 1, h - 1);
            const float *c00 = image + 3 * ((int64_t)y0 * w + x0), *c01 = image + 3 * ((int64_t)y0 * w + x1);
            const float *c10 = image + 3 * ((int64_t)y1 * w + x0), *c11 = image + 3 * ((int64_t)y1 * w + x1);
#pragma unroll
            for (int c = 0; c < 3; c++) {
                const double top = (double)c00[c] * (1.0 - fx) + (double)c01[c] * fx;
                const double bot = (double)c10[c] * (1.0 - fx) + (double)c11[c] * fx;
                colors[3 * i + c] = (float)(top * (1.0 - fy) + bot * fy);
            }
        }
    }
}

__global__ void zbuffer_fill_kernel(uint32_t *zbuf, int64_t npx) {
    pdl_wait();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x)
        zbuf[p] = 0xffffffffu;
}

__global__ void zbuffer_kernel(const float *__restrict__ points, int64_t m, const gs_camera *__restrict__ camp,
                               uint32_t *zbuf) {
    pdl_wait();
    __shared__ gs_camera cam;
    if (threadIdx.x == 0) cam = *camp;
    __syncthreads();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x) {
        const PointProj o = project_point(points + 3 * i, cam);
        // np.minimum.at(depth, (vi, ui), z): nearest wins; z > 0.01 so the fp32 bits order as values
        if (o.inside) atomicMin(zbuf + (int64_t)o.vi * cam.width + o.ui, __float_as_uint((float)o.z));
    }
}

__global__ void zbuffer_finish_kernel(const uint32_t *__restrict__ zbuf, float *depth, int64_t npx) {
    pdl_wait();
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
        const uint32_t b = zbuf[p];
        depth[p] = b == 0xffffffffu ? 0.0f : __uint_as_float(b);
    }
}

// init_from_points: log_scale = log(max(depth / focal, 1e-9)) (isotropic), identity quaternion,
// opacity logit(0.1), sh_low = (colour - 0.5) / C0, sh_high = 0; padding columns 0
__global__ void init_rows_kernel(const float *__restrict__ points, const float *__restrict__ colors,
                                 const float *__restrict__ depths, int64_t m, float focal, float *rows) {
    pdl_wait();
    const double C0 = 0.28209479177387814, logit01 = log(0.1 / 0.9);
    for (int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; idx < m * 16;
         idx += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = idx >> 4;
        const int c4 = (int)(idx & 15);
        float o[4];
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int col = 4 * c4 + e;
            double val = 0.0;
            if (col < 3) val = points[3 * i + col];
            else if (col < 6) val = log(fmax((double)depths[i] / (double)focal, 1e-9));
            else if (col == 6) val = 1.0;
            else if (col == 10) val = logit01;
            else if (col >= 11 && col < 14) val = ((double)colors[3 * i + col - 11] - 0.5) / C0;
            o[e] = (float)val;
        }
        reinterpret_cast<float4 *>(rows)[i * (GS_ROW / 4) + c4] = make_float4(o[0], o[1], o[2], o[3]);
    }
}

// 8-bit camera frame -> the fp32 target: v = k / 255 in FP64, rounded once -- bit-identical to
// the fp32 rounding of the reference's float64 image k / 255 (R/io_formats.py:52-57)
__global__ void u8_to_f32_kernel(const uint8_t *__restrict__ src, float *__restrict__ dst, int64_t n) {
    pdl_wait();
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = (float)((double)src[i] / 255.0);
}

}  // namespace gs

using namespace gs;

static unsigned grid_for(int64_t work) {
    const int64_t b = (work + 255) / 256;
    return (unsigned)(b < 8 * 148 ? (b > 0 ? b : 1) : 8 * 148);
}

extern "C" int gs_project_points(const float *points, int64_t m, const gs_camera *cam, const float *image,
                                 const float *opacity, float tau, float *u, float *v, int32_t *ui, int32_t *vi,
                                 float *z, uint8_t *flags, float *colors, void *stream) {
    if (m < 0 || (m > 0 && (!points || !cam))) {
        set_error("gs_project_points: bad arguments");
        return GS_ERR_ARG;
    }
    if (m == 0) return GS_OK;
    launch_pdl(project_points_kernel, grid_for(m), 256, 0, (cudaStream_t)stream, points, m, cam, image, opacity, tau, u, v,
                                                                        ui, vi, z, flags, colors);
    return check_launch("project_points_kernel");
}

extern "C" int gs_zbuffer(const float *points, int64_t m, const gs_camera *cam, int32_t width, int32_t height,
                          uint32_t *zbuf, float *depth, void *stream) {
    if (m < 0 || width <= 0 || height <= 0 || !zbuf || !depth || (m > 0 && (!points || !cam))) {
        set_error("gs_zbuffer: bad arguments");
        return GS_ERR_ARG;
    }
    const int64_t npx = (int64_t)width * height;
    cudaStream_t st = (cudaStream_t)stream;
    launch_pdl(zbuffer_fill_kernel, grid_for(npx), 256, 0, st, zbuf, npx);
    int rc = check_launch("zbuffer_fill_kernel");
    if (rc) return rc;
    if (m > 0) {
        launch_pdl(zbuffer_kernel, grid_for(m), 256, 0, st, points, m, cam, zbuf);
        if ((rc = check_launch("zbuffer_kernel"))) return rc;
    }
    launch_pdl(zbuffer_finish_kernel, grid_for(npx), 256, 0, st, zbuf, depth, npx);
    return check_launch("zbuffer_finish_kernel");
}

extern "C" int gs_init_rows(const float *points, const float *colors, const float *depths, int64_t m, float focal,
                            float *rows, void *stream) {
    if (m < 0 || (m > 0 && (!points || !colors || !depths || !rows))) {
        set_error("gs_init_rows: bad arguments");
        return GS_ERR_ARG;
    }
    if (m == 0) return GS_OK;
    launch_pdl(init_rows_kernel, grid_for(m * 16), 256, 0, (cudaStream_t)stream, points, colors, depths, m, focal, rows);
    return check_launch("init_rows_kernel");
}

extern "C" int gs_decode_u8(const uint8_t *src, float *dst, int64_t n, void *stream) {
    if (n < 0 || (n > 0 && (!src || !dst))) {
        set_error("gs_decode_u8: bad arguments");
        return GS_ERR_ARG;
    }
    if (n == 0) return GS_OK;
    launch_pdl(u8_to_f32_kernel, grid_for(n), 256, 0, (cudaStream_t)stream, src, dst, n);
    return check_launch("u8_to_f32_kernel");
}
