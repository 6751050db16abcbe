// track.cu -- photometric pose refinement on the device (sm_100a).
//
// R/odometry.py:305-336 photometric_refine: n_iters of (forward -> tracking loss (L1 + D-SSIM,
// lam 0.5) -> gradient masked by image-gradient and rendered-opacity gates -> pose gradient
// (gs_chain_pose, mode 3) -> Adam on the 6-vector -> left-multiplied SO(3) / translation update).
// The pose lives on the device (FP64 state) and is written into the view's camera after every
// step, so the whole loop is one graph-capturable launch sequence with no host round trip.
#include "common.cuh"

namespace gs {

// img_mask = hypot(np.gradient(gray)) > gate, gray = mean over the channels (R/odometry.py:314-316);
// np.gradient: central differences inside, one-sided at the borders
__global__ void track_mask_kernel(const float *__restrict__ image, int w, int h, float gate, uint8_t *mask) {
    pdl_wait();
    const int64_t npx = (int64_t)w * h;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
        const int y = (int)(p / w), x = (int)(p % w);
        auto gray = [&](int yy, int xx) {
            const float *c = image + 3 * ((int64_t)yy * w + xx);
            return ((double)c[0] + (double)c[1] + (double)c[2]) / 3.0;
        };
        double gx = 0.0, gy = 0.0;
        if (w > 1) {
            if (x == 0) gx = gray(y, 1) - gray(y, 0);
            else if (x == w - 1) gx = gray(y, w - 1) - gray(y, w - 2);
            else gx = 0.5 * (gray(y, x + 1) - gray(y, x - 1));
        }
        if (h > 1) {
            if (y == 0) gy = gray(1, x) - gray(0, x);
            else if (y == h - 1) gy = gray(h - 1, x) - gray(h - 2, x);
            else gy = 0.5 * (gray(y + 1, x) - gray(y - 1, x));
        }
        mask[p] = hypot(gx, gy) > (double)gate ? 1 : 0;
    }
}

// g_color *= img_mask & (opacity > gate) (R/odometry.py:325-326)
__global__ void track_grad_kernel(gs_frame f, const uint8_t *__restrict__ mask, float gate) {
    pdl_wait();
    const int64_t npx = (int64_t)f.width * f.height;
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < npx; p += (int64_t)gridDim.x * blockDim.x) {
        if (!(mask[p] && f.opacity[p] > gate)) {
            f.g_color[3 * p] = 0.0f;
            f.g_color[3 * p + 1] = 0.0f;
            f.g_color[3 * p + 2] = 0.0f;
        }
    }
}

// R/geometry.py:42-59 exp_so3 (Rodrigues, Taylor coefficients below 1e-8 rad)
__device__ void exp_so3(const double phi[3], double R[9]) {
    const double t2 = phi[0] * phi[0] + phi[1] * phi[1] + phi[2] * phi[2], t = sqrt(t2);
    const bool small = t < 1e-8;
    const double a = small ? 1.0 - t2 / 6.0 : sin(t) / t;
    const double b = small ? 0.5 - t2 / 24.0 : (1.0 - cos(t)) / t2;
    const double K[9] = {0.0, -phi[2], phi[1], phi[2], 0.0, -phi[0], -phi[1], phi[0], 0.0};
    for (int i = 0; i < 3; i++)
        for (int j = 0; j < 3; j++) {
            double kk = 0.0;
            for (int q = 0; q < 3; q++) kk += K[3 * i + q] * K[3 * q + j];
            R[3 * i + j] = (i == j ? 1.0 : 0.0) + a * K[3 * i + j] + b * kk;
        }
}

// state (FP64): rot_cw 0-8, trans_cw 9-11, m 12-17, v 18-23, iteration 24
__global__ void pose_adam_kernel(gs_view *view, double *state, const double *__restrict__ g, float lr) {
    pdl_wait();
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    const double it = state[24] + 1.0;
    state[24] = it;
    double step[6];
    for (int k = 0; k < 6; k++) {
        const double m = 0.9 * state[12 + k] + 0.1 * g[k];
        const double v = 0.999 * state[18 + k] + 0.001 * g[k] * g[k];
        state[12 + k] = m;
        state[18 + k] = v;
        const double mh = m / (1.0 - pow(0.9, it)), vh = v / (1.0 - pow(0.999, it));
        step[k] = -(double)lr * mh / (sqrt(vh) + 1e-15);
    }
    double E[9], Rn[9], tn[3];
    exp_so3(step + 3, E);
    for (int i = 0; i < 3; i++) {
        for (int j = 0; j < 3; j++)
            Rn[3 * i + j] = E[3 * i] * state[j] + E[3 * i + 1] * state[3 + j] + E[3 * i + 2] * state[6 + j];
        tn[i] = E[3 * i] * state[9] + E[3 * i + 1] * state[10] + E[3 * i + 2] * state[11] + step[i];
    }
    for (int k = 0; k < 9; k++) state[k] = Rn[k];
    for (int k = 0; k < 3; k++) state[9 + k] = tn[k];
    gs_camera &c = view->cam;
    for (int k = 0; k < 9; k++) c.rot_cw[k] = (float)Rn[k];
    for (int k = 0; k < 3; k++) {
        c.trans_cw[k] = (float)tn[k];
        c.center[k] = (float)-(Rn[k] * tn[0] + Rn[3 + k] * tn[1] + Rn[6 + k] * tn[2]);  // -R^T t
    }
}

}  // namespace gs

using namespace gs;

extern "C" int gs_track_mask(const float *image, int32_t width, int32_t height, float grad_gate, uint8_t *mask,
                             void *stream) {
    if (!image || !mask || width <= 0 || height <= 0) {
        set_error("gs_track_mask: bad arguments");
        return GS_ERR_ARG;
    }
    launch_pdl(track_mask_kernel, 4 * 148, 256, 0, (cudaStream_t)stream, image, width, height, grad_gate, mask);
    return check_launch("track_mask_kernel");
}

extern "C" int gs_track_grad(const gs_frame *f, const uint8_t *img_mask, float opac_gate, void *stream) {
    if (!f || !img_mask) {
        set_error("gs_track_grad: null argument");
        return GS_ERR_ARG;
    }
    launch_pdl(track_grad_kernel, 4 * 148, 256, 0, (cudaStream_t)stream, *f, img_mask, opac_gate);
    return check_launch("track_grad_kernel");
}

extern "C" int gs_pose_adam(gs_view *view, double *state, const double *pose_grad, float lr, void *stream) {
    if (!view || !state || !pose_grad) {
        set_error("gs_pose_adam: null argument");
        return GS_ERR_ARG;
    }
    launch_pdl(pose_adam_kernel, 1, 32, 0, (cudaStream_t)stream, view, state, pose_grad, lr);
    return check_launch("pose_adam_kernel");
}
