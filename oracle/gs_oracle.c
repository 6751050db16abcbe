/*
 * gs_oracle.c -- TEST INFRASTRUCTURE ONLY (parity checker + CPU baseline).
 *
 * A plain-C, float64 restatement of the reference's Gaussian map-optimisation
 * iteration (Gaussian-LIC2 CPU re-expression, /root/reference/pkg/src/splatslam),
 * plus an fp32 restatement of the bit-exact binning stages.  Only tests/,
 * __graft_entry__.smoke() and bench.py (cpu_baseline / --impl reference) may
 * load this library; the product path (paper_2507_04004_b200) never does.
 *
 * R/ = /root/reference/pkg/src/splatslam/.  Every function cites the reference
 * lines it follows.  Parity is pinned against tests/golden/ npz files produced by
 * tests/golden/make_golden.py from the reference itself.
 *
 * Compile with -ffp-contract=off (no FMA contraction): the float64 part then
 * evaluates the same IEEE operations, in the same order, as the reference's
 * numpy/numba code, and the fp32 part evaluates exactly the operation sequence
 * DESIGN.md specifies for the GPU's binning decision path.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define TILE 16
#define BUCKET 32
static const double CULL_ALPHA = 1.0 / 255.0;   /* R/rasterizer.py:42 */
static const double EARLY_STOP_T = 1e-4;        /* R/rasterizer.py:43 */
static const double DILATION = 0.3;             /* R/gaussians.py:33 */
static const double NEAR_CLIP = 0.01;           /* R/gaussians.py:34 */
static const double ALPHA_CLAMP = 0.99;         /* R/gaussians.py:35 */

/* SH constants, R/gaussians.py:24-30 */
static const double SH_C0 = 0.28209479177387814;
static const double SH_C1 = 0.4886025119029199;
static const double SH_C2[5] = {1.0925484305920792, -1.0925484305920792, 0.31539156525252005,
                                -1.0925484305920792, 0.5462742152960396};
static const double SH_C3[7] = {-0.5900435899266435, 2.890611442640554, -0.4570457994644658,
                                0.3731763325901154, -0.4570457994644658, 1.445305721320277,
                                -0.5900435899266435};

/* Parameter row layout: the order of GaussianMap.parameters() (R/gaussians.py:150-153)
 * flattened: pos 0..2, log_scale 3..5, quat 6..9 (wxyz), opacity_logit 10,
 * sh_low 11..13, sh_high 14..58 ((15,3) row-major). */
#define NP 59

typedef struct {
    int width, height;
    double fx, fy, cx, cy;
    double rot_cw[9]; /* row-major world->camera */
    double trans_cw[3];
} or_camera;

void or_set_threads(int n) {
#ifdef _OPENMP
    if (n > 0) omp_set_num_threads(n);
#else
    (void)n;
#endif
}

int or_get_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

void or_free(void *p) { free(p); }

/* ------------------------------------------------------------------------- */
/* SH basis and its gradient: R/gaussians.py:51-99                           */

static void sh_basis(const double d[3], double b[16]) {
    double x = d[0], y = d[1], z = d[2];
    double xx = x * x, yy = y * y, zz = z * z;
    double xy = x * y, yz = y * z, xz = x * z;
    b[0] = SH_C0;
    b[1] = -SH_C1 * y;
    b[2] = SH_C1 * z;
    b[3] = -SH_C1 * x;
    b[4] = SH_C2[0] * xy;
    b[5] = SH_C2[1] * yz;
    b[6] = SH_C2[2] * (2.0 * zz - xx - yy);
    b[7] = SH_C2[3] * xz;
    b[8] = SH_C2[4] * (xx - yy);
    b[9] = SH_C3[0] * y * (3.0 * xx - yy);
    b[10] = SH_C3[1] * xy * z;
    b[11] = SH_C3[2] * y * (4.0 * zz - xx - yy);
    b[12] = SH_C3[3] * z * (2.0 * zz - 3.0 * xx - 3.0 * yy);
    b[13] = SH_C3[4] * x * (4.0 * zz - xx - yy);
    b[14] = SH_C3[5] * z * (xx - yy);
    b[15] = SH_C3[6] * x * (xx - 3.0 * yy);
}

static void sh_basis_grad(const double d[3], double g[16][3]) {
    double x = d[0], y = d[1], z = d[2];
    memset(g, 0, sizeof(double) * 48);
    g[1][1] = -SH_C1;
    g[2][2] = SH_C1;
    g[3][0] = -SH_C1;
    g[4][0] = SH_C2[0] * y; g[4][1] = SH_C2[0] * x; g[4][2] = 0.0;
    g[5][0] = 0.0; g[5][1] = SH_C2[1] * z; g[5][2] = SH_C2[1] * y;
    g[6][0] = SH_C2[2] * (-2 * x); g[6][1] = SH_C2[2] * (-2 * y); g[6][2] = SH_C2[2] * (4 * z);
    g[7][0] = SH_C2[3] * z; g[7][1] = 0.0; g[7][2] = SH_C2[3] * x;
    g[8][0] = SH_C2[4] * (2 * x); g[8][1] = SH_C2[4] * (-2 * y); g[8][2] = 0.0;
    g[9][0] = SH_C3[0] * (6 * x * y); g[9][1] = SH_C3[0] * (3 * x * x - 3 * y * y); g[9][2] = 0.0;
    g[10][0] = SH_C3[1] * (y * z); g[10][1] = SH_C3[1] * (x * z); g[10][2] = SH_C3[1] * (x * y);
    g[11][0] = SH_C3[2] * (-2 * x * y); g[11][1] = SH_C3[2] * (4 * z * z - x * x - 3 * y * y);
    g[11][2] = SH_C3[2] * (8 * y * z);
    g[12][0] = SH_C3[3] * (-6 * x * z); g[12][1] = SH_C3[3] * (-6 * y * z);
    g[12][2] = SH_C3[3] * (6 * z * z - 3 * x * x - 3 * y * y);
    g[13][0] = SH_C3[4] * (4 * z * z - 3 * x * x - y * y); g[13][1] = SH_C3[4] * (-2 * x * y);
    g[13][2] = SH_C3[4] * (8 * x * z);
    g[14][0] = SH_C3[5] * (2 * x * z); g[14][1] = SH_C3[5] * (-2 * y * z); g[14][2] = SH_C3[5] * (x * x - y * y);
    g[15][0] = SH_C3[6] * (3 * x * x - 3 * y * y); g[15][1] = SH_C3[6] * (-6 * x * y); g[15][2] = 0.0;
}

/* eval_sh: R/gaussians.py:102-111.  colors = max(pre, 0); pre = B0*sh_low + sum_k B_k sh_high_k + 0.5 */
void or_eval_sh(int64_t n, const double *sh_low, const double *sh_high, const double *dirs,
                double *colors, double *preclamp) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double b[16];
        sh_basis(dirs + 3 * i, b);
        for (int c = 0; c < 3; c++) {
            double acc = 0.0;
            for (int k = 0; k < 15; k++) acc += b[k + 1] * sh_high[45 * i + 3 * k + c];
            double pre = b[0] * sh_low[3 * i + c] + acc + 0.5;
            preclamp[3 * i + c] = pre;
            colors[3 * i + c] = pre > 0.0 ? pre : 0.0;
        }
    }
}

/* quat_rotmats: R/gaussians.py:156-170 (normalised wxyz quaternion -> R) */
static void quat_rot(const double q0[4], double R[9]) {
    double nrm = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
    double w = q0[0] / nrm, x = q0[1] / nrm, y = q0[2] / nrm, z = q0[3] / nrm;
    R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
    R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
    R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

/* project: R/gaussians.py:180-215 (+ covariance_from :173-177).
 * Outputs (all optional except mean2d/conic/cov2d/depth/valid):
 *   mu_cam (n,3) mean2d (n,2) cov2d (n,4 = 00,01,10,11) conic (n,3) depth (n) valid (n)
 *   jproj (n,6) m (n,6) cov3d (n,9) */
void or_project(int64_t n, const double *params, const or_camera *cam, double *mu_cam,
                double *mean2d, double *cov2d, double *conic, double *depth, uint8_t *valid,
                double *jproj, double *mmat, double *cov3d) {
    const double *Rc = cam->rot_cw;
    const double *tc = cam->trans_cw;
    double fx = cam->fx, fy = cam->fy, cx = cam->cx, cy = cam->cy;
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const double *p = params + (size_t)NP * i;
        double mu[3];
        for (int r = 0; r < 3; r++) mu[r] = (p[0] * Rc[3 * r] + p[1] * Rc[3 * r + 1] + p[2] * Rc[3 * r + 2]) + tc[r];
        double z = mu[2];
        int v = z > NEAR_CLIP;
        double zs = v ? z : 1.0;
        double mx = fx * mu[0] / zs + cx, my = fy * mu[1] / zs + cy;
        double J[6] = {fx / zs, 0.0, -fx * mu[0] / (zs * zs), 0.0, fy / zs, -fy * mu[1] / (zs * zs)};
        double M[6];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                M[3 * r + c] = J[3 * r] * Rc[c] + J[3 * r + 1] * Rc[3 + c] + J[3 * r + 2] * Rc[6 + c];
        double R[9];
        quat_rot(p + 6, R);
        double s2[3] = {exp(2.0 * p[3]), exp(2.0 * p[4]), exp(2.0 * p[5])};
        double S[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) S[3 * a + b] = R[3 * a] * s2[0] * R[3 * b] + R[3 * a + 1] * s2[1] * R[3 * b + 1] +
                                                   R[3 * a + 2] * s2[2] * R[3 * b + 2];
        double MS[6];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                MS[3 * r + c] = M[3 * r] * S[c] + M[3 * r + 1] * S[3 + c] + M[3 * r + 2] * S[6 + c];
        double C[4];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++)
                C[2 * r + c] = MS[3 * r] * M[3 * c] + MS[3 * r + 1] * M[3 * c + 1] + MS[3 * r + 2] * M[3 * c + 2];
        C[0] += DILATION;
        C[3] += DILATION;
        double det = C[0] * C[3] - C[1] * C[1];
        v = v && (det > 1e-12) && isfinite(det);
        double dets = v ? det : 1.0;
        if (mu_cam) memcpy(mu_cam + 3 * i, mu, sizeof mu);
        mean2d[2 * i] = mx;
        mean2d[2 * i + 1] = my;
        memcpy(cov2d + 4 * i, C, sizeof C);
        conic[3 * i] = C[3] / dets;
        conic[3 * i + 1] = -C[1] / dets;
        conic[3 * i + 2] = C[0] / dets;
        depth[i] = z;
        valid[i] = (uint8_t)v;
        if (jproj) memcpy(jproj + 6 * i, J, sizeof J);
        if (mmat) memcpy(mmat + 6 * i, M, sizeof M);
        if (cov3d) memcpy(cov3d + 9 * i, S, sizeof S);
    }
}

/* forward preamble: R/rasterizer.py:445-452 (sigmoid opacity, camera->Gaussian dirs, SH) */
void or_preamble(int64_t n, const double *params, const or_camera *cam, double *opac, double *dirs,
                 double *u_norm, double *colors, double *preclamp) {
    const double *Rc = cam->rot_cw, *t = cam->trans_cw;
    double C[3];
    for (int c = 0; c < 3; c++) C[c] = -(Rc[c] * t[0] + Rc[3 + c] * t[1] + Rc[6 + c] * t[2]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        const double *p = params + (size_t)NP * i;
        opac[i] = 1.0 / (1.0 + exp(-p[10]));
        double u[3] = {p[0] - C[0], p[1] - C[1], p[2] - C[2]};
        double nrm = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        if (nrm < 1e-12) nrm = 1.0;
        u_norm[i] = nrm;
        double d[3] = {u[0] / nrm, u[1] / nrm, u[2] / nrm};
        memcpy(dirs + 3 * i, d, sizeof d);
        double b[16];
        sh_basis(d, b);
        for (int c = 0; c < 3; c++) {
            double acc = 0.0;
            for (int k = 0; k < 15; k++) acc += b[k + 1] * p[14 + 3 * k + c];
            double pre = b[0] * p[11 + c] + acc + 0.5;
            preclamp[3 * i + c] = pre;
            colors[3 * i + c] = pre > 0.0 ? pre : 0.0;
        }
    }
}

/* ------------------------------------------------------------------------- */
/* tile binning, float64: R/rasterizer.py:84-219                             */

static double exact_tile_min_q(double mx, double my, double ca, double cb, double cc, int x0, int x1, int y0,
                               int y1) { /* R/rasterizer.py:125-147 */
    double qmin = 1e300;
    for (int py = y0; py <= y1; py++) {
        double dy = py - my;
        double xs = mx - cb * dy / ca;
        double xfd = floor(xs);
        /* clamp before the int conversion (same candidate set as the reference) */
        if (xfd < x0 - 1) xfd = x0 - 1;
        if (xfd > x1 + 1) xfd = x1 + 1;
        int xf = (int)xfd;
        for (int k = 0; k < 2; k++) {
            int xc = xf + k;
            if (xc < x0) xc = x0;
            else if (xc > x1) xc = x1;
            double dx = xc - mx;
            double q = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy;
            if (q < qmin) qmin = q;
        }
    }
    return qmin;
}

typedef struct {
    int32_t tile;
    double depth;
    int64_t splat;
} pair64;

static int cmp_pair64(const void *a, const void *b) {
    const pair64 *x = (const pair64 *)a, *y = (const pair64 *)b;
    if (x->depth < y->depth) return -1;
    if (x->depth > y->depth) return 1;
    return (x->splat > y->splat) - (x->splat < y->splat);
}

/* cull_tiles: R/rasterizer.py:169-219.  cov2d is (n,4).  Returns E (entries) and a
 * malloc'd entry_splat (int64, E) through *out_entries; tile_offsets (T+1) is caller
 * memory.  The final order equals np.lexsort((splat, depth[splat], tile)). */
int64_t or_cull_tiles(int64_t n, const double *mean2d, const double *conic, const double *cov2d,
                      const double *opac, const double *depth, const uint8_t *valid, int width, int height,
                      int cull, int64_t **out_entries, int64_t *tile_offsets) {
    int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    int n_tiles = tiles_x * tiles_y;
    int32_t *tx0 = malloc(sizeof(int32_t) * (n > 0 ? n : 1) * 4);
    int32_t *tx1 = tx0 + n, *ty0 = tx1 + n, *ty1 = ty0 + n;
    int64_t *cnt = malloc(sizeof(int64_t) * (n + 1));
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        cnt[i] = 0;
        tx0[i] = 0; tx1[i] = -1; ty0[i] = 0; ty1[i] = -1;
        if (!valid[i]) continue;
        if (cull) {
            const double *C = cov2d + 4 * i;
            /* _max_eigenvalue :84-88 and influence_radius :91-102 */
            double half_tr = 0.5 * (C[0] + C[3]);
            double dd = 0.25 * (C[0] - C[3]) * (C[0] - C[3]) + C[1] * C[1];
            double lam = half_tr + sqrt(dd > 0.0 ? dd : 0.0);
            if (!(opac[i] * exp(0.0) > CULL_ALPHA)) continue;
            double r = sqrt(2.0 * log(255.0 * opac[i]) * lam) + 1e-6;
            if (!(r > 0)) continue;
            double mx = mean2d[2 * i], my = mean2d[2 * i + 1];
            if ((mx + r < 0) || (mx - r > width - 1) || (my + r < 0) || (my - r > height - 1)) continue;
            double f;
            f = floor((mx - r) / TILE); tx0[i] = f < 0 ? 0 : (f > tiles_x - 1 ? tiles_x - 1 : (int)f);
            f = floor((mx + r) / TILE); tx1[i] = f < 0 ? 0 : (f > tiles_x - 1 ? tiles_x - 1 : (int)f);
            f = floor((my - r) / TILE); ty0[i] = f < 0 ? 0 : (f > tiles_y - 1 ? tiles_y - 1 : (int)f);
            f = floor((my + r) / TILE); ty1[i] = f < 0 ? 0 : (f > tiles_y - 1 ? tiles_y - 1 : (int)f);
            /* _cull_pairs :150-166 per candidate tile */
            int64_t k = 0;
            for (int ty = ty0[i]; ty <= ty1[i]; ty++)
                for (int tx = tx0[i]; tx <= tx1[i]; tx++) {
                    int x0 = tx * TILE, y0 = ty * TILE;
                    int x1 = x0 + TILE - 1 < width - 1 ? x0 + TILE - 1 : width - 1;
                    int y1 = y0 + TILE - 1 < height - 1 ? y0 + TILE - 1 : height - 1;
                    double q = exact_tile_min_q(mx, my, conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], x0, x1, y0, y1);
                    double a = opac[i] * exp(-0.5 * q);
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    if (a >= CULL_ALPHA) k++;
                }
            cnt[i] = k;
        } else {
            tx0[i] = 0; tx1[i] = tiles_x - 1; ty0[i] = 0; ty1[i] = tiles_y - 1;
            cnt[i] = (int64_t)n_tiles;
        }
    }
    /* bucket by tile (counting sort), then sort each tile by (depth, splat) */
    int64_t *tile_cnt = calloc((size_t)n_tiles + 1, sizeof(int64_t));
    int64_t total = 0;
    for (int64_t i = 0; i < n; i++) total += cnt[i];
    pair64 *pairs = malloc(sizeof(pair64) * (total > 0 ? total : 1));
    /* emit in splat order (R/rasterizer.py:113-122), keeping only culled-in pairs */
    int64_t pos = 0;
    for (int64_t i = 0; i < n; i++) {
        if (cnt[i] == 0) continue;
        double mx = mean2d[2 * i], my = mean2d[2 * i + 1];
        for (int ty = ty0[i]; ty <= ty1[i]; ty++)
            for (int tx = tx0[i]; tx <= tx1[i]; tx++) {
                if (cull) {
                    int x0 = tx * TILE, y0 = ty * TILE;
                    int x1 = x0 + TILE - 1 < width - 1 ? x0 + TILE - 1 : width - 1;
                    int y1 = y0 + TILE - 1 < height - 1 ? y0 + TILE - 1 : height - 1;
                    double q = exact_tile_min_q(mx, my, conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], x0, x1, y0, y1);
                    double a = opac[i] * exp(-0.5 * q);
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    if (!(a >= CULL_ALPHA)) continue;
                }
                pairs[pos].tile = ty * tiles_x + tx;
                pairs[pos].depth = depth[i];
                pairs[pos].splat = i;
                tile_cnt[pairs[pos].tile + 1]++;
                pos++;
            }
    }
    for (int t = 0; t < n_tiles; t++) tile_cnt[t + 1] += tile_cnt[t];
    pair64 *sorted = malloc(sizeof(pair64) * (total > 0 ? total : 1));
    int64_t *fill = malloc(sizeof(int64_t) * (n_tiles + 1));
    memcpy(fill, tile_cnt, sizeof(int64_t) * (n_tiles + 1));
    for (int64_t e = 0; e < total; e++) sorted[fill[pairs[e].tile]++] = pairs[e];
#pragma omp parallel for schedule(dynamic, 4)
    for (int t = 0; t < n_tiles; t++)
        qsort(sorted + tile_cnt[t], (size_t)(tile_cnt[t + 1] - tile_cnt[t]), sizeof(pair64), cmp_pair64);
    int64_t *ent = malloc(sizeof(int64_t) * (total > 0 ? total : 1));
    for (int64_t e = 0; e < total; e++) ent[e] = sorted[e].splat;
    memcpy(tile_offsets, tile_cnt, sizeof(int64_t) * (n_tiles + 1));
    free(tx0); free(cnt); free(tile_cnt); free(pairs); free(sorted); free(fill);
    *out_entries = ent;
    return total;
}

/* ------------------------------------------------------------------------- */
/* fp32 binning restatement (bit-exact target for the GPU)                    */
/* Same stages as R/rasterizer.py:84-219 evaluated in IEEE fp32 with the      */
/* operation sequence of DESIGN.md "binning decision path"; the GPU kernels   */
/* evaluate the identical sequence with __f*_rn intrinsics.                   */

/* deterministic natural log for x >= 1 (fp32, explicit fmaf) */
static float det_logf(float x) {
    union { float f; uint32_t u; } b = {x};
    int e = (int)((b.u >> 23) & 0xffu) - 127;
    b.u = (b.u & 0x7fffffu) | 0x3f800000u;
    float m = b.f;
    if (m > 1.41421353816986083984375f) { m = m * 0.5f; e += 1; }
    float s = (m - 1.0f) / (m + 1.0f);
    float s2 = s * s;
    float p = fmaf(s2, 0.111111111938953399658203125f, 0.14285714924335479736328125f);
    p = fmaf(p, s2, 0.20000000298023223876953125f);
    p = fmaf(p, s2, 0.3333333432674407958984375f);
    p = fmaf(p, s2, 1.0f);
    float lm = (2.0f * s) * p;
    return fmaf((float)e, 0.693147182464599609375f, lm);
}

float or_det_logf(float x) { return det_logf(x); }

static float f32_tile_min_q(float mx, float my, float ca, float cb, float cc, int x0, int x1, int y0, int y1) {
    float qmin = INFINITY;
    for (int py = y0; py <= y1; py++) {
        float dy = (float)py - my;
        float xs = mx - (cb * dy) / ca;
        float lo = (float)(x0 - 1), hi = (float)(x1 + 1);
        if (!(xs >= lo)) xs = lo; /* also maps NaN to lo */
        if (xs > hi) xs = hi;
        int xf = (int)floorf(xs);
        for (int k = 0; k < 2; k++) {
            int xc = xf + k;
            if (xc < x0) xc = x0;
            else if (xc > x1) xc = x1;
            float dx = (float)xc - mx;
            float q = ((ca * dx) * dx + ((2.0f * cb) * dx) * dy) + (cc * dy) * dy;
            if (q < qmin) qmin = q;
        }
    }
    return qmin;
}

typedef struct {
    int32_t tile;
    uint32_t dbits;
    int32_t splat;
} pair32;

static int cmp_pair32(const void *a, const void *b) {
    const pair32 *x = (const pair32 *)a, *y = (const pair32 *)b;
    if (x->dbits != y->dbits) return x->dbits < y->dbits ? -1 : 1;
    return (x->splat > y->splat) - (x->splat < y->splat);
}

/* splat tile rectangle + cut (returns 0 when the splat has no candidate tile) */
static int f32_rect(const float *cov2d3, float o, float mx, float my, int width, int height, int tiles_x,
                    int tiles_y, int *rx0, int *rx1, int *ry0, int *ry1, float *qcut) {
    float c00 = cov2d3[0], c01 = cov2d3[1], c11 = cov2d3[2];
    float half_tr = 0.5f * (c00 + c11);
    float df = c00 - c11;
    float dd = 0.25f * (df * df) + c01 * c01;
    float lam = half_tr + sqrtf(dd > 0.0f ? dd : 0.0f);
    if (!(o > (float)(1.0 / 255.0))) return 0;
    float L = det_logf(255.0f * o);
    float r = sqrtf((2.0f * L) * lam) + 1e-6f;
    if (!(r > 0.0f)) return 0;
    if ((mx + r < 0.0f) || (mx - r > (float)(width - 1)) || (my + r < 0.0f) || (my - r > (float)(height - 1)))
        return 0;
    float f;
    f = floorf((mx - r) * 0.0625f); *rx0 = f < 0.0f ? 0 : (f > (float)(tiles_x - 1) ? tiles_x - 1 : (int)f);
    f = floorf((mx + r) * 0.0625f); *rx1 = f < 0.0f ? 0 : (f > (float)(tiles_x - 1) ? tiles_x - 1 : (int)f);
    f = floorf((my - r) * 0.0625f); *ry0 = f < 0.0f ? 0 : (f > (float)(tiles_y - 1) ? tiles_y - 1 : (int)f);
    f = floorf((my + r) * 0.0625f); *ry1 = f < 0.0f ? 0 : (f > (float)(tiles_y - 1) ? tiles_y - 1 : (int)f);
    *qcut = 2.0f * L;
    return 1;
}

/* splat2d inputs are the GPU's own fp32 values: mean2d (n,2), conic (n,3), cov2d (n,3 = 00,01,11),
 * opac (n), depth (n), valid (n).  Outputs: *out_entries (malloc'd int32, E), tile_offsets (T+1,
 * int32), touched (n, u8).  Keep rule (q-domain form of R/rasterizer.py:163-166):
 * qmin <= 2*ln(255 o). */
int64_t or_bin_f32(int64_t n, const float *mean2d, const float *conic, const float *cov2d, const float *opac,
                   const float *depth, const uint8_t *valid, int width, int height, int cull,
                   int32_t **out_entries, int32_t *tile_offsets, uint8_t *touched) {
    int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    int n_tiles = tiles_x * tiles_y;
    int64_t *cnt = malloc(sizeof(int64_t) * (n + 1));
    int32_t *rect = malloc(sizeof(int32_t) * 4 * (n > 0 ? n : 1));
    float *qc = malloc(sizeof(float) * (n > 0 ? n : 1));
#pragma omp parallel for schedule(dynamic, 256)
    for (int64_t i = 0; i < n; i++) {
        cnt[i] = 0;
        int32_t *R = rect + 4 * i;
        R[0] = 0; R[1] = -1; R[2] = 0; R[3] = -1;
        if (!valid[i]) continue;
        if (!cull) {
            R[0] = 0; R[1] = tiles_x - 1; R[2] = 0; R[3] = tiles_y - 1;
            cnt[i] = n_tiles;
            continue;
        }
        float mx = mean2d[2 * i], my = mean2d[2 * i + 1];
        if (!f32_rect(cov2d + 3 * i, opac[i], mx, my, width, height, tiles_x, tiles_y, &R[0], &R[1], &R[2], &R[3],
                      &qc[i])) {
            R[1] = -1; R[3] = -1;
            continue;
        }
        int64_t k = 0;
        for (int ty = R[2]; ty <= R[3]; ty++)
            for (int tx = R[0]; tx <= R[1]; tx++) {
                int x0 = tx * TILE, y0 = ty * TILE;
                int x1 = x0 + TILE - 1 < width - 1 ? x0 + TILE - 1 : width - 1;
                int y1 = y0 + TILE - 1 < height - 1 ? y0 + TILE - 1 : height - 1;
                float q = f32_tile_min_q(mx, my, conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], x0, x1, y0, y1);
                if (q <= qc[i]) k++;
            }
        cnt[i] = k;
    }
    int64_t total = 0;
    for (int64_t i = 0; i < n; i++) total += cnt[i];
    pair32 *pairs = malloc(sizeof(pair32) * (total > 0 ? total : 1));
    int64_t *tile_cnt = calloc((size_t)n_tiles + 1, sizeof(int64_t));
    int64_t pos = 0;
    for (int64_t i = 0; i < n; i++) {
        touched[i] = cnt[i] > 0;
        if (cnt[i] == 0) continue;
        int32_t *R = rect + 4 * i;
        float mx = mean2d[2 * i], my = mean2d[2 * i + 1];
        union { float f; uint32_t u; } db = {depth[i]};
        for (int ty = R[2]; ty <= R[3]; ty++)
            for (int tx = R[0]; tx <= R[1]; tx++) {
                if (cull) {
                    int x0 = tx * TILE, y0 = ty * TILE;
                    int x1 = x0 + TILE - 1 < width - 1 ? x0 + TILE - 1 : width - 1;
                    int y1 = y0 + TILE - 1 < height - 1 ? y0 + TILE - 1 : height - 1;
                    float q = f32_tile_min_q(mx, my, conic[3 * i], conic[3 * i + 1], conic[3 * i + 2], x0, x1, y0, y1);
                    if (!(q <= qc[i])) continue;
                }
                pairs[pos].tile = ty * tiles_x + tx;
                pairs[pos].dbits = db.u;
                pairs[pos].splat = (int32_t)i;
                tile_cnt[pairs[pos].tile + 1]++;
                pos++;
            }
    }
    for (int t = 0; t < n_tiles; t++) tile_cnt[t + 1] += tile_cnt[t];
    pair32 *sorted = malloc(sizeof(pair32) * (total > 0 ? total : 1));
    int64_t *fill = malloc(sizeof(int64_t) * (n_tiles + 1));
    memcpy(fill, tile_cnt, sizeof(int64_t) * (n_tiles + 1));
    for (int64_t e = 0; e < total; e++) sorted[fill[pairs[e].tile]++] = pairs[e];
#pragma omp parallel for schedule(dynamic, 4)
    for (int t = 0; t < n_tiles; t++)
        qsort(sorted + tile_cnt[t], (size_t)(tile_cnt[t + 1] - tile_cnt[t]), sizeof(pair32), cmp_pair32);
    int32_t *ent = malloc(sizeof(int32_t) * (total > 0 ? total : 1));
    for (int64_t e = 0; e < total; e++) ent[e] = sorted[e].splat;
    for (int t = 0; t <= n_tiles; t++) tile_offsets[t] = (int32_t)tile_cnt[t];
    free(cnt); free(rect); free(qc); free(pairs); free(tile_cnt); free(sorted); free(fill);
    *out_entries = ent;
    return total;
}

/* ------------------------------------------------------------------------- */
/* forward blend: R/rasterizer.py:226-293 (checkpoints omitted: the backward */
/* below replays the identical per-pixel recurrence instead)                  */

void or_forward_blend(const int64_t *entry_splat, const int64_t *tile_offsets, const double *mean2d,
                      const double *conic, const double *opac, const double *colors, const double *depth,
                      int width, int height, int early_stop, double *out_color, double *out_depth,
                      double *out_opac, double *out_trans, int32_t *n_contrib) {
    int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    int n_tiles = tiles_x * tiles_y;
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < n_tiles; t++) {
        int x0 = (t % tiles_x) * TILE, y0 = (t / tiles_x) * TILE;
        int tw = width - x0 < TILE ? width - x0 : TILE;
        int th = height - y0 < TILE ? height - y0 : TILE;
        int64_t start = tile_offsets[t], stop = tile_offsets[t + 1];
        for (int py = 0; py < th; py++)
            for (int px = 0; px < tw; px++) {
                double T = 1.0, acc[3] = {0, 0, 0}, accd = 0.0;
                int32_t cnt = 0;
                for (int64_t e = start; e < stop; e++) {
                    int64_t g = entry_splat[e];
                    double dy = (double)(y0 + py) - mean2d[2 * g + 1];
                    double dx = (double)(x0 + px) - mean2d[2 * g];
                    double ca = conic[3 * g], cb = conic[3 * g + 1], cc = conic[3 * g + 2];
                    double q = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy;
                    double a = opac[g] * exp(-0.5 * q);
                    if (a > ALPHA_CLAMP) a = ALPHA_CLAMP;
                    double w = a * T;
                    acc[0] += colors[3 * g] * w;
                    acc[1] += colors[3 * g + 1] * w;
                    acc[2] += colors[3 * g + 2] * w;
                    accd += depth[g] * w;
                    T *= 1.0 - a;
                    cnt = (int32_t)(e - start + 1);
                    if (early_stop && T < EARLY_STOP_T) break;
                }
                size_t p = (size_t)(y0 + py) * width + (x0 + px);
                out_color[3 * p] = acc[0];
                out_color[3 * p + 1] = acc[1];
                out_color[3 * p + 2] = acc[2];
                out_depth[p] = accd;
                out_opac[p] = 1.0 - T;
                out_trans[p] = T;
                n_contrib[p] = cnt;
            }
    }
}

/* backward blend: R/rasterizer.py:296-435.  Per-entry gradient slots accumulate over the
 * tile's pixels in pixel order (the staggered lane schedule visits a fixed entry's pixels
 * in increasing order), then reduce to splats in global entry order.  Output per splat:
 * g2d (n,10) = mean2d(2) conic(3) opacity(1) color(3) depth(1); touched (n). */
void or_backward_blend(int64_t n, const int64_t *entry_splat, const int64_t *tile_offsets,
                       const double *mean2d, const double *conic, const double *opac, const double *colors,
                       const double *depth, int width, int height, const double *g_color_img,
                       const double *g_depth_img, const double *g_opac_img, const double *total_rgb,
                       const double *total_d, const double *final_t, const int32_t *n_contrib, double *g2d,
                       uint8_t *touched) {
    int tiles_x = (width + TILE - 1) / TILE, tiles_y = (height + TILE - 1) / TILE;
    int n_tiles = tiles_x * tiles_y;
    int64_t E = tile_offsets[n_tiles];
    double *ge = calloc((size_t)(E > 0 ? E : 1) * 10, sizeof(double));
#pragma omp parallel for schedule(dynamic, 1)
    for (int t = 0; t < n_tiles; t++) {
        int x0 = (t % tiles_x) * TILE, y0 = (t / tiles_x) * TILE;
        int tw = width - x0 < TILE ? width - x0 : TILE;
        int th = height - y0 < TILE ? height - y0 : TILE;
        int64_t start = tile_offsets[t], stop = tile_offsets[t + 1];
        if (stop == start) continue;
        /* pixel order p = py*16 + px, i.e. row-major inside the tile */
        for (int py = 0; py < th; py++)
            for (int px = 0; px < tw; px++) {
                size_t pp = (size_t)(y0 + py) * width + (x0 + px);
                int32_t cnt = n_contrib[pp];
                double gc0 = g_color_img[3 * pp], gc1 = g_color_img[3 * pp + 1], gc2 = g_color_img[3 * pp + 2];
                double gd = g_depth_img[pp], go = g_opac_img[pp];
                double tr0 = total_rgb[3 * pp], tr1 = total_rgb[3 * pp + 1], tr2 = total_rgb[3 * pp + 2];
                double td = total_d[pp], fin = final_t[pp];
                double T = 1.0, pre0 = 0, pre1 = 0, pre2 = 0, pred = 0;
                for (int64_t e = start; e < stop && (e - start) < cnt; e++) {
                    int64_t g = entry_splat[e];
                    double mx = mean2d[2 * g], my = mean2d[2 * g + 1];
                    double dx = (double)(x0 + px) - mx;
                    double dy = (double)(y0 + py) - my;
                    double ca = conic[3 * g], cb = conic[3 * g + 1], cc = conic[3 * g + 2];
                    double op = opac[g];
                    double q = ca * dx * dx + 2.0 * cb * dx * dy + cc * dy * dy;
                    double araw = op * exp(-0.5 * q);
                    double a = araw <= ALPHA_CLAMP ? araw : ALPHA_CLAMP;
                    double w = a * T;
                    double c0 = colors[3 * g], c1 = colors[3 * g + 1], c2 = colors[3 * g + 2];
                    double dep = depth[g];
                    double *s = ge + 10 * e;
                    s[6] += w * gc0;
                    s[7] += w * gc1;
                    s[8] += w * gc2;
                    s[9] += w * gd;
                    double tnext = T * (1.0 - a);
                    double s0 = tr0 - (pre0 + c0 * w);
                    double s1 = tr1 - (pre1 + c1 * w);
                    double s2 = tr2 - (pre2 + c2 * w);
                    double sd = td - (pred + dep * w);
                    double so = tnext - fin;
                    double dl = (T * (c0 * gc0 + c1 * gc1 + c2 * gc2 + dep * gd + go) -
                                 (s0 * gc0 + s1 * gc1 + s2 * gc2 + sd * gd + so * go) / (1.0 - a));
                    if (araw <= ALPHA_CLAMP) {
                        double gq = dl * (-0.5 * a);
                        s[5] += dl * (a / op);
                        s[2] += gq * dx * dx;
                        s[3] += gq * 2.0 * dx * dy;
                        s[4] += gq * dy * dy;
                        s[0] += gq * (-2.0 * (ca * dx + cb * dy));
                        s[1] += gq * (-2.0 * (cb * dx + cc * dy));
                    }
                    pre0 += c0 * w;
                    pre1 += c1 * w;
                    pre2 += c2 * w;
                    pred += dep * w;
                    T = tnext;
                }
            }
    }
    memset(g2d, 0, sizeof(double) * 10 * (size_t)n);
    memset(touched, 0, (size_t)n);
    for (int64_t e = 0; e < E; e++) { /* _reduce_entries :413-435 */
        int64_t g = entry_splat[e];
        touched[g] = 1;
        g2d[10 * g + 0] += ge[10 * e + 0];
        g2d[10 * g + 1] += ge[10 * e + 1];
        g2d[10 * g + 2] += ge[10 * e + 2];
        g2d[10 * g + 3] += ge[10 * e + 3];
        g2d[10 * g + 4] += ge[10 * e + 4];
        g2d[10 * g + 5] += ge[10 * e + 5];
        g2d[10 * g + 6] += ge[10 * e + 6];
        g2d[10 * g + 7] += ge[10 * e + 7];
        g2d[10 * g + 8] += ge[10 * e + 8];
        g2d[10 * g + 9] += ge[10 * e + 9];
    }
    free(ge);
}

/* ------------------------------------------------------------------------- */
/* chain rule to attributes: R/rasterizer.py:559-644 (+ _quat_partials :490-499) */

static void quat_partials(const double q0[4], double dR[4][9]) {
    double nrm = sqrt(q0[0] * q0[0] + q0[1] * q0[1] + q0[2] * q0[2] + q0[3] * q0[3]);
    double w = q0[0] / nrm, x = q0[1] / nrm, y = q0[2] / nrm, z = q0[3] / nrm;
    double dw[9] = {0, -z, y, z, 0, -x, -y, x, 0};
    double dx[9] = {0, y, z, y, -2 * x, -w, z, w, -2 * x};
    double dy[9] = {-2 * y, x, w, x, 0, z, -w, z, -2 * y};
    double dz[9] = {-2 * z, -w, x, w, -2 * z, y, x, y, 0};
    for (int k = 0; k < 9; k++) {
        dR[0][k] = 2.0 * dw[k];
        dR[1][k] = 2.0 * dx[k];
        dR[2][k] = 2.0 * dy[k];
        dR[3][k] = 2.0 * dz[k];
    }
}

/* grads (n, 59) rows; only touched rows are written, others zeroed. */
/* pose_parts (nullable, n x 6): per-Gaussian terms of the 6-dof pose gradient (rho, theta) on
 * the left tangent of T_cw (R/rasterizer.py:646-657); the caller sums them over touched ids. */
void or_chain_pose(int64_t n, const double *params, const or_camera *cam, const double *g2d,
                   const uint8_t *touched, double *grads, double *pose_parts);
void or_chain(int64_t n, const double *params, const or_camera *cam, const double *g2d, const uint8_t *touched,
              double *grads) {
    or_chain_pose(n, params, cam, g2d, touched, grads, NULL);
}
void or_chain_pose(int64_t n, const double *params, const or_camera *cam, const double *g2d,
                   const uint8_t *touched, double *grads, double *pose_parts) {
    const double *Rc = cam->rot_cw, *tc = cam->trans_cw;
    double fx = cam->fx, fy = cam->fy;
    double Cc[3];
    for (int c = 0; c < 3; c++) Cc[c] = -(Rc[c] * tc[0] + Rc[3 + c] * tc[1] + Rc[6 + c] * tc[2]);
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        double *G = grads + (size_t)NP * i;
        memset(G, 0, sizeof(double) * NP);
        if (pose_parts) memset(pose_parts + (size_t)6 * i, 0, sizeof(double) * 6);
        if (!touched[i]) continue;
        const double *p = params + (size_t)NP * i;
        const double *g = g2d + 10 * i;
        /* recompute the projection records (R/gaussians.py:188-202) */
        double mu[3];
        for (int r = 0; r < 3; r++) mu[r] = (p[0] * Rc[3 * r] + p[1] * Rc[3 * r + 1] + p[2] * Rc[3 * r + 2]) + tc[r];
        double z = mu[2];
        double zs = z > NEAR_CLIP ? z : 1.0;
        double J[6] = {fx / zs, 0.0, -fx * mu[0] / (zs * zs), 0.0, fy / zs, -fy * mu[1] / (zs * zs)};
        double M[6];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                M[3 * r + c] = J[3 * r] * Rc[c] + J[3 * r + 1] * Rc[3 + c] + J[3 * r + 2] * Rc[6 + c];
        double R[9];
        quat_rot(p + 6, R);
        double s[3] = {exp(p[3]), exp(p[4]), exp(p[5])};
        double s2[3] = {exp(2.0 * p[3]), exp(2.0 * p[4]), exp(2.0 * p[5])};
        double S[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) S[3 * a + b] = R[3 * a] * s2[0] * R[3 * b] + R[3 * a + 1] * s2[1] * R[3 * b + 1] +
                                                   R[3 * a + 2] * s2[2] * R[3 * b + 2];
        double MS[6], C2[4];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 3; c++)
                MS[3 * r + c] = M[3 * r] * S[c] + M[3 * r + 1] * S[3 + c] + M[3 * r + 2] * S[6 + c];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++)
                C2[2 * r + c] = MS[3 * r] * M[3 * c] + MS[3 * r + 1] * M[3 * c + 1] + MS[3 * r + 2] * M[3 * c + 2];
        C2[0] += DILATION;
        C2[3] += DILATION;
        double det = C2[0] * C2[3] - C2[1] * C2[1];
        double cm[4] = {C2[3] / det, -C2[1] / det, -C2[1] / det, C2[0] / det};
        /* conic -> cov2d gradient :584-592 */
        double gcm[4] = {g[2], 0.5 * g[3], 0.5 * g[3], g[4]};
        double t1[4], gcov[4];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) t1[2 * r + c] = cm[2 * r] * gcm[c] + cm[2 * r + 1] * gcm[2 + c];
        for (int r = 0; r < 2; r++)
            for (int c = 0; c < 2; c++) gcov[2 * r + c] = -(t1[2 * r] * cm[c] + t1[2 * r + 1] * cm[2 + c]);
        /* :595-597 */
        double gS[9], gM[6], gJ[6], tmp[6];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++) tmp[3 * a + b] = gcov[2 * a] * M[b] + gcov[2 * a + 1] * M[3 + b];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) gS[3 * a + b] = M[a] * tmp[b] + M[3 + a] * tmp[3 + b];
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                gM[3 * a + b] = 2.0 * (tmp[3 * a] * S[b] + tmp[3 * a + 1] * S[3 + b] + tmp[3 * a + 2] * S[6 + b]);
        for (int a = 0; a < 2; a++)
            for (int b = 0; b < 3; b++)
                gJ[3 * a + b] = gM[3 * a] * Rc[3 * b] + gM[3 * a + 1] * Rc[3 * b + 1] + gM[3 * a + 2] * Rc[3 * b + 2];
        /* :600-611 */
        double z2 = z * z, z3 = z * z * z;
        double gx = gJ[2] * (-fx / z2);
        double gy = gJ[5] * (-fy / z2);
        double gz = (gJ[0] * (-fx / z2) + gJ[4] * (-fy / z2) + gJ[2] * (2.0 * fx * mu[0] / z3) +
                     gJ[5] * (2.0 * fy * mu[1] / z3));
        gx += g[0] * fx / z;
        gy += g[1] * fy / z;
        gz += (-g[0] * fx * mu[0] / z2 - g[1] * fy * mu[1] / z2);
        gz += g[9];
        for (int c = 0; c < 3; c++) G[c] = gx * Rc[c] + gy * Rc[3 + c] + gz * Rc[6 + c];
        /* :613-626 */
        double gN[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++)
                gN[3 * a + b] = 2.0 * (gS[3 * a] * R[b] * s[b] + gS[3 * a + 1] * R[3 + b] * s[b] + gS[3 * a + 2] * R[6 + b] * s[b]);
        for (int j = 0; j < 3; j++) {
            double ds = R[j] * gN[j] + R[3 + j] * gN[3 + j] + R[6 + j] * gN[6 + j];
            G[3 + j] = ds * s[j];
        }
        double gR[9];
        for (int a = 0; a < 3; a++)
            for (int b = 0; b < 3; b++) gR[3 * a + b] = gN[3 * a + b] * s[b];
        double dR[4][9];
        quat_partials(p + 6, dR);
        double gqu[4];
        for (int k = 0; k < 4; k++) {
            double acc = 0.0;
            for (int m = 0; m < 9; m++) acc += gR[m] * dR[k][m];
            gqu[k] = acc;
        }
        double qn = sqrt(p[6] * p[6] + p[7] * p[7] + p[8] * p[8] + p[9] * p[9]);
        double qh[4] = {p[6] / qn, p[7] / qn, p[8] / qn, p[9] / qn};
        double dot = gqu[0] * qh[0] + gqu[1] * qh[1] + gqu[2] * qh[2] + gqu[3] * qh[3];
        for (int k = 0; k < 4; k++) G[6 + k] = (gqu[k] - qh[k] * dot) / qn;
        /* :629-630 */
        double o = 1.0 / (1.0 + exp(-p[10]));
        G[10] = g[5] * o * (1.0 - o);
        /* :633-644 */
        double u[3] = {p[0] - Cc[0], p[1] - Cc[1], p[2] - Cc[2]};
        double un = sqrt(u[0] * u[0] + u[1] * u[1] + u[2] * u[2]);
        if (un < 1e-12) un = 1.0;
        double d[3] = {u[0] / un, u[1] / un, u[2] / un};
        double b[16], bg[16][3];
        sh_basis(d, b);
        sh_basis_grad(d, bg);
        double gcol[3];
        for (int c = 0; c < 3; c++) {
            double acc = 0.0;
            for (int k = 0; k < 15; k++) acc += b[k + 1] * p[14 + 3 * k + c];
            double pre = b[0] * p[11 + c] + acc + 0.5;
            gcol[c] = pre > 0.0 ? g[6 + c] : 0.0;
        }
        for (int c = 0; c < 3; c++) G[11 + c] = b[0] * gcol[c];
        for (int k = 0; k < 15; k++)
            for (int c = 0; c < 3; c++) G[14 + 3 * k + c] = b[k + 1] * gcol[c];
        double gdir[3] = {0, 0, 0};
        for (int k = 0; k < 16; k++) {
            double sc = 0.0;
            for (int c = 0; c < 3; c++) sc += (k == 0 ? p[11 + c] : p[14 + 3 * (k - 1) + c]) * gcol[c];
            for (int dd = 0; dd < 3; dd++) gdir[dd] += bg[k][dd] * sc;
        }
        double gd = gdir[0] * d[0] + gdir[1] * d[1] + gdir[2] * d[2];
        double gu[3];
        for (int c = 0; c < 3; c++) {
            gu[c] = (gdir[c] - d[c] * gd) / un;
            G[c] += gu[c];
        }
        if (pose_parts) {
            /* :647-657 -- translation: g_mu_cam + R_cw gu (the view-direction path);
             * rotation: mu_cam x g_mu_cam + the covariance path through M = J R_cw with
             * X = (J^T gM) R_cw^T, theta += (X21 - X12, X02 - X20, X10 - X01) */
            double *P6 = pose_parts + (size_t)6 * i;
            const double gmu[3] = {gx, gy, gz};
            for (int r = 0; r < 3; r++) P6[r] = gmu[r] + (Rc[3 * r] * gu[0] + Rc[3 * r + 1] * gu[1] + Rc[3 * r + 2] * gu[2]);
            P6[3] = mu[1] * gz - mu[2] * gy;
            P6[4] = mu[2] * gx - mu[0] * gz;
            P6[5] = mu[0] * gy - mu[1] * gx;
            double grc[9], X[9];
            for (int a = 0; a < 3; a++)
                for (int b = 0; b < 3; b++) grc[3 * a + b] = J[a] * gM[b] + J[3 + a] * gM[3 + b];
            for (int a = 0; a < 3; a++)
                for (int k = 0; k < 3; k++)
                    X[3 * a + k] = grc[3 * a] * Rc[3 * k] + grc[3 * a + 1] * Rc[3 * k + 1] + grc[3 * a + 2] * Rc[3 * k + 2];
            P6[3] += X[7] - X[5];
            P6[4] += X[2] - X[6];
            P6[5] += X[3] - X[1];
        }
    }
}

/* sparse_adam_step: R/rasterizer.py:707-725 (per-splat step counter t, eps 1e-15).
 * lr_cols (59) = learning rate per parameter column. */
void or_adam(int64_t n, double *params, const double *grads, const uint8_t *touched, double *m, double *v,
             int64_t *t, const double *lr_cols) {
#pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < n; i++) {
        if (!touched[i]) continue;
        t[i] += 1;
        double bc1 = 1.0 - pow(0.9, (double)t[i]);
        double bc2 = 1.0 - pow(0.999, (double)t[i]);
        for (int k = 0; k < NP; k++) {
            size_t j = (size_t)NP * i + k;
            double g = grads[j];
            double mm = m[j] * 0.9 + (1 - 0.9) * g;
            double vv = v[j] * 0.999 + (1 - 0.999) * g * g;
            m[j] = mm;
            v[j] = vv;
            double mh = mm / bc1, vh = vv / bc2;
            params[j] -= lr_cols[k] * mh / (sqrt(vh) + 1e-15);
        }
    }
}

/* ------------------------------------------------------------------------- */
/* losses: R/losses.py:15-161                                                */

static void gauss_kernel(double K[11]) { /* :22-25 */
    double s = 0.0;
    for (int i = 0; i < 11; i++) {
        double x = i - 5;
        K[i] = exp(-(x * x) / (2.0 * 1.5 * 1.5));
        s += K[i];
    }
    for (int i = 0; i < 11; i++) K[i] /= s;
}

static int reflect(int j, int n) { /* :31-42, j in [-5, n+5) */
    if (n == 1) return 0;
    int period = 2 * n - 2;
    int a = j < 0 ? -j : j;
    a %= period;
    return a >= n ? period - a : a;
}

/* _blur (:45-52) on a (h, w, c) image, c channels interleaved */
static void blur(const double *img, int h, int w, int c, double *out, double *tmp) {
    double K[11];
    gauss_kernel(K);
    /* rows (axis 0) first, then columns (axis 1) - separable, matching convolve1d order */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            for (int ch = 0; ch < c; ch++) {
                double acc = 0.0;
                for (int t = 0; t < 11; t++) acc += K[10 - t] * img[((size_t)reflect(y + t - 5, h) * w + x) * c + ch];
                tmp[((size_t)y * w + x) * c + ch] = acc;
            }
    /* columns need the row-blurred image at reflected columns */
#pragma omp parallel for schedule(static)
    for (int y = 0; y < h; y++)
        for (int x = 0; x < w; x++)
            for (int ch = 0; ch < c; ch++) {
                double acc = 0.0;
                for (int t = 0; t < 11; t++) acc += K[10 - t] * tmp[((size_t)y * w + reflect(x + t - 5, w)) * c + ch];
                out[((size_t)y * w + x) * c + ch] = acc;
            }
}

/* _blur_adjoint (:55-69): zero-embed, correlate with the flipped kernel, fold reflections */
static void blur_adjoint(const double *g, int h, int w, int c, double *out) {
    double K[11];
    gauss_kernel(K);
    int ph = h + 10, pw = w + 10;
    double *pad = calloc((size_t)ph * pw * c, sizeof(double));
    double *pad2 = calloc((size_t)ph * pw * c, sizeof(double));
    /* axis 0: padded rows j in [0, ph): sum_t Kflip... convolve1d(g_embed, K[::-1]) */
#pragma omp parallel for schedule(static)
    for (int j = 0; j < ph; j++)
        for (int x = 0; x < w; x++)
            for (int ch = 0; ch < c; ch++) {
                double acc = 0.0;
                for (int t = 0; t < 11; t++) {
                    int src = j + 5 - t; /* convolve1d with K[::-1] == correlate with K */
                    int yy = src - 5;
                    if (yy < 0 || yy >= h) continue;
                    acc += K[t] * g[((size_t)yy * w + x) * c + ch];
                }
                pad[((size_t)j * pw + (x + 5)) * c + ch] = acc;
            }
#pragma omp parallel for schedule(static)
    for (int j = 0; j < ph; j++)
        for (int i = 0; i < pw; i++)
            for (int ch = 0; ch < c; ch++) {
                double acc = 0.0;
                for (int t = 0; t < 11; t++) {
                    int src = i + 5 - t;
                    if (src < 5 || src >= w + 5) continue;
                    acc += K[t] * pad[((size_t)j * pw + src) * c + ch];
                }
                pad2[((size_t)j * pw + i) * c + ch] = acc;
            }
    /* fold rows then columns (np.add.at in index order) */
    double *rows = calloc((size_t)h * pw * c, sizeof(double));
    for (int j = 0; j < ph; j++) {
        int r = reflect(j - 5, h);
        for (size_t k = 0; k < (size_t)pw * c; k++) rows[(size_t)r * pw * c + k] += pad2[(size_t)j * pw * c + k];
    }
    memset(out, 0, sizeof(double) * (size_t)h * w * c);
    for (int y = 0; y < h; y++)
        for (int i = 0; i < pw; i++) {
            int cc = reflect(i - 5, w);
            for (int ch = 0; ch < c; ch++) out[((size_t)y * w + cc) * c + ch] += rows[((size_t)y * pw + i) * c + ch];
        }
    free(pad);
    free(pad2);
    free(rows);
}

/* dssim_and_grad (:89-119) + photometric_loss (:122-130).  a, b, grad: (h, w, c). */
double or_photometric_loss(const double *a, const double *b, int h, int w, int c, double lam, double *grad,
                           double *out_l1, double *out_dssim) {
    size_t n = (size_t)h * w * c;
    double *buf = malloc(sizeof(double) * n * 14);
    double *ua = buf, *ub = buf + n, *uaa = buf + 2 * n, *uab = buf + 3 * n, *ubb = buf + 4 * n;
    double *tmp = buf + 5 * n, *prod = buf + 6 * n, *gua = buf + 7 * n, *guaa = buf + 8 * n, *guab = buf + 9 * n;
    double *A1 = buf + 10 * n, *A2 = buf + 11 * n, *A3 = buf + 12 * n;
    blur(a, h, w, c, ua, tmp);
    blur(b, h, w, c, ub, tmp);
    for (size_t k = 0; k < n; k++) prod[k] = a[k] * a[k];
    blur(prod, h, w, c, uaa, tmp);
    for (size_t k = 0; k < n; k++) prod[k] = a[k] * b[k];
    blur(prod, h, w, c, uab, tmp);
    for (size_t k = 0; k < n; k++) prod[k] = b[k] * b[k];
    blur(prod, h, w, c, ubb, tmp);
    const double C1 = 0.01 * 0.01, C2 = 0.03 * 0.03;
    double ssum = 0.0;
    for (size_t k = 0; k < n; k++) {
        double va = uaa[k] - ua[k] * ua[k];
        double vb = ubb[k] - ub[k] * ub[k];
        double vab = uab[k] - ua[k] * ub[k];
        double a1 = 2.0 * ua[k] * ub[k] + C1;
        double a2 = 2.0 * vab + C2;
        double b1 = ua[k] * ua[k] + ub[k] * ub[k] + C1;
        double b2 = va + vb + C2;
        double den = b1 * b2;
        double S = (a1 * a2) / den;
        ssum += S;
        double g1 = (2.0 * ub[k] * a2 - 2.0 * a1 * ub[k]) / den - S * (2.0 * ua[k] / b1) + S * (2.0 * ua[k] / b2);
        gua[k] = g1 / (double)n;
        guaa[k] = (-S / b2) / (double)n;
        guab[k] = (2.0 * a1 / den) / (double)n;
    }
    blur_adjoint(gua, h, w, c, A1);
    blur_adjoint(guaa, h, w, c, A2);
    blur_adjoint(guab, h, w, c, A3);
    double l1 = 0.0;
    for (size_t k = 0; k < n; k++) l1 += fabs(a[k] - b[k]);
    l1 /= (double)n;
    double dssim = 0.5 * (1.0 - ssum / (double)n);
    for (size_t k = 0; k < n; k++) {
        double d = a[k] - b[k];
        double sg = (d > 0) - (d < 0);
        double gm = A1[k] + 2.0 * a[k] * A2[k] + b[k] * A3[k];
        grad[k] = (1.0 - lam) * (sg / (double)n) + lam * (-0.5 * gm);
    }
    free(buf);
    if (out_l1) *out_l1 = l1;
    if (out_dssim) *out_dssim = dssim;
    return (1.0 - lam) * l1 + lam * dssim;
}

/* depth_ratio_loss (:133-154), dense form; gd/go are (h*w). */
double or_depth_ratio_loss(const double *depth, const double *opac, const double *sparse, int64_t npx, double guard,
                           double *gd, double *go) {
    int64_t nv = 0;
    for (int64_t k = 0; k < npx; k++) nv += sparse[k] > 0;
    memset(gd, 0, sizeof(double) * npx);
    memset(go, 0, sizeof(double) * npx);
    if (nv == 0) return 0.0;
    double val = 0.0;
    for (int64_t k = 0; k < npx; k++) {
        if (!(sparse[k] > 0)) continue;
        double so = opac[k] > guard ? opac[k] : guard;
        double r = depth[k] / so - sparse[k];
        val += fabs(r);
        double s = (double)((r > 0) - (r < 0)) / (double)nv;
        gd[k] = s / so;
        go[k] = opac[k] >= guard ? -s * depth[k] / (so * so) : 0.0;
    }
    return val / (double)nv;
}
