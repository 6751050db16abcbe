/*
 * gslic.h -- C ABI of the B200-native (sm_100a) Gaussian map-optimisation hot path.
 *
 * Drop-in boundary for the reference's Python entry points (R/ = splatslam package of
 * /root/reference/pkg/src).  Each entry point cites the reference function it replaces:
 *
 *   gs_preprocess   R/gaussians.py:180-215 project + R/rasterizer.py:445-452 (sigmoid, view
 *                   dirs, eval_sh R/gaussians.py:102-111) + influence_radius :91-102
 *   gs_bin          R/rasterizer.py:169-219 cull_tiles (+ touched of _reduce_entries :424)
 *   gs_render_fwd   R/rasterizer.py:226-293 _forward_kernel
 *   gs_loss         R/losses.py:157-161 mapping_loss (photometric :122-130 with
 *                   dssim_and_grad :89-119, depth_ratio_loss :133-154 on a LiDAR K-list)
 *   gs_render_bwd   R/rasterizer.py:296-435 _backward_kernel + _reduce_entries
 *   gs_chain_adam   R/rasterizer.py:559-644 _chain_to_attributes fused with
 *                   R/rasterizer.py:707-725 sparse_adam_step
 *   gs_chain        _chain_to_attributes only, accumulating parameter-row gradients
 *                   (multi-view / multi-GPU batches; followed by an allreduce + gs_adam)
 *   gs_chain_pose   _chain_to_attributes(with_pose=True) R/rasterizer.py:646-657
 *   gs_adam         sparse_adam_step on parameter-row gradients + a touched mask
 *
 * Conventions
 *   - Every pointer is a DEVICE pointer unless named host_*; the caller owns all memory.
 *   - The library never allocates and keeps no global state: transient per-view state lives
 *     in a caller-provided workspace carved by gs_frame_layout().  Calls are re-entrant;
 *     each runs on the caller's stream (cudaStream_t passed as void*).
 *   - Parameter rows: float32, GS_ROW floats per Gaussian, columns in the order of
 *     GaussianMap.parameters() (R/gaussians.py:150-153) = the Gaussian PLY field order
 *     (R/gaussians.py:255-256): pos 0-2, log_scale 3-5, quat(wxyz) 6-9, opacity_logit 10,
 *     sh_low 11-13, sh_high 14-58; 59-63 padding.
 *   - Return value: GS_OK or an error code; gs_last_error() gives a thread-local message.
 *     Codes map onto the reference taxonomy (R/errors.py): GS_ERR_ARG/DIMS -> DomainError,
 *     GS_ERR_WORKSPACE/CAPACITY -> DataError, GS_ERR_CUDA -> NumericalError-class runtime error.
 */
#ifndef GSLIC_H
#define GSLIC_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GS_ROW 64       /* floats per parameter row (59 used) */
#define GS_NPARAM 59
#define GS_TILE 16
#define GS_SMALL_CAND 16 /* candidate tiles culled per thread; larger footprints go warp-wide */
#define GS_G2D 20      /* int64 words per screen-space gradient row: 10 fields (mean2d 2, conic 3, opacity 1,
                          color 3, depth 1), each a fixed-point pair (hi, lo), value = hi 2^-24 + lo 2^-64
                          (integer atomics: sums are bit-identical run to run) */
#define GS_G2D_FIELDS 10
#define GS_LOSS_RING 64 /* per-iteration losses kept by an engine workspace (gs_frame.loss) */
#define GS_SPLAT 16    /* floats per 2D splat record: (mx, my, a, beta) (gamma, opacity, depth, qcut)
                          (r, g, b, 1 - opacity) (b, c, touched slot as int bits, 0); conic = (a, b, c), and the blend evaluates
                          q = a (dx + beta dy)^2 + gamma dy^2 with beta = b / a, gamma = (a c - b^2) / a */

enum {
    GS_OK = 0,
    GS_ERR_ARG = 1,
    GS_ERR_DIMS = 2,
    GS_ERR_WORKSPACE = 3,
    GS_ERR_CAPACITY = 4,
    GS_ERR_CUDA = 5
};

/* counters[] slots (int32, device) written by the pipeline */
enum {
    GS_CNT_ACTIVE = 0,   /* reserved (0) */
    GS_CNT_ENTRIES = 1,  /* E = kept (splat, tile) pairs */
    GS_CNT_TOUCHED = 2,  /* splats with >= 1 kept pair */
    GS_CNT_OVERFLOW = 3, /* nonzero when E exceeded entry_capacity (downstream kernels no-op) */
    GS_CNT_ENTRIES_EFF = 4, /* E, or 0 after an overflow (what the downstream kernels use) */
    GS_CNT_BIG = 5,      /* Gaussians culled warp-cooperatively (many candidate tiles) */
    GS_CNT_LOSS_TICKET = 6, /* blocks of the loss kernel done (the last one finalises; self-resetting) */
    GS_CNT_BIG_BITS = 7, /* words of big_bits in use */
    GS_CNT_SLOTS = 16,
    /* slots 8-15: look-back tickets; second half of the counters array: */
    GS_CNT_HUGE = 16,    /* reserved (0): huge slots are big-list indices below GS_HUGE_CAP */
    GS_CNT_HUGE_E = 17,  /* their kept pairs */
    GS_CNT_SMALL_E = 18, /* entries binned through the per-tile buckets */
    GS_CNT_HUGE_N = 19,  /* huge Gaussians with >= 1 kept tile (records in depth order) */
    GS_CNT_CULLQ1 = 20,  /* tiles left ambiguous by the band bounds of large footprints (cull_queue) */
    GS_CNT_LAZY = 21,    /* 1: gs_bin(GS_BIN_LAZY) left the tile lists unmaterialised */
    GS_CNT_ANYFLAG = 22, /* lazy lists: some tile needs its bucket (blend continuation) */
    GS_CNT_FLAGGED = 23, /* lazy lists: how many (their ids in a tile_scratch segment) */
    GS_CNT_FWD_CLEARED = 24 /* 1: the frame's forward cleared the g2d rows (GS_FWD_CLEAR_G2D); 0: with
                               lazy lists the chain rule clears each row after reading it */
};

#define GS_HUGE_CAND 256 /* candidate tiles above which a Gaussian is binned per tile */
#define GS_HUGE_CAP 4096 /* at most this many such Gaussians per view (the rest take the sort) */
#define GS_MAX_TILES 65536 /* tiles per view (4096 x 4096 px): bounds the per-CTA cull bitmaps */

/* Pinhole camera, world->camera (R/rasterizer.py:47-67).  Pixel centres are integers. */
typedef struct gs_camera {
    int32_t width, height;
    float fx, fy, cx, cy;
    float rot_cw[9]; /* row-major */
    float trans_cw[3];
    float center[3]; /* -rot_cw^T trans_cw (filled by gs_camera_init) */
} gs_camera;

/* One training view: camera + its supervision (resident in device memory). */
typedef struct gs_view {
    gs_camera cam;
    const float *target;      /* (H, W, 3) image */
    const int32_t *lidar_idx; /* (K,) pixel index y*W+x of LiDAR returns (sparse_depth > 0) */
    const float *lidar_z;     /* (K,) LiDAR depth */
    int32_t lidar_k;
    int32_t pad_;
} gs_view;

/* Transient per-view state, carved from one workspace by gs_frame_layout(). */
typedef struct gs_frame {
    int64_t n;               /* Gaussians */
    int64_t entry_capacity;  /* max kept (splat, tile) pairs */
    int32_t width, height, tiles_x, tiles_y;
    /* per Gaussian */
    float *splat2d;          /* n x GS_SPLAT records (see GS_SPLAT) */
    float *cov2d;            /* n x 4: c00 c01 c11 radius */
    int32_t *rect;           /* n x 8: per-Gaussian 32-B binning record: tile rect tx0 tx1 ty0 ty1 (empty:
                                tx1 < tx0), keep bits (uint64, first 64 candidate tiles) or the large
                                footprint's bitmap base, kept (Gaussian, tile) pairs, pad */
    uint8_t *valid;          /* n: near-plane & det test (R/gaussians.py:190-208) */
    uint8_t *touched;        /* n: >= 1 kept pair (R/rasterizer.py:424) */
    int32_t *touched_list;   /* n: compacted touched ids (unordered) */
    int64_t *g2d;            /* n x GS_G2D screen-space gradients, fixed-point accumulators; row k belongs to
                                touched_list[k] (its slot is also float 14 of its splat record) */
    float *grad_rows;        /* n x GS_ROW parameter gradients in touched-list order */
    float *bias_corr;        /* n x 2 reciprocal Adam bias corrections 1/(1-b1^t), 1/(1-b2^t) (touched-list order) */
    uint64_t *keep_bits;     /* unused (in the rect records) */
    int32_t *kept;           /* unused (in the rect records) */
    int32_t *big_list;       /* n: Gaussians with > GS_SMALL_CAND candidate tiles (warp-culled) */
    int32_t *big_slot;       /* n: huge slot (or -1) per big_list entry */
    int32_t *cull_queue;     /* cull_queue_cap x 2: (big index, tx << 16 | ty) left open by the band bounds */
    int64_t cull_queue_cap;
    int32_t *huge;           /* screen-covering Gaussians in depth order: GS_HUGE_CAP records of 8
                                ints (id, depth bits, slot), their ids, their 64-bit keys */
    uint32_t *huge_mask;     /* tiles x GS_HUGE_CAP/32: bit j of word w <-> the (32w+j)-th huge
                                Gaussian in depth order keeps the tile */
    uint32_t *huge_mask_t;   /* GS_HUGE_CAP x ceil(tiles/32): per huge slot, its kept tiles */
    int32_t *tile_scratch;   /* 5 x (tiles + 1): bucket counts / fill cursors, huge counts, bucket
                                offsets, list mode per tile, last huge record per tile */
    uint64_t *tile_minkey;   /* tiles: smallest bucketed (depth << 32 | id) key per tile */
    uint32_t *big_bits;      /* cull bitmaps of the large-footprint Gaussians (base in keep_bits) */
    int64_t big_bits_words;  /* capacity of big_bits; overflowing Gaussians are re-culled at emit */
    /* sort buffers */
    uint64_t *keys_a, *keys_b; /* entry_capacity: per-tile buckets of (depth << 32 | id) keys, merge scratch */
    /* per entry / tile */
    int32_t *entry_splat;    /* entry_capacity */
    int32_t *tile_offsets;   /* tiles + 1 */
    int32_t *counters;       /* GS_CNT_SLOTS */
    /* per pixel */
    float *color;            /* H x W x 3  (un-normalised, background 0) */
    float *depth;            /* H x W      (sum z w) */
    float *opacity;          /* H x W      (1 - T) */
    float *trans;            /* H x W      (T) */
    int32_t *n_contrib;      /* H x W */
    float *g_color;          /* H x W x 3  dL/dcolor */
    float *g_depth;          /* H x W      xi dLd/ddepth */
    float *g_opac;           /* H x W      xi dLd/dopacity */
    double *loss_parts;      /* per-block partial sums */
    double *loss;            /* 8 + 5 GS_LOSS_RING: total, photometric, depth, dssim, running sum
                                (GS_LOSS_ACCUMULATE), -, ring position, -, then the per-iteration loss
                                ring: with GS_LOSS_ACCUMULATE iteration i writes its total to
                                loss[8 + i % GS_LOSS_RING] (i counted from the workspace's layout)
                                and a snapshot of counters[0..8) to the int32 words
                                8 (i % GS_LOSS_RING) .. + 8 after loss[8 + GS_LOSS_RING] */
    int64_t loss_blocks;
    int64_t *pose_acc;       /* 12: fixed-point accumulators of the pose gradient (gs_chain_pose) */
    float *ssim_g;           /* 3 x H x W x 4: SSIM-map partials per channel (d/d mu_a, d/d var sum,
                                d/d sigma_ab, -), written and read by gs_loss */
} gs_frame;

/* ---- setup ---------------------------------------------------------------- */
/* The workspace (>= gs_workspace_size bytes, 256-B aligned) must be zero-filled once before its
 * first use; afterwards frames reuse it without clearing. */
size_t gs_workspace_size(int64_t n, int32_t width, int32_t height, int64_t entry_capacity);
int gs_frame_layout(int64_t n, int32_t width, int32_t height, int64_t entry_capacity, void *ws,
                    size_t ws_bytes, gs_frame *out);
/* fills cam->center from rot_cw / trans_cw (host struct) */
void gs_camera_init(gs_camera *host_cam);
const char *gs_last_error(void);
int gs_version(void);

/* ---- the iteration ------------------------------------------------------------------ */
/* R/gaussians.py:180-215 + R/rasterizer.py:445-452: projection, EWA covariance, SH colour,
 * opacity sigmoid, influence radius, tile rectangle and cut; also resets touched[]. */
int gs_preprocess(const gs_frame *f, const float *params, const gs_view *view, void *stream);
/* flags = GS_PP_LAZY_SH (the iteration engine): SH colours only for the Gaussians that can be
 * blended (kept in >= 1 tile, or large footprints still to be culled); the others' colour slots
 * are left 0 and their SH columns are never read.  gs_preprocess(...) = gs_preprocess_ex(..., 0). */
#define GS_PP_LAZY_SH 1
int gs_preprocess_ex(const gs_frame *f, const float *params, const gs_view *view, int32_t flags, void *stream);

/* R/rasterizer.py:169-219: depth sort of active Gaussians, exact per-tile cull, (tile|depth)
 * ordered entries, tile ranges, touched mask + list; zeroes touched g2d rows.
 * cull=0 reproduces the reference's cull=False (every valid Gaussian in every tile). */
int gs_bin(const gs_frame *f, int32_t cull, void *stream);
/* cull = GS_BIN_LAZY (the iteration engine): cull as cull=1, but the tile lists are not
 * materialised.  A tile's list is its screen-covering Gaussians (depth-ordered masks) followed by
 * its depth-sorted bucket; gs_render_fwd sorts and merges buckets only for the tiles whose blend
 * gets that far (or whose bucket interleaves with the screen-covering ones).  entry_splat is then
 * valid only for those tiles; tile_offsets, touched and the rendered images are always complete. */
#define GS_BIN_LAZY 2

/* R/rasterizer.py:226-293 */
int gs_render_fwd(const gs_frame *f, int32_t early_stop, void *stream);
/* flags: GS_FWD_EARLY_STOP (the reference's early termination, as gs_render_fwd's early_stop);
 * GS_FWD_CLEAR_G2D: the forward also clears the g2d rows of the touched slots 0..nt-1 (in its
 * epilogue, as whole lines that stay in L2), so a following gs_render_bwd_ex(.., GS_BWD_ROWS_ZERO)
 * starts from zero, and the chain rule only reads them.  Without it (and with lazy lists) the
 * chain rule clears each row after reading it instead.  An engine keeps one choice for all its
 * iterations: the forward's clear pays at ~100k+ touched Gaussians, the chain's below. */
#define GS_FWD_EARLY_STOP 1
#define GS_FWD_CLEAR_G2D 2
int gs_render_fwd_ex(const gs_frame *f, int32_t flags, void *stream);

/* R/losses.py:157-161 with the depth term on the view's LiDAR K-list; writes g_color,
 * g_depth, g_opac and loss[0..3]. */
int gs_loss(const gs_frame *f, const gs_view *view, float lam, float xi, void *stream);
/* flags: GS_LOSS_TABLES_READY -- the per-axis reflection tables of this image size are already in
 * the workspace (a previous gs_loss built them): skip rebuilding; GS_LOSS_ACCUMULATE -- also add
 * the total to loss[4] (a running sum the caller resets). gs_loss(...) = gs_loss_ex(..., 0). */
#define GS_LOSS_TABLES_READY 1
#define GS_LOSS_ACCUMULATE 2
/* GS_LOSS_DEPTH_GRADS_ZERO -- g_depth / g_opac are zero on entry (fresh workspace, or the previous
 * gs_render_bwd_ex ran with GS_BWD_CLEAR_DEPTH_GRADS): only the LiDAR pixels are written, and the
 * depth term runs alongside the photometric kernel's tail. */
#define GS_LOSS_DEPTH_GRADS_ZERO 4
int gs_loss_ex(const gs_frame *f, const gs_view *view, float lam, float xi, int32_t flags, void *stream);

/* R/rasterizer.py:296-435: accumulates g2d rows of touched Gaussians. */
int gs_render_bwd(const gs_frame *f, void *stream);
/* flags = GS_BWD_ROWS_ZERO: the caller guarantees the touched Gaussians' g2d rows are zero (the
 * engines: gs_render_fwd_ex(.., GS_FWD_CLEAR_G2D) cleared rows 0..nt-1, or the previous chain rule
 * cleared the rows it read), so they are not cleared first. */
#define GS_BWD_ROWS_ZERO 1
/* GS_BWD_CLEAR_DEPTH_GRADS: the backward resets g_depth / g_opac to zero after reading them (the
 * protocol of GS_LOSS_DEPTH_GRADS_ZERO) */
#define GS_BWD_CLEAR_DEPTH_GRADS 2
int gs_render_bwd_ex(const gs_frame *f, int32_t flags, void *stream);

/* R/rasterizer.py:559-644 + :707-725 fused.  lr_cols: device (GS_ROW) per-column rates.
 * adam_t: per-Gaussian step counter (int32). */
int gs_chain_adam(const gs_frame *f, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                  const gs_view *view, const float *lr_cols, void *stream);

/* gs_chain_adam split over touched-list chunks so that the chain rule of chunk i+1 (stage 0,
 * FP64-latency-bound) can run concurrently with the Adam stream of chunk i (stage 1, HBM-bound)
 * on a second stream: stage 0 of a chunk must precede its stage 1; chunks are disjoint. */
int gs_chain_adam_part(const gs_frame *f, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                       const gs_view *view, const float *lr_cols, int32_t stage, int32_t part, int32_t nparts,
                       void *stream);

/* Multi-GPU batch step over peer memory: the ranks' gradient-row allreduce fused
 * with the sparse Adam update (R/rasterizer.py:707-725) in one persistent kernel per rank.
 * grads / packed / gready / rdone: world device pointers each (this rank's own and its peers',
 * opened with gs_ipc_import), packed >= u x 60 floats, the flags zero-initialised u64 words;
 * idx[0..u): the union of touched ids (id order, identical on every rank); epoch: 1, 2, ... per
 * step.  Rank r sums its shard [u r / world, u (r+1) / world) over the ranks in rank order into
 * packed[r], then every rank applies the update for every shard from its owner's packed rows,
 * clearing my_grads rows and touched flags (as gs_adam_packed).  keep (optional, u x 60): the
 * reduced rows.  *err = 1 if a peer never arrived (bounded waits). */
int gs_p2p_reduce_adam(int32_t world, int32_t rank, const float *const *grads, const float *const *packed,
                       uint64_t *const *gready, uint64_t *const *rdone, uint64_t epoch, int64_t u,
                       const int32_t *idx, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                       const float *lr_cols, float *my_grads, uint8_t *touched, uint32_t *ticket, float *keep,
                       int32_t *err, void *stream);

/* CUDA IPC for gs_p2p_reduce_adam: the 64-byte handle of the allocation holding ptr and ptr's
 * offset in it; a peer's pointer from (handle, offset) (base: for gs_ipc_close). */
int gs_ipc_export(const void *ptr, uint8_t *handle, int64_t *offset);
int gs_ipc_import(const uint8_t *handle, int64_t offset, void **ptr, void **base);
int gs_ipc_close(void *base);

/* R/rasterizer.py:559-644 only: grads[row] += d loss / d params (rows of GS_ROW floats);
 * touched_accum[i] |= touched[i]. */
int gs_chain(const gs_frame *f, const float *params, float *grads, uint8_t *touched_accum, const gs_view *view,
             void *stream);

/* backward(with_pose=True) (R/rasterizer.py:543-556, pose part :646-657): as gs_chain, plus the
 * 6-dof pose gradient (rho, theta) on the left tangent of T_cw, written to pose[6] (device FP64,
 * overwritten).  grads and touched_accum both NULL: the pose gradient only (the tracker's
 * photometric_refine, R/odometry.py:305-336). */
int gs_chain_pose(const gs_frame *f, const float *params, float *grads, uint8_t *touched_accum,
                  const gs_view *view, double *pose, void *stream);

/* R/rasterizer.py:707-725 over a dense touched mask (n entries) and gradient rows. */
int gs_adam(float *params, float *adam_m, float *adam_v, int32_t *adam_t, const float *grads,
            const uint8_t *touched, int64_t n, const float *lr_cols, void *stream);

/* ---- batch reduction (multi-view / multi-GPU) -------------------------------- */
/* idx[0 .. *count) = the i with flags[i] != 0, ascending (device-side, no host sync; identical on
 * every rank for identical flags).  scratch: ceil(n / 1024) ints. */
int gs_compact_flags(const uint8_t *flags, int64_t n, int32_t *idx, int32_t *count, int32_t *scratch, void *stream);
/* packed[i] = rows[idx[i]][0:60] for i < min(*count, cap) (the 59 parameters + 1 pad, 16-B aligned):
 * the union's gradient rows, contiguous for the allreduce. */
int gs_gather_rows(const float *rows, const int32_t *idx, const int32_t *count, int64_t cap, float *packed,
                   void *stream);
/* sparse_adam_step (R/rasterizer.py:707-725) over rows idx[first .. first + num) clipped to *count,
 * gradient row i from packed[i] (60 floats) or, with packed == NULL, from grads[idx[i]]; the step
 * counters advance; grads rows (when given) and touched flags (when given) of those rows are
 * cleared for the next batch. */
int gs_adam_packed(float *params, float *adam_m, float *adam_v, int32_t *adam_t, const float *packed,
                   const int32_t *idx, const int32_t *count, int64_t first, int64_t num, const float *lr_cols,
                   float *grads, uint8_t *touched, void *stream);

/* ---- helpers for the reference-shaped Python API ------------------------------------- */
/* dense sparse_depth (H,W) -> K-list (idx, z) in pixel order; count written to *k_out (device
 * int32).  idx must hold H*W + ceil(H*W/1024) ints (the tail is scratch), z H*W floats. */
int gs_lidar_compact(const float *sparse_depth, int32_t width, int32_t height, int32_t *idx, float *z,
                     int32_t *k_out, void *stream);
/* R/gaussians.py:180-215 full records: mu_cam (n,3) mean2d (n,2) cov2d (n,4) conic (n,3) depth (n)
 * valid (n) jproj (n,6) m (n,6) cov3d (n,9); any output pointer may be NULL. */
int gs_project(const float *params, int64_t n, const gs_camera *cam, float *mu_cam, float *mean2d,
               float *cov2d, float *conic, float *depth, uint8_t *valid, float *jproj, float *mmat,
               float *cov3d, void *stream);
/* R/gaussians.py:102-111 */
int gs_eval_sh(const float *sh_low, const float *sh_high, const float *dirs, int64_t n, float *colors,
               float *preclamp, void *stream);
/* Pack externally supplied 2D splats (mean2d, conic, cov2d(3), opacity, depth, valid) into
 * the frame so gs_bin can run stand-alone (R/rasterizer.py:169 cull_tiles signature). */
int gs_pack_splats(const gs_frame *f, const float *mean2d, const float *conic, const float *cov2d3,
                   const float *opacity, const float *depth, const uint8_t *valid, const float *colors,
                   void *stream);

/* ---- keyframe preparation --------------------------------------- */
/* R/mapper.py:69-81 project_points over m world points (m x 3), FP64, rounded pixel centres
 * (round half to even, as np.round); optional outputs (NULL = skip): u, v, ui, vi, z, flags
 * (bit 0 inside the image, bit 1 "fresh": inside and opacity[vi, ui] < tau, the expand_map test
 * of R/mapper.py:222-225; needs opacity (H, W)), colors (m x 3, bilinear_color R/mapper.py:84-98
 * of image (H, W, 3)).  cam is a DEVICE pointer. */
int gs_project_points(const float *points, int64_t m, const gs_camera *cam, const float *image,
                      const float *opacity, float tau, float *u, float *v, int32_t *ui, int32_t *vi,
                      float *z, uint8_t *flags, float *colors, void *stream);
/* R/mapper.py:101-107 zbuffer_project: dense (height, width) sparse-depth map, the nearest point
 * per pixel, 0 where no point lands.  zbuf: width * height uint32 scratch. */
int gs_zbuffer(const float *points, int64_t m, const gs_camera *cam, int32_t width, int32_t height,
               uint32_t *zbuf, float *depth, void *stream);
/* R/gaussians.py:227-248 init_from_points: m parameter rows (GS_ROW floats each) from points
 * (m x 3), colours (m x 3), camera depths (m) and the focal length. */
int gs_init_rows(const float *points, const float *colors, const float *depths, int64_t m, float focal,
                 float *rows, void *stream);

/* 8-bit frame (n bytes, e.g. an RGB camera image) -> float32 k / 255 (computed in FP64, rounded
 * once: bit-identical to the fp32 rounding of a float64 image loaded from PNG, R/io_formats.py:52-57) */
int gs_decode_u8(const uint8_t *src, float *dst, int64_t n, void *stream);

/* ---- photometric pose refinement (SURVEY.md 8f row 2, R/odometry.py:305-336) ------------- */
/* img_mask[p] = |np.gradient(mean over channels of image)| > grad_gate (R/odometry.py:314-316) */
int gs_track_mask(const float *image, int32_t width, int32_t height, float grad_gate, uint8_t *mask, void *stream);
/* f->g_color *= img_mask & (f->opacity > opac_gate) (R/odometry.py:325-326) */
int gs_track_grad(const gs_frame *f, const uint8_t *img_mask, float opac_gate, void *stream);
/* One Adam step on the pose tangent (R/odometry.py:328-335): state (device FP64, 25) = rot_cw[9],
 * trans_cw[3], m[6], v[6], iteration; rot <- exp_so3(step[3:]) rot, trans <- exp_so3(step[3:])
 * trans + step[:3]; the view's camera (rot, trans, centre) is rewritten in place. */
int gs_pose_adam(gs_view *view, double *state, const double *pose_grad, float lr, void *stream);

#ifdef __cplusplus
}
#endif
#endif /* GSLIC_H */
