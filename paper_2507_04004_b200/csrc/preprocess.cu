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
    bool touched = false, big = false;
    if (i < n) {
        const float *p = srow[warp][lane];
        float4 *s2 = reinterpret_cast<float4 *>(f.splat2d) + 3 * i;
        float4 *cv = reinterpret_cast<float4 *>(f.cov2d) + i;
        int4 *rc = reinterpret_cast<int4 *>(f.rect) + i;
        if (!near_ok) {
            float z = (p[0] * cam.rot_cw[6] + p[1] * cam.rot_cw[7] + p[2] * cam.rot_cw[8]) + cam.trans_cw[2];
            s2[0] = make_float4(0.f, 0.f, 0.f, 0.f);
            s2[1] = make_float4(0.f, 0.f, z, 0.f);
            s2[2] = make_float4(0.f, 0.f, 0.f, 0.f);
            *cv = make_float4(0.f, 0.f, 0.f, -1.f);
            *rc = make_int4(0, -1, 0, -1);
            f.valid[i] = 0;
            f.kept[i] = 0;
            f.keys_a[i] = (0xffffffffull << 32) | (uint64_t)i;
        } else {
            // FP64 projection, rounded once to fp32: mu_cam = R p + t cancels for Gaussians near
            // the 0.01 m clip plane, and fp32 would shift their whole footprint
            ProjectedT<double> pd;
            project_full<double>(p, cam, pd);
            Projected pr;
            pr.mu[2] = (float)pd.mu[2];
            pr.mx = (float)pd.mx;
            pr.my = (float)pd.my;
            pr.c00 = (float)pd.c00;
            pr.c01 = (float)pd.c01;
            pr.c11 = (float)pd.c11;
            pr.ca = (float)pd.ca;
            pr.cb = (float)pd.cb;
            pr.cc = (float)pd.cc;
            pr.valid = pd.valid;
            const float op = 1.0f / (1.0f + expf(-p[10]));
            // view direction camera->Gaussian (R/rasterizer.py:447-451) and SH colour
            const float u0 = p[0] - cam.center[0], u1 = p[1] - cam.center[1], u2 = p[2] - cam.center[2];
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
                const float pre = b[0] * p[11 + c] + acc + 0.5f;
                col[c] = pre > 0.0f ? pre : 0.0f;
            }
            int4 rect = make_int4(0, -1, 0, -1);
            float qcut = 0.0f, radius = -1.0f;
            const bool active = pr.valid && tile_rect(pr.c00, pr.c01, pr.c11, op, pr.mx, pr.my, f.width, f.height,
                                                      f.tiles_x, f.tiles_y, rect, qcut, radius);
            if (!active) rect = make_int4(0, -1, 0, -1);
            // exact per-tile cull of the rectangle (R/rasterizer.py:150-166), fused here for small
            // footprints; large ones are culled warp-cooperatively by cull_big_kernel
            const int ncand = (rect.y - rect.x + 1) * (rect.w - rect.z + 1);
            big = active && ncand > GS_SMALL_CAND;
            uint64_t bits = 0ull;
            const int kept = (active && !big)
                                 ? cull_rect(pr.mx, pr.my, pr.ca, pr.cb, pr.cc, qcut, rect, f.width, f.height, bits)
                                 : 0;
            touched = kept > 0;
            s2[0] = make_float4(pr.mx, pr.my, pr.ca, pr.cb);
            s2[1] = make_float4(pr.cc, op, pr.mu[2], qcut);
            // 1 - opacity = sigmoid(-logit), kept exact for the blend's 1 - alpha
            s2[2] = make_float4(col[0], col[1], col[2], 1.0f / (1.0f + expf(p[10])));
            *cv = make_float4(pr.c00, pr.c01, pr.c11, radius);
            *rc = rect;
            f.valid[i] = pr.valid ? 1 : 0;
            f.kept[i] = kept;
            f.keep_bits[i] = bits;
            f.keys_a[i] = touched ? (((uint64_t)__float_as_uint(pr.mu[2]) << 32) | (uint64_t)i)
                                  : ((0xffffffffull << 32) | (uint64_t)i);
        }
        f.touched[i] = touched ? 1 : 0;
    }
    warp_append(touched, (int32_t)i, &f.counters[GS_CNT_TOUCHED], f.touched_list);
    warp_append(big, (int32_t)i, &f.counters[GS_CNT_BIG], f.big_list);
}

// Exact cull of the large-footprint Gaussians (> GS_SMALL_CAND candidate tiles), one CTA per
// Gaussian, same decision as cull_rect:
//   A) every candidate tile is classified by continuous bounds of q over its pixel rectangle
//      (q is convex: its maximum is at a corner; the lower bound is the one of tile_keep) with
//      a margin far above the fp32 evaluation error, so "surely kept" / "surely culled" agree
//      with the exact integer-grid test.  Only tiles straddling the qcut boundary are queued;
//   B) the queued tiles get the exact per-row test, 16 lanes per tile (one pixel row each).
// Results go to a shared-memory bitmap: by candidate index (big_bits, for the emit) or, for
// screen-covering Gaussians with a huge slot, by tile index (huge_mask_t row of the slot,
// transposed into depth order by huge_transpose_kernel).
constexpr int BIG_THREADS = 256;
constexpr int CB_WORDS = GS_MAX_TILES / 32;
constexpr int CB_QCAP = 2048;

// 1: every pixel of the tile has q <= qcut; 0: none has; -1: decide exactly
__device__ __forceinline__ int tile_class(float mx, float my, float ca, float cb, float cc, float qcut, float kx,
                                          float ky, int x0, int x1, int y0, int y1) {
    const float ax0 = (float)x0 - mx, ax1 = (float)x1 - mx, ay0 = (float)y0 - my, ay1 = (float)y1 - my;
    const float scale = ca * fmaxf(ax0 * ax0, ax1 * ax1) + cc * fmaxf(ay0 * ay0, ay1 * ay1);
    const float margin = 1e-5f * scale + 1e-6f;
    const float tb = 2.0f * cb;
    const float xx0 = ca * ax0 * ax0, xx1 = ca * ax1 * ax1, yy0 = cc * ay0 * ay0, yy1 = cc * ay1 * ay1;
    float qmax = xx0 + tb * ax0 * ay0 + yy0;
    qmax = fmaxf(qmax, xx1 + tb * ax1 * ay0 + yy0);
    qmax = fmaxf(qmax, xx0 + tb * ax0 * ay1 + yy1);
    qmax = fmaxf(qmax, xx1 + tb * ax1 * ay1 + yy1);
    if (qmax + margin < qcut) return 1;
    if (!(ax0 <= 0.0f && ax1 >= 0.0f && ay0 <= 0.0f && ay1 >= 0.0f)) {
        float qc = 3.0e38f;
        const float ys[2] = {ay0, ay1}, xs[2] = {ax0, ax1};
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const float y = ys[k];
            const float dx = fminf(fmaxf(kx * y, ax0), ax1);  // kx = -cb/ca
            qc = fminf(qc, ca * dx * dx + tb * dx * y + cc * y * y);
            const float x = xs[k];
            const float dy = fminf(fmaxf(ky * x, ay0), ay1);  // ky = -cb/cc
            qc = fminf(qc, ca * x * x + tb * x * dy + cc * dy * dy);
        }
        if (qc - margin > qcut) return 0;
    }
    return -1;
}

__global__ void __launch_bounds__(BIG_THREADS) cull_big_kernel(gs_frame f, int allow_huge) {
    __shared__ uint32_t s_bits[CB_WORDS];
    __shared__ int32_t s_queue[CB_QCAP];
    __shared__ int s_nq, s_slot, s_cnt;
    __shared__ int64_t s_base;
    const int tid = threadIdx.x, lane = tid & 31;
    const int T = f.tiles_x * f.tiles_y, tw = (T + 31) >> 5;
    const int64_t nb = f.counters[GS_CNT_BIG];
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int g = f.big_list[b];
        const float4 s0 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g];
        const float4 s1 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g + 1];
        const float mx = s0.x, my = s0.y, ca = s0.z, cb = s0.w, cc = s1.x, qcut = s1.w;
        const int4 r = reinterpret_cast<const int4 *>(f.rect)[g];
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        const int words = (ncand + 31) >> 5;
        // the bounds are conservative (margin), so their minimisers need not be exact
        const float kx = __fdividef(-cb, ca), ky = __fdividef(-cb, cc);
        if (tid == 0) {
            s_cnt = 0;
            s_nq = 0;
            // screen-covering Gaussians take a huge slot: their kept tiles are recorded per
            // tile and they skip the emit + sort
            int slot = -1;
            if (allow_huge && ncand > GS_HUGE_CAND) {
                slot = atomicAdd(&f.counters[GS_CNT_HUGE], 1);
                if (slot >= GS_HUGE_CAP) slot = -1;
            }
            s_slot = slot;
            // the others keep a cull bitmap for the emit (on overflow the emit re-culls)
            int64_t base = -1;
            if (slot < 0) {
                base = atomicAdd(&f.counters[GS_CNT_BIG_BITS], words);
                if (base + words > f.big_bits_words) base = -1;
            }
            s_base = base;
        }
        __syncthreads();
        const int slot = s_slot;
        const int64_t base = s_base;
        const bool by_tile = slot >= 0;
        const int nwords = by_tile ? tw : words;
        for (int w = tid; w < nwords; w += BIG_THREADS) s_bits[w] = 0u;
        __syncthreads();
        // A) classification; (tx, ty) of candidate c advance incrementally (no divides)
        {
            const int sy = BIG_THREADS / nx, sx = BIG_THREADS % nx;
            int ty = r.z + tid / nx, tx = r.x + tid % nx;
            for (int c = tid; c < ncand; c += BIG_THREADS) {
                const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
                const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
                int cls = tile_class(mx, my, ca, cb, cc, qcut, kx, ky, x0, x1, y0, y1);
                if (cls < 0) {
                    const unsigned amb = __activemask();
                    const unsigned lt = amb & ((1u << lane) - 1u);
                    int q0 = 0;
                    if (lt == 0u) q0 = atomicAdd(&s_nq, __popc(amb));
                    const int q = __shfl_sync(amb, q0, __ffs(amb) - 1) + __popc(lt);
                    if (q < CB_QCAP) s_queue[q] = c;
                    else cls = tile_keep(mx, my, ca, cb, cc, qcut, x0, x1, y0, y1) ? 1 : 0;
                }
                // one shared atomic per distinct bitmap word of the warp
                const int bit = by_tile ? ty * f.tiles_x + tx : c;
                const unsigned act = __activemask();
                const unsigned peers = __match_any_sync(act, bit >> 5);
                const unsigned word = __reduce_or_sync(peers, cls > 0 ? 1u << (bit & 31) : 0u);
                if (lane == __ffs(peers) - 1 && word) atomicOr(&s_bits[bit >> 5], word);
                tx += sx;
                ty += sy;
                if (tx > r.y) {
                    tx -= nx;
                    ty++;
                }
            }
        }
        __syncthreads();
        // B) exact test of the queued tiles: 16 lanes per tile, one pixel row per lane
        {
            const int nq = min(s_nq, CB_QCAP);
            const int grp = tid >> 4, row = tid & 15;
            for (int q0 = 0; q0 < nq; q0 += BIG_THREADS / 16) {  // uniform trip count: ballots are warp-wide
                const int qi = q0 + grp;
                bool hit = false;
                int c = 0, tx = 0, ty = 0;
                if (qi < nq) {
                    c = s_queue[qi];
                    ty = r.z + c / nx;
                    tx = r.x + c % nx;
                    const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
                    const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
                    if (y0 + row <= y1) hit = row_hits(mx, my, ca, cb, cc, qcut, x0, x1, y0 + row);
                }
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (row == 0 && ((bal >> (lane & 16)) & 0xffffu)) {
                    const int bit = by_tile ? ty * f.tiles_x + tx : c;
                    atomicOr(&s_bits[bit >> 5], 1u << (bit & 31));
                }
            }
        }
        __syncthreads();
        int count = 0;
        for (int w = tid; w < nwords; w += BIG_THREADS) {
            const uint32_t v = s_bits[w];
            count += __popc(v);
            if (by_tile) f.huge_mask_t[(int64_t)slot * tw + w] = v;
            else if (base >= 0) f.big_bits[base + w] = v;
        }
        for (int o = 16; o > 0; o >>= 1) count += __shfl_xor_sync(0xffffffffu, count, o);
        if (lane == 0 && count) atomicAdd(&s_cnt, count);
        __syncthreads();
        if (tid == 0) {
            const int kept = s_cnt;
            f.kept[g] = kept;
            f.keep_bits[g] = (uint64_t)base;  // bitmap base for large footprints (-1: none)
            if (slot >= 0 && kept > 0) {  // kept < 0 encodes the huge slot
                f.kept[g] = -(1 + slot);
                atomicAdd(&f.counters[GS_CNT_HUGE_E], kept);
            }
            f.touched[g] = kept > 0;
            if (kept > 0) {
                f.keys_a[g] = ((uint64_t)__float_as_uint(s1.z) << 32) | (uint64_t)g;
                f.touched_list[atomicAdd(&f.counters[GS_CNT_TOUCHED], 1)] = g;
            }
        }
        __syncthreads();
    }
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
    const float ca = conic[3 * i], cb = conic[3 * i + 1], cc = conic[3 * i + 2];
    uint64_t bits = 0ull;
    const bool big = active && (rect.y - rect.x + 1) * (rect.w - rect.z + 1) > GS_SMALL_CAND;
    const int kept = (active && !big) ? cull_rect(mx, my, ca, cb, cc, qcut, rect, f.width, f.height, bits)
                                      : (big ? -1 : 0);
    float4 *s2 = reinterpret_cast<float4 *>(f.splat2d) + 3 * i;
    s2[0] = make_float4(mx, my, ca, cb);
    s2[1] = make_float4(cc, o, depth[i], qcut);
    s2[2] = colors ? make_float4(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2], 1.0f - o)
                   : make_float4(0.f, 0.f, 0.f, 1.0f - o);
    reinterpret_cast<float4 *>(f.cov2d)[i] = make_float4(c00, c01, c11, radius);
    reinterpret_cast<int4 *>(f.rect)[i] = rect;
    f.valid[i] = v;
    f.kept[i] = kept;
    f.keep_bits[i] = bits;
    f.touched[i] = kept > 0;
    f.keys_a[i] = kept > 0 ? (((uint64_t)__float_as_uint(depth[i]) << 32) | (uint64_t)i) : ((0xffffffffull << 32) | (uint64_t)i);
}

// the touched and large-footprint lists of the pack path (unordered; consumers are order
// independent)
__global__ void touched_list_kernel(gs_frame f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int k = i < f.n ? f.kept[i] : 0;
    if (k < 0) f.kept[i] = 0;
    warp_append(k > 0, (int32_t)i, &f.counters[GS_CNT_TOUCHED], f.touched_list);
    warp_append(k < 0, (int32_t)i, &f.counters[GS_CNT_BIG], f.big_list);
}

// Ordered compaction of sparse_depth > 0 into the K-list (np.flatnonzero order), two passes:
// per-chunk counts, then each chunk sums its predecessors' counts and writes in order.
constexpr int LC_CHUNK = 1024;

__global__ void lidar_count_kernel(const float *__restrict__ sparse, int64_t npx, int32_t *chunk_cnt) {
    __shared__ int s;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const int64_t p = (int64_t)blockIdx.x * LC_CHUNK + threadIdx.x;
    const bool hit = p < npx && sparse[p] > 0.0f;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&s, __popc(m));
    __syncthreads();
    if (threadIdx.x == 0) chunk_cnt[blockIdx.x] = s;
}

__global__ void lidar_write_kernel(const float *__restrict__ sparse, int64_t npx, const int32_t *__restrict__ chunk_cnt,
                                   int32_t *idx, float *z, int32_t *k_out) {
    __shared__ int s_warp[LC_CHUNK / 32];
    __shared__ int s_base;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    int acc = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += LC_CHUNK) acc += chunk_cnt[c];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_base, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t p = (int64_t)blockIdx.x * LC_CHUNK + threadIdx.x;
    const float v = p < npx ? sparse[p] : 0.0f;
    const bool hit = v > 0.0f;
    const unsigned m = __ballot_sync(0xffffffffu, hit);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int before = s_base;
    for (int w = 0; w < warp; w++) before += s_warp[w];
    if (hit) {
        const int pos = before + __popc(m & ((1u << lane) - 1u));
        idx[pos] = (int32_t)p;
        z[pos] = v;
    }
    if (blockIdx.x == gridDim.x - 1 && threadIdx.x == 0) {
        int tot = s_base;
        for (int w = 0; w < LC_CHUNK / 32; w++) tot += s_warp[w];
        *k_out = tot;
    }
}

}  // namespace gs

using namespace gs;

extern "C" int gs_preprocess(const gs_frame *f, const float *params, const gs_view *view, void *stream) {
    if (!f || !params || !view) {
        set_error("gs_preprocess: null argument");
        return GS_ERR_ARG;
    }
    cudaMemsetAsync(f->counters, 0, sizeof(int32_t) * GS_CNT_SLOTS * 2, (cudaStream_t)stream);
    if (f->n == 0) return GS_OK;
    int64_t warps = (f->n + 31) / 32;
    int blocks = (int)((warps + PP_WARPS - 1) / PP_WARPS);
    preprocess_kernel<<<blocks, PP_THREADS, 0, (cudaStream_t)stream>>>(*f, params, view);
    int rc = check_launch("preprocess_kernel");
    if (rc) return rc;
    int tb = 0, rb = 0;
    const int allow_huge = compact_words(f->n, f->tiles_x * f->tiles_y, &tb, &rb) ? 1 : 0;
    cull_big_kernel<<<8 * 148, 256, 0, (cudaStream_t)stream>>>(*f, allow_huge);
    return check_launch("cull_big_kernel");
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
    cudaMemsetAsync(f->counters, 0, sizeof(int32_t) * GS_CNT_SLOTS * 2, (cudaStream_t)stream);
    if (f->n == 0) return GS_OK;
    pack_kernel<<<(unsigned)((f->n + 127) / 128), 128, 0, (cudaStream_t)stream>>>(*f, mean2d, conic, cov2d3, opacity,
                                                                                   depth, valid, colors);
    int rc = check_launch("pack_kernel");
    if (rc) return rc;
    touched_list_kernel<<<(unsigned)((f->n + 255) / 256), 256, 0, (cudaStream_t)stream>>>(*f);
    if ((rc = check_launch("touched_list_kernel"))) return rc;
    int tb = 0, rb = 0;
    const int allow_huge = compact_words(f->n, f->tiles_x * f->tiles_y, &tb, &rb) ? 1 : 0;
    cull_big_kernel<<<8 * 148, 256, 0, (cudaStream_t)stream>>>(*f, allow_huge);
    return check_launch("cull_big_kernel");
}

extern "C" int gs_lidar_compact(const float *sparse_depth, int32_t width, int32_t height, int32_t *idx, float *z,
                                int32_t *k_out, void *stream) {
    // idx has room for npx + ceil(npx / 1024) ints; the tail holds the per-chunk counts
    const int64_t npx = (int64_t)width * height;
    const unsigned chunks = (unsigned)((npx + LC_CHUNK - 1) / LC_CHUNK);
    if (chunks == 0) return GS_OK;
    int32_t *scratch = idx + npx;
    lidar_count_kernel<<<chunks, LC_CHUNK, 0, (cudaStream_t)stream>>>(sparse_depth, npx, scratch);
    int rc = check_launch("lidar_count_kernel");
    if (rc) return rc;
    lidar_write_kernel<<<chunks, LC_CHUNK, 0, (cudaStream_t)stream>>>(sparse_depth, npx, scratch, idx, z, k_out);
    return check_launch("lidar_write_kernel");
}
