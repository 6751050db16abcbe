// preprocess.cu -- projection / EWA covariance / SH colour / tile rectangle (sm_100a).
//
// R/gaussians.py:180-215 (project), R/rasterizer.py:445-452 (sigmoid, camera->Gaussian view
// directions, eval_sh R/gaussians.py:102-111), R/rasterizer.py:84-102 + 183-194 (influence
// radius and tile rectangle).  One thread per Gaussian; each warp stages the geometry of its 32
// parameter rows through shared memory with coalesced cp.async, and the SH columns only of the
// Gaussians that need a colour.
#include <algorithm>

#include "common.cuh"

namespace gs {

constexpr int PP_WARPS = 4;
constexpr int PP_THREADS = PP_WARPS * 32;
#ifndef PP_CTAS
#define PP_CTAS 5
#endif
constexpr int PP_CTAS_PER_SM = PP_CTAS;  // persistent grid: shared memory allows five
#ifndef PP_EVICT_FRAC
#define PP_EVICT_FRAC 1.0  // fraction of the drawable rows' SH lines marked evict-last
#endif
#define PP_STR2(x) #x
#define PP_STR(x) PP_STR2(x)

__device__ __forceinline__ void pp_cp_async16(void *smem, const void *gmem) {
    const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(sa), "l"(gmem));
}
__device__ __forceinline__ void pp_cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void pp_cp_wait_1() { asm volatile("cp.async.wait_group 1;\n" ::: "memory"); }

// Per warp, batches of 32 Gaussians flow through a software pipeline (two geometry slots):
//   A  the geometry chunks (floats 0-15 of each row: pos, log_scale, quat, opacity logit,
//      sh_low, sh_high[0]) of batch b+1 stream in (cp.async) while batch b is projected,
//      its radius / rectangle computed and its small footprints culled;
//   SH the remaining 176 B of a row (sh_high[0..14], floats 16-58) are fetched only for the
//      Gaussians that need a colour, issued once batch b's geometry is known, and consumed one
//      iteration later (colour of batch b-1), so the fetch latency hides behind batch b+1.
// Which Gaussians need a colour: every one in front of the camera for the reference-shaped API
// (ctx["colors"], R/rasterizer.py:452); only those that can be blended -- kept in >= 1 tile, or
// large footprints still to be culled -- for the iteration engine (GS_PP_LAZY_SH).  The
// engine's parameter reads fall from 256 B to ~64 B for the Gaussians that are not drawn.
struct PPGeom {  // chunk c of row r at c ^ ((r >> 1) & 3): 8 consecutive rows hit distinct banks
    float4 row[32][4];
};
struct PPSh {  // 11 chunks per row, 176-B row stride (conflict-free without a swizzle)
    float4 row[32][11];
};
struct PPWarp {  // 9.6 KB: five 4-warp CTAs per SM
    PPGeom geom[2];
    PPSh sh;
};

__device__ __forceinline__ float4 pp_geom(const PPGeom &g, int r, int c) { return g.row[r][c ^ ((r >> 1) & 3)]; }
__device__ __forceinline__ void pp_cp_wait_0() { asm volatile("cp.async.wait_group 0;\n" ::: "memory"); }

// colour of one Gaussian (R/rasterizer.py:447-452, eval_sh R/gaussians.py:102-111) from its
// geometry chunks and its staged sh_high chunks
__device__ __forceinline__ float3 pp_colour(const float4 &c0, const float4 &c2, const float4 &c3, const PPSh &sh, int r,
                                            const gs_camera &cam) {
    const float u0 = c0.x - cam.center[0], u1 = c0.y - cam.center[1], u2 = c0.z - cam.center[2];
    float un = sqrtf(u0 * u0 + u1 * u1 + u2 * u2);
    if (un < 1e-12f) un = 1.0f;
    float b[16];
    const float run = 1.0f / un;
    sh_basis(u0 * run, u1 * run, u2 * run, b);
    // floats 11-15: sh_low 0-2 (c2.w, c3.x, c3.y), sh_high[0] (c3.z, c3.w)
    float acc[3] = {b[1] * c3.z, b[1] * c3.w, 0.0f};
#pragma unroll
    for (int c = 4; c < 15; c++) {  // sh_high floats 16..58
        const float4 v = sh.row[r][c - 4];
        const float e4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int e = 0; e < 4; e++) {
            const int fi = 4 * c + e - 14;  // sh_high flat index (k * 3 + channel)
            if (fi < 45) acc[fi % 3] += b[fi / 3 + 1] * e4[e];
        }
    }
    const float low[3] = {c2.w, c3.x, c3.y};
    float col[3];
#pragma unroll
    for (int c = 0; c < 3; c++) {
        const float pre = b[0] * low[c] + acc[c] + 0.5f;
        col[c] = pre > 0.0f ? pre : 0.0f;
    }
    return make_float3(col[0], col[1], col[2]);
}

// Exact cull of the small rectangles (<= GS_SMALL_CAND candidate tiles) of a warp's 32
// Gaussians, shared by the whole warp: the candidates of all flagged lanes are laid end to end
// (warp prefix sum) and each round every lane tests one (Gaussian, tile) pair -- the owner and
// its parameters fetched by shuffles -- so the warp runs at full width whatever the mix of
// rectangle sizes (a lane-serial loop over each lane's own candidates runs at the width of the
// largest).  Returns the calling lane's keep bits in candidate order (ty-major, then tx), the
// same bits and decision arithmetic as cull_rect.
__device__ __forceinline__ uint32_t warp_cull_small(bool flag, float mx, float my, float ca, float cb, float cc,
                                                    float qcut, int4 r, int width, int height) {
    const int lane = threadIdx.x & 31;
    const int nx = r.y - r.x + 1;
    const int nc = flag ? nx * (r.w - r.z + 1) : 0;
    int pre = nc;  // inclusive prefix of the candidate counts
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += y;
    }
    const int total = __shfl_sync(0xffffffffu, pre, 31);
    const int start = pre - nc;  // exclusive prefix: this lane's first pair
    uint32_t bits = 0u;
    for (int base = 0; base < total; base += 32) {
        const int idx = base + lane;
        // owner = the lane whose [start, start + nc) holds idx: the first lane with pre > idx
        int lo = 0, hi = 31;
#pragma unroll
        for (int it = 0; it < 5; it++) {
            const int mid = (lo + hi) >> 1;
            if (__shfl_sync(0xffffffffu, pre, mid) > idx) hi = mid;
            else lo = mid + 1;
        }
        const int own = lo;
        const int c = idx - __shfl_sync(0xffffffffu, start, own);
        const float omx = __shfl_sync(0xffffffffu, mx, own), omy = __shfl_sync(0xffffffffu, my, own);
        const float oca = __shfl_sync(0xffffffffu, ca, own), ocb = __shfl_sync(0xffffffffu, cb, own);
        const float occ = __shfl_sync(0xffffffffu, cc, own), oq = __shfl_sync(0xffffffffu, qcut, own);
        const int orx = __shfl_sync(0xffffffffu, r.x, own), orz = __shfl_sync(0xffffffffu, r.z, own);
        const int onx = __shfl_sync(0xffffffffu, nx, own);
        bool keep = false;
        if (idx < total) {
            const int dy = small_div(c, __frcp_rn((float)onx));
            const int tx = orx + c - dy * onx, ty = orz + dy;
            const int x0 = tx * GS_TILE, x1 = min(x0 + GS_TILE - 1, width - 1);
            const int y0 = ty * GS_TILE, y1 = min(y0 + GS_TILE - 1, height - 1);
            keep = tile_keep(omx, omy, oca, ocb, occ, oq, x0, x1, y0, y1);
        }
        const uint32_t m = __ballot_sync(0xffffffffu, keep);
        // this lane's pairs inside the round [base, base + 32)
        const int a = max(start, base) - base, e = min(start + nc, base + 32) - base;
        if (a < e) {
            const uint32_t seg = (e - a == 32) ? m : ((m >> a) & ((1u << (e - a)) - 1u));
            bits |= seg << (base + a - start);
        }
    }
    return bits;
}

// Persistent warps over batches of 32 Gaussians (pipeline above).
template <bool LAZY_SH>
__global__ void __launch_bounds__(PP_THREADS, PP_CTAS_PER_SM) preprocess_kernel(gs_frame f, const float *__restrict__ params,
                                                                const gs_view *__restrict__ view) {
    pdl_wait();
    extern __shared__ float4 pp_raw[];
    PPWarp *ws_all = reinterpret_cast<PPWarp *>(pp_raw);
    __shared__ gs_camera scam;
    if (threadIdx.x == 0) scam = view->cam;
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    PPWarp &W = ws_all[warp];
    const int64_t n = f.n;
    const int64_t nbatch = (n + 31) / 32;
    const int64_t stride = (int64_t)gridDim.x * PP_WARPS;
    const gs_camera &cam = scam;
    auto issue_geom = [&](int64_t batch, PPGeom &g) {  // 4 chunks per row, 8 rows per instruction
        const int64_t base = batch * 32;
#pragma unroll
        for (int j = 0; j < 4; j++) {
            const int r = 8 * j + (lane >> 2), c = lane & 3;
            if (base + r < n) pp_cp_async16(&g.row[r][c ^ ((r >> 1) & 3)], params + (base + r) * GS_ROW + 4 * c);
        }
        pp_cp_commit();
    };
    int64_t batch = (int64_t)blockIdx.x * PP_WARPS + warp;
    if (batch < nbatch) issue_geom(batch, W.geom[0]);
    pp_cp_commit();  // (empty) SH group of the batch before the first
    bool prev_need = false;
    int64_t prev_i = -1;
    // the previous batch's colour inputs (position, logit, sh_low, sh_high[0]) stay in registers,
    // so its geometry slot can take the next batch: two slots instead of three
    float4 pc0 = make_float4(0.f, 0.f, 0.f, 0.f), pc2 = pc0, pc3 = pc0;
    int slot = 0;
    for (; batch < nbatch; batch += stride, slot ^= 1) {
        if (batch + stride < nbatch) issue_geom(batch + stride, W.geom[slot ^ 1]);
        else pp_cp_commit();
        pp_cp_wait_1();  // this batch's geometry and the previous batch's SH chunks have landed
        __syncwarp();
        const PPGeom &G = W.geom[slot];
        const int64_t i = batch * 32 + lane;
        bool touched = false, big = false, need = false, front = false, small = false;
        Projected pr;
        double pca = 0.0, pcb = 0.0, pcc = 0.0;  // FP64 conic (the blend's factored record)
        float op = 0.0f, qcut = 0.0f, radius = -1.0f, logit = 0.0f;
        int4 rect = make_int4(0, -1, 0, -1);
        // 1) per lane: near-plane test and FP64 projection, radius and tile rectangle
        if (i < n) {
            float pk[11];
            {
                const float4 c0 = pp_geom(G, lane, 0), c1 = pp_geom(G, lane, 1), c2 = pp_geom(G, lane, 2);
                pk[0] = c0.x; pk[1] = c0.y; pk[2] = c0.z; pk[3] = c0.w;
                pk[4] = c1.x; pk[5] = c1.y; pk[6] = c1.z; pk[7] = c1.w;
                pk[8] = c2.x; pk[9] = c2.y; pk[10] = c2.z;
            }
            logit = pk[10];
            // near-plane test (R/gaussians.py:188-191)
            const float zf = (pk[0] * cam.rot_cw[6] + pk[1] * cam.rot_cw[7] + pk[2] * cam.rot_cw[8]) + cam.trans_cw[2];
            if (!(zf > GS_NEAR_CLIP)) {
                if (!LAZY_SH) {  // the engine never reads the records of Gaussians it cannot draw
                    float4 *s2 = reinterpret_cast<float4 *>(f.splat2d) + GS_SPLAT / 4 * i;
                    s2[0] = make_float4(0.f, 0.f, 0.f, 0.f);
                    s2[1] = make_float4(0.f, 0.f, zf, 0.f);
                    s2[2] = make_float4(0.f, 0.f, 0.f, 0.f);
                    s2[3] = make_float4(0.f, 0.f, 0.f, 0.f);
                    reinterpret_cast<float4 *>(f.cov2d)[i] = make_float4(0.f, 0.f, 0.f, -1.f);
                    bin_store(f, i, make_int4(0, -1, 0, -1), 0ull, 0);
                    f.valid[i] = 0;
                    f.touched[i] = 0;
                }
            } else {
                front = true;
                // FP64 projection, rounded once to fp32: mu_cam = R p + t cancels for Gaussians
                // near the 0.01 m clip plane, and fp32 would shift their whole footprint
                ProjectedT<double> pd;
                project_full<double>(pk, cam, pd);
                pr.mu[2] = (float)pd.mu[2];
                pr.mx = (float)pd.mx;
                pr.my = (float)pd.my;
                pr.c00 = (float)pd.c00;
                pr.c01 = (float)pd.c01;
                pr.c11 = (float)pd.c11;
                pr.ca = (float)pd.ca;
                pr.cb = (float)pd.cb;
                pr.cc = (float)pd.cc;
                pca = pd.ca;
                pcb = pd.cb;
                pcc = pd.cc;
                pr.valid = pd.valid;
                op = 1.0f / (1.0f + expf(-pk[10]));
                const bool active = pr.valid && tile_rect(pr.c00, pr.c01, pr.c11, op, pr.mx, pr.my, f.width,
                                                          f.height, f.tiles_x, f.tiles_y, rect, qcut, radius);
                if (!active) rect = make_int4(0, -1, 0, -1);
                const int ncand = (rect.y - rect.x + 1) * (rect.w - rect.z + 1);
                big = active && ncand > GS_SMALL_CAND;
                small = active && !big;
            }
        }
        // 2) the warp together: exact per-tile cull of the small rectangles (R/rasterizer.py:150-166),
        //    one (Gaussian, candidate tile) pair per lane and round -- large footprints go to the
        //    big_* kernels
        const uint32_t bits = warp_cull_small(small, pr.mx, pr.my, pr.ca, pr.cb, pr.cc, qcut, rect, f.width, f.height);
        // 3) per lane: outputs
        if (front) {
            const int kept = __popc(bits);
            touched = kept > 0;
            need = LAZY_SH ? (touched || big) : true;
            // the engine (LAZY_SH) writes only what the binning and the blend read: the records of
            // the Gaussians that can be drawn (kept in a tile, or large footprints still to be
            // culled); the reference-shaped API writes every record (out.ctx["proj"], R/gaussians.py:180-215)
            if (need) {
                splat_store(f.splat2d, i, pr.mx, pr.my, pca, pcb, pcc, op, pr.mu[2], qcut);
                bin_store(f, i, rect, bits, kept);
            }
            if (!LAZY_SH) {
                // (the colour, s2[2].xyz, follows one iteration later; 1 - opacity = sigmoid(-logit)
                // is kept exact for the blend's 1 - alpha)
                reinterpret_cast<float4 *>(f.cov2d)[i] = make_float4(pr.c00, pr.c01, pr.c11, radius);
                f.valid[i] = pr.valid ? 1 : 0;
                f.touched[i] = touched ? 1 : 0;
            }
            if (kept > 0)  // binning buckets
                count_kept_tiles(f.tile_scratch, reinterpret_cast<unsigned long long *>(f.tile_minkey),
                                 ((unsigned long long)__float_as_uint(pr.mu[2]) << 32) | (uint32_t)i, rect, bits,
                                 f.tiles_x);
        }
        touched_append(f, touched, (int32_t)i);
        warp_append(big, (int32_t)i, &f.counters[GS_CNT_BIG], f.big_list);
        // colour of the previous batch (its SH chunks landed with this batch's geometry)
        if (prev_need) {
            const float3 col = pp_colour(pc0, pc2, pc3, W.sh, lane, cam);
            reinterpret_cast<float4 *>(f.splat2d)[GS_SPLAT / 4 * prev_i + 2] =
                make_float4(col.x, col.y, col.z, 1.0f / (1.0f + expf(pc2.z)));
        }
        if (need) {
            pc0 = pp_geom(G, lane, 0);
            pc2 = pp_geom(G, lane, 2);
            pc3 = pp_geom(G, lane, 3);
        }
        __syncwarp();  // the SH buffer and this geometry slot are free again
        if (need) {
            const float *src = params + i * GS_ROW + 16;
            if (LAZY_SH) {
                // the engine's drawable Gaussians are (nearly) the touched ones, whose rows the
                // chain rule + Adam re-read at the end of the iteration: their lines are marked
                // evict-last, so more of them are still in L2 then (chain DRAM reads -4 %)
                uint64_t pol;
                asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, " PP_STR(PP_EVICT_FRAC) ";" : "=l"(pol));
#pragma unroll
                for (int c = 0; c < 11; c++)
                    asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;\n" ::"r"(
                                     (unsigned)__cvta_generic_to_shared(&W.sh.row[lane][c])),
                                 "l"(src + 4 * c), "l"(pol));
            } else {
#pragma unroll
                for (int c = 0; c < 11; c++) pp_cp_async16(&W.sh.row[lane][c], src + 4 * c);
            }
        }
        pp_cp_commit();
        prev_need = need;
        prev_i = i;
    }
    if (prev_need) {  // drain: the last batch's colour
        pp_cp_wait_0();
        const float3 col = pp_colour(pc0, pc2, pc3, W.sh, lane, cam);
        reinterpret_cast<float4 *>(f.splat2d)[GS_SPLAT / 4 * prev_i + 2] = make_float4(col.x, col.y, col.z, 1.0f / (1.0f + expf(pc2.z)));
    }
}

// Exact cull of the large-footprint Gaussians (> GS_SMALL_CAND candidate tiles), same decision
// as cull_rect, one warp per Gaussian (big_bands_kernel / big_exact_kernel below).  Output bitmaps: big_bits by
// candidate index (for the emit) or, for screen-covering Gaussians with a huge slot, by tile
// index (huge_mask_t row of the slot, transposed into depth order by huge_transpose_kernel).

// Per-tile bounds: 1 if every pixel of the tile has q <= qcut (its four corners, q convex),
// 0 if none has (lower bound over the rectangle, as tile_keep), -1: decide exactly.  Evaluated in
// FP64 on the fp32 inputs, so the bounds are (to ~1e-16) those of the exact quadratic; the margin
// only has to cover the fp32 evaluation error of the exact test: quad_q rounds each of its three
// terms <= 4 times (dx, dy included) and sums twice, |q_fp32 - q| <= 6u (|T1| + |T2| + |T3|) <=
// 12u (a dx^2 + c dy^2) = 7.2e-7 scale (u = 2^-24, |2b dx dy| <= a dx^2 + c dy^2).  A 2e-6 scale
// margin keeps 2.8x of that in hand.  kx ~ -cb/ca, ky ~ -cb/cc locate the edge minima: an error
// there raises the bound by a (dx err)^2 ~ 1e-14 scale, far inside the margin.
constexpr double CULL_MARGIN = 2e-6;

__device__ __forceinline__ int tile_class(float mx, float my, float ca, float cb, float cc, float qcut, float kx,
                                          float ky, int x0, int x1, int y0, int y1) {
    const double a = ca, c = cc, tb = 2.0 * (double)cb;
    const double ax0 = (double)x0 - mx, ax1 = (double)x1 - mx, ay0 = (double)y0 - my, ay1 = (double)y1 - my;
    const double xx0 = a * ax0 * ax0, xx1 = a * ax1 * ax1, yy0 = c * ay0 * ay0, yy1 = c * ay1 * ay1;
    const double margin = CULL_MARGIN * (fmax(xx0, xx1) + fmax(yy0, yy1)) + 1e-6;
    double qmax = xx0 + tb * ax0 * ay0 + yy0;
    qmax = fmax(qmax, xx1 + tb * ax1 * ay0 + yy0);
    qmax = fmax(qmax, xx0 + tb * ax0 * ay1 + yy1);
    qmax = fmax(qmax, xx1 + tb * ax1 * ay1 + yy1);
    if (qmax + margin < (double)qcut) return 1;
    if (!(ax0 <= 0.0 && ax1 >= 0.0 && ay0 <= 0.0 && ay1 >= 0.0)) {
        double qc = 1e300;
        const double ys[2] = {ay0, ay1}, xs[2] = {ax0, ax1};
#pragma unroll
        for (int k = 0; k < 2; k++) {
            const double y = ys[k];
            const double dx = fmin(fmax((double)kx * y, ax0), ax1);
            qc = fmin(qc, a * dx * dx + tb * dx * y + c * y * y);
            const double x = xs[k];
            const double dy = fmin(fmax((double)ky * x, ay0), ay1);
            qc = fmin(qc, a * x * x + tb * x * dy + c * dy * dy);
        }
        if (qc - margin > (double)qcut) return 0;
    }
    return -1;
}

// Per-Gaussian constants of the band bounds.  E(k) = {q <= k} is an ellipse: its x-extent over
// a band's rows bounds the possibly-kept tiles (k = qp = qcut + margin), and a tile whose four
// corner pixels lie in E(qm), qm = qcut - margin, has every pixel inside (q is convex).  The
// discriminants are formed in FP64 (no cancellation), the square roots in fp32: their ~1e-7
// relative error moves the extents by <= 1e-7 of the half-width, which the eps widening in x
// (1e-3 + 1e-6 (|mx| + half-width) px) covers ten times over.  The margin (CULL_MARGIN of the
// rectangle's scale) covers the fp32 evaluation error of the exact test, as in tile_class.
struct BandConst {
    double mx, my, a, b, det, inv_a, qm, qp, dymax, dyr, eps;
    bool ok;
};

__device__ __forceinline__ BandConst band_const(float mx, float my, float ca, float cb, float cc, float qcut, int4 r) {
    BandConst k;
    k.mx = mx;
    k.my = my;
    k.a = ca;
    k.b = cb;
    const double c = cc;
    k.det = k.a * c - k.b * k.b;
    const double ax = fmax(fabs((double)(r.x * GS_TILE) - k.mx), fabs((double)(r.y * GS_TILE + GS_TILE) - k.mx));
    const double ay = fmax(fabs((double)(r.z * GS_TILE) - k.my), fabs((double)(r.w * GS_TILE + GS_TILE) - k.my));
    const double margin = CULL_MARGIN * (k.a * ax * ax + c * ay * ay) + 1e-6;
    k.qm = (double)qcut - margin;
    k.qp = (double)qcut + margin;
    k.ok = k.a > 0.0 && c > 0.0 && k.det > 0.0 && k.qp > 0.0 && isfinite(k.det) && isfinite(margin);
    k.inv_a = k.ok ? 1.0 / k.a : 0.0;
    k.dymax = k.ok ? (double)sqrtf((float)(k.a * k.qp / k.det)) * (1.0 + 1e-6) : 0.0;
    k.dyr = k.ok ? -k.b / c * (double)sqrtf((float)(k.qp * c / k.det)) : 0.0;  // dy of the rightmost point
    const double hw = k.ok ? (double)sqrtf((float)(k.qp * c / k.det)) : 0.0;
    k.eps = 1e-3 + 1e-6 * (fabs(k.mx) + hw);
    return k;
}

// (pl, kl, kr, pr): tiles outside [pl, pr] surely culled, [kl, kr] surely kept (empty if
// kl > kr), the rest ambiguous
__device__ __forceinline__ int4 band_ranges(const BandConst &k, int ty, int4 r, int width, int height, int tiles_x) {
    const int y0 = ty * GS_TILE, y1 = min(y0 + GS_TILE - 1, height - 1);
    if (!k.ok) return make_int4(r.x, r.y + 1, r.y, r.y);
    const double D0 = (double)y0 - k.my, D1 = (double)y1 - k.my;
    const double lo = fmax(D0, -k.dymax), hi = fmin(D1, k.dymax);
    if (lo > hi) return make_int4(r.x, r.y + 1, r.y, r.x - 1);  // the band misses E(qp)
    const double dyr = fmin(fmax(k.dyr, lo), hi), dyl = fmin(fmax(-k.dyr, lo), hi);
    const double sr = sqrtf((float)fmax(0.0, k.a * k.qp - k.det * dyr * dyr));
    const double sl = sqrtf((float)fmax(0.0, k.a * k.qp - k.det * dyl * dyl));
    const double xr = k.mx + (-k.b * dyr + sr) * k.inv_a + k.eps;
    const double xl = k.mx + (-k.b * dyl - sl) * k.inv_a - k.eps;
    // tile t spans pixels [16t, min(16t+15, W-1)]: possible iff 16t+15 >= xl and 16t <= xr
    const int pl = (int)fmax((double)r.x, fmin((double)r.y + 1.0, ceil((xl - 15.0) * 0.0625)));
    const int pr = (int)fmin((double)r.y, fmax((double)r.x - 1.0, floor(xr * 0.0625)));
    if (pl > pr) return make_int4(r.x, r.y + 1, r.y, r.x - 1);
    int4 out = make_int4(pl, pr + 1, pr, pr);
    if (k.qm > 0.0) {
        const double d0 = k.a * k.qm - k.det * D0 * D0, d1 = k.a * k.qm - k.det * D1 * D1;
        if (d0 > 0.0 && d1 > 0.0) {
            const double s0 = sqrtf((float)d0), s1 = sqrtf((float)d1);
            const double il = k.mx + fmax(-k.b * D0 - s0, -k.b * D1 - s1) * k.inv_a + k.eps;
            const double ir = k.mx + fmin(-k.b * D0 + s0, -k.b * D1 + s1) * k.inv_a - k.eps;
            if (il <= ir) {
                int kl = (int)fmax(-1.0, fmin(1e9, ceil(il * 0.0625)));
                int kr = ((double)(width - 1) <= ir) ? tiles_x - 1
                                                     : (int)fmax(-2.0, fmin(1e9, floor((ir - 15.0) * 0.0625)));
                kl = max(kl, pl);
                kr = min(kr, pr);
                if (kl <= kr) out = make_int4(pl, kl, kr, pr);
            }
        }
    }
    return out;
}

// Sets bits [b0, b1] of a warp's shared-memory bitmap (bands of one Gaussian share words).
__device__ __forceinline__ void set_bit_range(uint32_t *bits, int b0, int b1) {
    for (int w = b0 >> 5; w <= (b1 >> 5); w++) {
        const int lo_b = max(b0, w << 5) - (w << 5), hi_b = min(b1, (w << 5) + 31) - (w << 5);
        const uint32_t m = (hi_b - lo_b == 31) ? 0xffffffffu : (((1u << (hi_b - lo_b + 1)) - 1u) << lo_b);
        atomicOr(&bits[w], m);
    }
}

// Exact resolution of up to 32 (tile, Gaussian) pairs held one per lane: cls = tile_class on
// entry (1 kept, 0 culled, -1 open); the open tiles are decided four per round, 8 lanes per tile
// and two pixel rows per lane (row_hits), with the owner's parameters fetched by shuffles.
__device__ __forceinline__ int resolve_open(int cls, const SplatCull &s, int x0, int x1, int y0, int y1) {
    const int lane = threadIdx.x & 31, grp = lane >> 3, sub = lane & 7;
    unsigned amb = __ballot_sync(0xffffffffu, cls < 0);
    while (amb) {
        int mine = -1;
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int l = amb ? __ffs(amb) - 1 : -1;
            if (l >= 0) amb &= amb - 1u;
            if (k == grp) mine = l;
        }
        const int src = mine >= 0 ? mine : 0;
        const float smx = __shfl_sync(0xffffffffu, s.mx, src), smy = __shfl_sync(0xffffffffu, s.my, src);
        const float sca = __shfl_sync(0xffffffffu, s.ca, src), scb = __shfl_sync(0xffffffffu, s.cb, src);
        const float scc = __shfl_sync(0xffffffffu, s.cc, src), sq = __shfl_sync(0xffffffffu, s.qcut, src);
        const int sx0 = __shfl_sync(0xffffffffu, x0, src), sx1 = __shfl_sync(0xffffffffu, x1, src);
        const int sy0 = __shfl_sync(0xffffffffu, y0, src), sy1 = __shfl_sync(0xffffffffu, y1, src);
        bool hit = false;
        if (mine >= 0) {
            const int ya = sy0 + sub, yb = sy0 + sub + 8;
            hit = (ya <= sy1 && row_hits(smx, smy, sca, scb, scc, sq, sx0, sx1, ya)) ||
                  (yb <= sy1 && row_hits(smx, smy, sca, scb, scc, sq, sx0, sx1, yb));
        }
        const unsigned bal = __ballot_sync(0xffffffffu, hit);
#pragma unroll
        for (int k = 0; k < 4; k++) {
            const int owner = __shfl_sync(0xffffffffu, mine, 8 * k);
            if (lane == owner && owner >= 0) cls = ((bal >> (8 * k)) & 0xffu) ? 1 : 0;
        }
    }
    return cls;
}

__device__ __forceinline__ uint64_t big_key(const gs_frame &f, int g) {
    return ((uint64_t)__float_as_uint(splat_depth(f.splat2d, g)) << 32) | (uint32_t)g;
}

// Publishes one large-footprint Gaussian once its bitmap is complete (the whole warp calls it
// with the same arguments; `bits` = its bitmap, shared or global): kept count, touched and the
// non-huge kept tiles into the binning's bucket counts.  The touched-list entry and the huge key
// staging are reserved per CTA by the callers.  Returns the kept count.
template <bool GLOBAL>
__device__ __forceinline__ int big_publish(const gs_frame &f, int g, int slot, const uint32_t *bits, int nwords,
                                           int4 r) {
    const int lane = threadIdx.x & 31;
    // rows in global memory were completed by other SMs' atomics: read them at L2
    auto word = [&](int w) -> uint32_t { return GLOBAL ? __ldcg(bits + w) : bits[w]; };
    int kept = 0;
    for (int w = lane; w < nwords; w += 32) kept += __popc(word(w));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) kept += __shfl_xor_sync(0xffffffffu, kept, o);
    const bool t = kept > 0;
    const uint64_t key = big_key(f, g);
    if (lane == 0) {
        bin_rec(f)[g].kept = (slot >= 0 && t) ? -(1 + slot) : kept;  // kept < 0 encodes the huge slot
        f.touched[g] = t;
    }
    if (t && slot < 0) {  // per-tile bucket counts (bitmap by candidate index)
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        for (int c = lane; c < ncand; c += 32) {
            if ((word(c >> 5) >> (c & 31)) & 1u) {
                const int tile = (r.z + c / nx) * f.tiles_x + r.x + c % nx;
                atomicAdd(&f.tile_scratch[tile], 1);
                atomicMin(reinterpret_cast<unsigned long long *>(f.tile_minkey) + tile, (unsigned long long)key);
            }
        }
    }
    return kept;
}

// Exact cull of the large-footprint Gaussians in two launches:
//   big_bands_kernel  one warp per Gaussian: lane 0 reserves the output (a huge slot: kept tiles
//                     by tile index in huge_mask_t; or a big_bits row by candidate index); lane j
//                     takes bands j, j + 32, ...: the band bounds give a run of surely-kept tiles
//                     (set in the warp's shared-memory bitmap) between runs of surely-culled
//                     ones; the ambiguous tiles of the 32 bands are laid end to end (warp prefix
//                     sum) and queued for big_exact_kernel (the long tail -- needle-shaped
//                     near-plane footprints leave thousands of tiles within the bounds' margin --
//                     would serialise a warp on one Gaussian; measured: resolving up to 64 tiles
//                     in the warp made this kernel 2.3x slower than queueing them all).  Only a
//                     Gaussian without an output row (big_bits overflow) or a full queue is
//                     resolved here.  The bitmap goes out as full rows (coalesced, no clearing
//                     pass); a Gaussian without queued tiles is published at once (touched-list
//                     and huge-list reservations aggregated per CTA), the others keep their
//                     queued count in kept[g];
//   big_exact_kernel  thread per queued tile: tile_class, the open tiles decided 8 lanes per
//                     tile; kept bits OR-ed into the Gaussian's row; the thread that retires a
//                     Gaussian's last queued tile publishes it (with its warp).
// Same decisions as tile_keep (bit-exact against the fp32 oracle restatement).
constexpr int BC_WARPS = 8;

__global__ void __launch_bounds__(BC_WARPS * 32, 2) big_bands_kernel(gs_frame f, int allow_huge) {
    pdl_wait();
    extern __shared__ uint32_t bc_raw[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int T = f.tiles_x * f.tiles_y, tw = (T + 31) >> 5;
    uint32_t *bm = bc_raw + warp * tw;
    const int64_t nb = f.counters[GS_CNT_BIG];
    const int64_t cap = f.cull_queue_cap;
    int2 *queue = reinterpret_cast<int2 *>(f.cull_queue);
    __shared__ int s_g[BC_WARPS], s_kept[BC_WARPS], s_slot[BC_WARPS];
    // CTA-uniform trip count: the touched-list / huge-list reservations are made once per CTA
    // and round (same-address atomics from every warp serialise in L2)
    for (int64_t b0 = (int64_t)blockIdx.x * BC_WARPS; b0 < nb; b0 += (int64_t)gridDim.x * BC_WARPS) {
        const int64_t b = b0 + warp;
        if (lane == 0) s_kept[warp] = 0;
        if (b < nb) {
            const int g = f.big_list[b];
            const int4 r = bin_rec(f)[g].rect;
            const SplatCull s = splat_cull(f.splat2d, g);
            const int nx = r.y - r.x + 1, nbands = r.w - r.z + 1, ncand = nx * nbands;
            // huge slot = the Gaussian's big-list index (no reservation atomic; slots of the others
            // stay unused)
            const int slot = (allow_huge && ncand > GS_HUGE_CAND && b < GS_HUGE_CAP) ? (int)b : -1;
            long long base = -1;
            if (lane == 0) {
                if (slot < 0) {  // bitmap by candidate index for the emit (overflow: the emit re-culls)
                    const int words = (ncand + 31) >> 5;
                    const long long bb = atomicAdd(&f.counters[GS_CNT_BIG_BITS], words);
                    base = bb + words > f.big_bits_words ? -1 : bb;
                }
            }
            base = __shfl_sync(0xffffffffu, base, 0);
            uint32_t *row = slot >= 0 ? f.huge_mask_t + (int64_t)slot * tw : (base >= 0 ? f.big_bits + base : nullptr);
            const int nwords = slot >= 0 ? tw : (ncand + 31) >> 5;
            for (int w = lane; w < nwords; w += 32) bm[w] = 0u;
            __syncwarp();
            const BandConst K = band_const(s.mx, s.my, s.ca, s.cb, s.cc, s.qcut, r);
            const float kx = __fdividef(-s.cb, s.ca), ky = __fdividef(-s.cb, s.cc);
            int queued = 0;
            for (int bi0 = 0; bi0 < nbands; bi0 += 32) {
                const int bi = bi0 + lane, ty = r.z + bi;
                int4 br = make_int4(0, 1, 0, -1);  // nothing
                if (bi < nbands) br = band_ranges(K, ty, r, f.width, f.height, f.tiles_x);
                const int bit0 = slot >= 0 ? ty * f.tiles_x : bi * nx - r.x;  // bit of tile tx: bit0 + tx
                const bool has_keep = br.y <= br.z;
                if (has_keep) set_bit_range(bm, bit0 + br.y, bit0 + br.z);
                // ambiguous: [pl, kl) and (kr, pr] (all of [pl, pr] when nothing is surely kept)
                const int left = has_keep ? br.y - br.x : max(0, br.w - br.x + 1);
                const int namb = has_keep ? left + (br.w - br.z) : left;
                int pre = namb;  // inclusive prefix over the warp's bands
    #pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    const int y = __shfl_up_sync(0xffffffffu, pre, o);
                    if (lane >= o) pre += y;
                }
                const int total = __shfl_sync(0xffffffffu, pre, 31);
                const int start = pre - namb;
                // many: queue them (a row must exist for the exact kernel to OR into)
                long long q0 = 0;
                const bool to_queue = total > 0 && row != nullptr;
                if (to_queue) {
                    if (lane == 0) q0 = atomicAdd(&f.counters[GS_CNT_CULLQ1], total);
                    q0 = __shfl_sync(0xffffffffu, q0, 0);
                    if (q0 + total > cap) q0 = -1;  // queue full: resolve here
                }
                if (to_queue && q0 >= 0) {
                    for (int c = 0; c < namb; c++) {
                        const int tx = c < left ? br.x + c : br.z + 1 + (c - left);
                        queue[q0 + start + c] = make_int2((int)b, (int)(((uint32_t)tx << 16) | (uint32_t)ty));
                    }
                    queued += total;
                    continue;
                }
                for (int p0 = 0; p0 < total; p0 += 32) {
                    const int idx = p0 + lane;
                    int lo = 0, hi = 31;  // owner band = the first lane with pre > idx
    #pragma unroll
                    for (int it = 0; it < 5; it++) {
                        const int mid = (lo + hi) >> 1;
                        if (__shfl_sync(0xffffffffu, pre, mid) > idx) hi = mid;
                        else lo = mid + 1;
                    }
                    const int own = lo;
                    const int c = idx - __shfl_sync(0xffffffffu, start, own);
                    const int oleft = __shfl_sync(0xffffffffu, left, own), obx = __shfl_sync(0xffffffffu, br.x, own);
                    const int obz = __shfl_sync(0xffffffffu, br.z, own), obit = __shfl_sync(0xffffffffu, bit0, own);
                    const int tx = c < oleft ? obx + c : obz + 1 + (c - oleft);
                    const int oty = r.z + bi0 + own;
                    const int x0 = tx * GS_TILE, y0 = oty * GS_TILE;
                    const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
                    int cls = 0;
                    if (idx < total) cls = tile_class(s.mx, s.my, s.ca, s.cb, s.cc, s.qcut, kx, ky, x0, x1, y0, y1);
                    cls = resolve_open(cls, s, x0, x1, y0, y1);
                    if (cls > 0) {
                        const int bit = obit + tx;
                        atomicOr(&bm[bit >> 5], 1u << (bit & 31));
                    }
                }
            }
            __syncwarp();
            if (row)
                for (int w = lane; w < nwords; w += 32) row[w] = bm[w];
            if (lane == 0) {
                f.big_slot[b] = slot;
                bin_rec(f)[g].bits = (uint64_t)base;  // bitmap base for large footprints (-1: none)
                if (queued) bin_rec(f)[g].kept = queued;  // countdown of big_exact_kernel
            }
            if (!queued) {
                const int kept = big_publish<false>(f, g, slot, bm, nwords, r);
                if (lane == 0) {
                    s_g[warp] = g;
                    s_kept[warp] = kept;
                    s_slot[warp] = slot;
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            int nt = 0, nh = 0, e = 0;
            for (int w = 0; w < BC_WARPS; w++)
                if (s_kept[w] > 0) {
                    nt++;
                    if (s_slot[w] >= 0) {
                        nh++;
                        e += s_kept[w];
                    }
                }
            if (nt) {
                int tb = atomicAdd(&f.counters[GS_CNT_TOUCHED], nt);
                int hb = nh ? atomicAdd(&f.counters[GS_CNT_HUGE_N], nh) : 0;
                if (e) atomicAdd(&f.counters[GS_CNT_HUGE_E], e);
                for (int w = 0; w < BC_WARPS; w++)
                    if (s_kept[w] > 0) {
                        f.touched_list[tb] = s_g[w];
                        splat_set_slot(f.splat2d, s_g[w], tb++);
                        if (s_slot[w] >= 0) {
                            if (hb < GS_HUGE_CAP) reinterpret_cast<uint64_t *>(f.huge + HSTAGE)[hb] = big_key(f, s_g[w]);
                            hb++;
                        }
                    }
            }
        }
        __syncthreads();  // the warps' bitmaps and the CTA's records are free for the next round
    }
}

__global__ void __launch_bounds__(256) big_exact_kernel(gs_frame f) {
    pdl_wait();
    const int64_t cap = f.cull_queue_cap;
    const int64_t nq = min((int64_t)f.counters[GS_CNT_CULLQ1], cap);
    const int2 *queue = reinterpret_cast<const int2 *>(f.cull_queue);
    const int tw = (f.tiles_x * f.tiles_y + 31) >> 5;
    const int lane = threadIdx.x & 31;
    // the Gaussians this CTA publishes in a round: their touched-list / huge-list reservations are
    // made once per CTA (same-address counter atomics from every publishing warp serialise in L2)
    __shared__ int s_np, s_tb, s_hb, s_wh[8], s_we[8];
    __shared__ int s_pg[256], s_pk[256], s_ps[256];
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < nq; i0 += (int64_t)gridDim.x * blockDim.x) {
        if (threadIdx.x == 0) s_np = 0;
        __syncthreads();
        const int64_t i = i0 + threadIdx.x;  // uniform trip count: the exact test is warp-wide
        int cls = 0, g = 0, b = 0, slot = -1;
        uint32_t *row = nullptr;
        SplatCull s{0.f, 0.f, 1.f, 0.f, 1.f, 0.f};
        int4 r = make_int4(0, -1, 0, -1);
        int x0 = 0, x1 = 0, y0 = 0, y1 = -1, bit = 0;
        if (i < nq) {
            const int2 e = queue[i];
            b = e.x;
            g = f.big_list[b];
            slot = f.big_slot[b];
            r = bin_rec(f)[g].rect;
            s = splat_cull(f.splat2d, g);
            const int tx = (int)((uint32_t)e.y >> 16), ty = e.y & 0xffff;
            row = slot >= 0 ? f.huge_mask_t + (int64_t)slot * tw : f.big_bits + (int64_t)bin_rec(f)[g].bits;
            bit = slot >= 0 ? ty * f.tiles_x + tx : (ty - r.z) * (r.y - r.x + 1) + (tx - r.x);
            x0 = tx * GS_TILE;
            y0 = ty * GS_TILE;
            x1 = min(x0 + GS_TILE - 1, f.width - 1);
            y1 = min(y0 + GS_TILE - 1, f.height - 1);
            cls = tile_class(s.mx, s.my, s.ca, s.cb, s.cc, s.qcut, __fdividef(-s.cb, s.ca), __fdividef(-s.cb, s.cc), x0,
                             x1, y0, y1);
        }
        cls = resolve_open(cls, s, x0, x1, y0, y1);
        // kept bits: one atomicOr per distinct bitmap word of the warp (queue entries of one
        // Gaussian are contiguous, so a warp's tiles share few words)
        uint32_t *wp = row + (bit >> 5);
        const unsigned same_word = __match_any_sync(0xffffffffu, (unsigned long long)wp);
        const uint32_t m = __reduce_or_sync(same_word, (i < nq && cls > 0) ? 1u << (bit & 31) : 0u);
        if (i < nq && m && lane == __ffs(same_word) - 1) atomicOr(wp, m);
        __threadfence();  // the bits are visible before the countdown that may retire the Gaussian
        // countdown: one atomicSub per distinct Gaussian of the warp; the lane that retires a
        // Gaussian's last queued tile publishes it (with its warp)
        const unsigned same_g = __match_any_sync(0xffffffffu, i < nq ? g : -1);
        bool last = false;
        if (i < nq && lane == __ffs(same_g) - 1) last = atomicSub(&bin_rec(f)[g].kept, __popc(same_g)) == __popc(same_g);
        unsigned fin = __ballot_sync(0xffffffffu, last);
        if (fin) __threadfence();
        while (fin) {  // the warp publishes each Gaussian whose last queued tile one of its lanes retired
            const int l = __ffs(fin) - 1;
            fin &= fin - 1u;
            const int gl = __shfl_sync(0xffffffffu, g, l), sl = __shfl_sync(0xffffffffu, slot, l);
            const int4 rl = make_int4(__shfl_sync(0xffffffffu, r.x, l), __shfl_sync(0xffffffffu, r.y, l),
                                      __shfl_sync(0xffffffffu, r.z, l), __shfl_sync(0xffffffffu, r.w, l));
            const uint32_t *rowl = reinterpret_cast<const uint32_t *>(__shfl_sync(0xffffffffu, (unsigned long long)row, l));
            const int nwords = sl >= 0 ? tw : ((rl.y - rl.x + 1) * (rl.w - rl.z + 1) + 31) >> 5;
            const int kept = big_publish<true>(f, gl, sl, rowl, nwords, rl);
            if (lane == 0 && kept > 0) {
                const int p = atomicAdd(&s_np, 1);  // (<= 256: one per retired queue entry)
                s_pg[p] = gl;
                s_pk[p] = kept;
                s_ps[p] = sl;
            }
        }
        __syncthreads();
        const int np = s_np;
        if (np > 0) {  // (CTA-uniform) record p is thread p's
            const int p = threadIdx.x, warp = threadIdx.x >> 5;
            const bool hug = p < np && s_ps[p] >= 0;
            const unsigned hm = __ballot_sync(0xffffffffu, hug);
            int e = hug ? s_pk[p] : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) e += __shfl_xor_sync(0xffffffffu, e, o);
            if (lane == 0) {
                s_wh[warp] = __popc(hm);
                s_we[warp] = e;
            }
            __syncthreads();
            if (threadIdx.x == 0) {
                int nh = 0, et = 0;
                for (int w = 0; w < 8; w++) {  // exclusive prefix of the warps' huge counts, in place
                    const int c = s_wh[w];
                    s_wh[w] = nh;
                    nh += c;
                    et += s_we[w];
                }
                s_tb = atomicAdd(&f.counters[GS_CNT_TOUCHED], np);
                s_hb = nh ? atomicAdd(&f.counters[GS_CNT_HUGE_N], nh) : 0;
                if (et) atomicAdd(&f.counters[GS_CNT_HUGE_E], et);
            }
            __syncthreads();
            if (p < np) {
                const int g = s_pg[p], ts = s_tb + p;
                f.touched_list[ts] = g;
                splat_set_slot(f.splat2d, g, ts);
                // kept screen-covering Gaussians: a staging slot each for the binning's huge sort
                // (binning.cu, HKEYS; the sort is by key, so the staging order is free)
                if (hug) {
                    const int h = s_hb + s_wh[warp] + __popc(hm & ((1u << lane) - 1u));
                    if (h < GS_HUGE_CAP) reinterpret_cast<uint64_t *>(f.huge + HSTAGE)[h] = big_key(f, g);
                }
            }
        }
        __syncthreads();  // s_np and the records are free for the next round
    }
}

// gs_project: full projection records for the project() API (R/gaussians.py:180-215)
__global__ void project_kernel(const float *__restrict__ params, int64_t n, const gs_camera *__restrict__ camp,
                               float *mu_cam, float *mean2d, float *cov2d, float *conic, float *depth,
                               uint8_t *valid, float *jproj, float *mmat, float *cov3d) {
    pdl_wait();
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
    pdl_wait();
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
    pdl_wait();
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
    if (kept > 0)  // binning buckets
        count_kept_tiles(f.tile_scratch, reinterpret_cast<unsigned long long *>(f.tile_minkey),
                         ((unsigned long long)__float_as_uint(depth[i]) << 32) | (uint32_t)i, rect, bits, f.tiles_x);
    splat_store(f.splat2d, i, mx, my, ca, cb, cc, o, depth[i], qcut);
    reinterpret_cast<float4 *>(f.splat2d)[GS_SPLAT / 4 * i + 2] = colors ? make_float4(colors[3 * i], colors[3 * i + 1], colors[3 * i + 2], 1.0f - o)
                   : make_float4(0.f, 0.f, 0.f, 1.0f - o);
    reinterpret_cast<float4 *>(f.cov2d)[i] = make_float4(c00, c01, c11, radius);
    bin_store(f, i, rect, bits, kept);
    f.valid[i] = v;
    f.touched[i] = kept > 0;
}

// the touched and large-footprint lists of the pack path (unordered; consumers are order
// independent)
__global__ void touched_list_kernel(gs_frame f) {
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int k = i < f.n ? bin_rec(f)[i].kept : 0;
    if (k < 0) bin_rec(f)[i].kept = 0;
    touched_append(f, k > 0, (int32_t)i);
    warp_append(k < 0, (int32_t)i, &f.counters[GS_CNT_BIG], f.big_list);
}

// Ordered compaction of sparse_depth > 0 into the K-list (np.flatnonzero order), two passes:
// per-chunk counts, then each chunk sums its predecessors' counts and writes in order.
constexpr int LC_CHUNK = 1024;

__global__ void lidar_count_kernel(const float *__restrict__ sparse, int64_t npx, int32_t *chunk_cnt) {
    pdl_wait();
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
    pdl_wait();
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

static int launch_big_cull(const gs_frame *f, int allow_huge, cudaStream_t st) {
    const int tw = (f->tiles_x * f->tiles_y + 31) >> 5;
    launch_pdl(big_bands_kernel, 2 * 148, BC_WARPS * 32, (size_t)BC_WARPS * tw * sizeof(uint32_t), st, *f, allow_huge);
    int rc = check_launch("big_bands_kernel");
    if (rc) return rc;
    launch_pdl(big_exact_kernel, 8 * 148, 256, 0, st, *f);
    return check_launch("big_exact_kernel");
}

namespace gs {
// a frame's per-view accumulators back to their initial state: counters 0, per-tile bucket and
// huge counts 0, per-tile smallest bucketed keys ~0
__global__ void __launch_bounds__(256) frame_reset_kernel(gs_frame f) {
    pdl_wait();
    const int T1 = f.tiles_x * f.tiles_y + 1;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < max(2 * T1, GS_CNT_SLOTS * 2); i += gridDim.x * blockDim.x) {
        if (i < 2 * T1) f.tile_scratch[i] = 0;
        if (i < T1) reinterpret_cast<unsigned long long *>(f.tile_minkey)[i] = ~0ull;
        if (i < GS_CNT_SLOTS * 2) f.counters[i] = 0;
    }
}
}  // namespace gs

static int launch_frame_reset(const gs_frame *f, cudaStream_t st) {
    const int T1 = f->tiles_x * f->tiles_y + 1;
    const unsigned blocks = (unsigned)std::min(148, (2 * T1 + 255) / 256);
    launch_pdl(frame_reset_kernel, blocks, 256, 0, st, *f);
    return check_launch("frame_reset_kernel");
}

extern "C" int gs_preprocess(const gs_frame *f, const float *params, const gs_view *view, void *stream) {
    return gs_preprocess_ex(f, params, view, 0, stream);
}

extern "C" int gs_preprocess_ex(const gs_frame *f, const float *params, const gs_view *view, int32_t flags,
                                void *stream) {
    if (!f || !params || !view || (flags & ~GS_PP_LAZY_SH)) {
        set_error("gs_preprocess: null argument or unknown flags");
        return GS_ERR_ARG;
    }
    // counters, per-tile bucket / huge counts (gs_bin reads them) and smallest keys: one kernel
    // (a graph node that keeps the launch chain programmatic, unlike three memsets)
    int rc0 = launch_frame_reset(f, (cudaStream_t)stream);
    if (rc0) return rc0;
    if (f->n == 0) return GS_OK;
    if (flags & GS_PP_LAZY_SH)
        launch_pdl(preprocess_kernel<true>, PP_CTAS_PER_SM * 148, PP_THREADS, PP_WARPS * sizeof(PPWarp), (cudaStream_t)stream, *f, params,
                                                                                                         view);
    else
        launch_pdl(preprocess_kernel<false>, PP_CTAS_PER_SM * 148, PP_THREADS, PP_WARPS * sizeof(PPWarp), (cudaStream_t)stream, *f, params,
                                                                                                          view);
    int rc = check_launch("preprocess_kernel");
    if (rc) return rc;
    // screen-covering Gaussians are binned per tile by bitmap (up to GS_HUGE_CAP per view)
    return launch_big_cull(f, 1, (cudaStream_t)stream);
}

extern "C" int gs_project(const float *params, int64_t n, const gs_camera *cam, float *mu_cam, float *mean2d,
                          float *cov2d, float *conic, float *depth, uint8_t *valid, float *jproj, float *mmat,
                          float *cov3d, void *stream) {
    if (n == 0) return GS_OK;
    launch_pdl(project_kernel, (unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream, 
        params, n, cam, mu_cam, mean2d, cov2d, conic, depth, valid, jproj, mmat, cov3d);
    return check_launch("project_kernel");
}

extern "C" int gs_eval_sh(const float *sh_low, const float *sh_high, const float *dirs, int64_t n, float *colors,
                          float *preclamp, void *stream) {
    if (n == 0) return GS_OK;
    launch_pdl(eval_sh_kernel, (unsigned)((n + 127) / 128), 128, 0, (cudaStream_t)stream, sh_low, sh_high, dirs, n, colors,
                                                                                   preclamp);
    return check_launch("eval_sh_kernel");
}

extern "C" int gs_pack_splats(const gs_frame *f, const float *mean2d, const float *conic, const float *cov2d3,
                              const float *opacity, const float *depth, const uint8_t *valid, const float *colors,
                              void *stream) {
    int rc0 = launch_frame_reset(f, (cudaStream_t)stream);
    if (rc0) return rc0;
    if (f->n == 0) return GS_OK;
    launch_pdl(pack_kernel, (unsigned)((f->n + 127) / 128), 128, 0, (cudaStream_t)stream, *f, mean2d, conic, cov2d3, opacity,
                                                                                   depth, valid, colors);
    int rc = check_launch("pack_kernel");
    if (rc) return rc;
    launch_pdl(touched_list_kernel, (unsigned)((f->n + 255) / 256), 256, 0, (cudaStream_t)stream, *f);
    if ((rc = check_launch("touched_list_kernel"))) return rc;
    // screen-covering Gaussians are binned per tile by bitmap (up to GS_HUGE_CAP per view)
    return launch_big_cull(f, 1, (cudaStream_t)stream);
}

extern "C" int gs_lidar_compact(const float *sparse_depth, int32_t width, int32_t height, int32_t *idx, float *z,
                                int32_t *k_out, void *stream) {
    // idx has room for npx + ceil(npx / 1024) ints; the tail holds the per-chunk counts
    const int64_t npx = (int64_t)width * height;
    const unsigned chunks = (unsigned)((npx + LC_CHUNK - 1) / LC_CHUNK);
    if (chunks == 0) return GS_OK;
    int32_t *scratch = idx + npx;
    launch_pdl(lidar_count_kernel, chunks, LC_CHUNK, 0, (cudaStream_t)stream, sparse_depth, npx, scratch);
    int rc = check_launch("lidar_count_kernel");
    if (rc) return rc;
    launch_pdl(lidar_write_kernel, chunks, LC_CHUNK, 0, (cudaStream_t)stream, sparse_depth, npx, scratch, idx, z, k_out);
    return check_launch("lidar_write_kernel");
}

namespace gs {
void init_preprocess_attrs() {
    cudaFuncSetAttribute(preprocess_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(PP_WARPS * sizeof(PPWarp)));
    cudaFuncSetAttribute(preprocess_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(PP_WARPS * sizeof(PPWarp)));
    cudaFuncSetAttribute(big_bands_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(BC_WARPS * ((GS_MAX_TILES + 31) / 32) * sizeof(uint32_t)));
    cudaFuncSetAttribute(preprocess_kernel<false>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(preprocess_kernel<true>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}
}  // namespace gs
