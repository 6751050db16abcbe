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
#include <algorithm>

#include "tilelist.cuh"

namespace gs {

constexpr int RT = 256;  // threads per tile CTA = pixels per tile
constexpr float NEG_HALF_LOG2E = -0.5f * GS_LOG2E;

// q = a (dx + beta dy)^2 + gamma dy^2 (the factored conic of the splat record, common.cuh);
// au = a (dx + beta dy) = a dx + b dy is returned for the mean gradient
__device__ __forceinline__ float quad(float a, float beta, float gamma, float dx, float dy, float &au) {
    const float u = fmaf(beta, dy, dx);
    au = a * u;
    return fmaf(au, u, gamma * dy * dy);
}

// alpha = min(o e^{-q/2}, 0.99) (R/rasterizer.py:270-272) and 1 - alpha.  1 - alpha is formed
// with one rounding (FMA) and is exactly 0.01 on the clamp, so the transmittance product does
// not pick up the cancellation of 1 - 0.99f.  (omo = 1 - o is carried in the splat record for
// the higher-accuracy variant 1 - o e = (1 - e) + (1 - o) e.)
// fast_ex2 / fast_rcp (common.cuh): MUFU without the IEEE range and rounding fix-ups (relative
// error ~2^-22; results below 2^-126 flush to 0, i.e. alpha < 1e-38): the blend and its adjoint
// use the same alpha.

__device__ __forceinline__ float blend_exp(float q) { return fast_ex2(NEG_HALF_LOG2E * q); }

__device__ __forceinline__ void alpha_oma(float op, float omo, float q, float &araw, float &alpha, float &oma) {
    (void)omo;
    const float e = blend_exp(q);
    araw = op * e;
    if (araw > GS_ALPHA_CLAMP) {
        alpha = GS_ALPHA_CLAMP;
        oma = 0.01f;
    } else {
        alpha = araw;
        oma = fmaf(-op, e, 1.0f);
    }
}

// Paired fp32 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2: one instruction, two lanes): the forward
// and backward threads own two pixels of one column (rows y and y + 8), whose blend / replay
// steps are the same instruction stream on different data.
__device__ __forceinline__ float2 f2(float v) { return make_float2(v, v); }
__device__ __forceinline__ float2 fma2(float2 a, float2 b, float2 c) { return __ffma2_rn(a, b, c); }
__device__ __forceinline__ float2 mul2(float2 a, float2 b) { return __fmul2_rn(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }

// alpha, 1 - alpha and the exponential of an entry for two pixels of one column, with exactly
// the operations of the scalar quad() / blend_exp() / alpha_oma() (IEEE per lane, same order), so
// every kernel sees bit-identical alphas
__device__ __forceinline__ void alpha2(const float4 &A, const float4 &B, float dx, float2 dy, float2 &au, float2 &e,
                                       float2 &alpha, float2 &om, bool &c0, bool &c1) {
    const float a = A.z, beta = A.w, gamma = B.x, op = B.y;
    const float2 u = fma2(f2(beta), dy, f2(dx));
    au = mul2(f2(a), u);
    const float2 q = fma2(au, u, mul2(mul2(f2(gamma), dy), dy));
    const float2 hq = mul2(f2(NEG_HALF_LOG2E), q);
    e = make_float2(fast_ex2(hq.x), fast_ex2(hq.y));
    const float2 araw = mul2(f2(op), e);
    c0 = araw.x > GS_ALPHA_CLAMP;
    c1 = araw.y > GS_ALPHA_CLAMP;
    alpha = make_float2(c0 ? GS_ALPHA_CLAMP : araw.x, c1 ? GS_ALPHA_CLAMP : araw.y);
    om = fma2(f2(-op), e, f2(1.0f));
    om = make_float2(c0 ? 0.01f : om.x, c1 ? 0.01f : om.y);
}

// One pixel's blend state (R/rasterizer.py:256-291).  Opacity is accumulated as sum(w) (== 1 - T
// exactly in real arithmetic): 1 - T in fp32 cancels for nearly transparent pixels, and the
// depth loss divides by it.
struct FwdPixel {
    float fx, fy, T, c0, c1, c2, dsum, osum;
    int cnt;
    bool inside, done;
};

// Two pixels of one column (rows y and y + 8): the paired forward thread.
struct FwdPair {
    float fx;
    float2 fy, T, c0, c1, c2, dsum, osum;
    int cnt0, cnt1;
    bool in0, in1, done0, done1;
};

struct FwdStage {
    float4 a[RT];  // mx my a beta
    float4 b[RT];  // gamma opacity depth qcut
    float4 c[RT];  // r g b 1-opacity
};

__device__ __forceinline__ FwdPixel fwd_pixel_init(const gs_frame &f, int tile) {
    FwdPixel p;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int px = tx * GS_TILE + (threadIdx.x & 15), py = ty * GS_TILE + (threadIdx.x >> 4);
    p.inside = px < f.width && py < f.height;
    p.fx = (float)px;
    p.fy = (float)py;
    p.T = 1.0f;
    p.c0 = p.c1 = p.c2 = p.dsum = p.osum = 0.0f;
    p.cnt = 0;
    p.done = !p.inside;
    return p;
}

__device__ __forceinline__ int64_t fwd_pixel_index(const gs_frame &f, int tile) {
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    return (int64_t)(ty * GS_TILE + (threadIdx.x >> 4)) * f.width + tx * GS_TILE + (threadIdx.x & 15);
}

__device__ __forceinline__ void fwd_pixel_store(const gs_frame &f, int tile, const FwdPixel &p) {
    if (!p.inside) return;
    const int64_t q = fwd_pixel_index(f, tile);
    f.color[3 * q] = p.c0;
    f.color[3 * q + 1] = p.c1;
    f.color[3 * q + 2] = p.c2;
    f.depth[q] = p.dsum;
    f.opacity[q] = p.osum;
    f.trans[q] = p.T;
    f.n_contrib[q] = p.cnt;
}

#ifndef FWD_PAIRS
#define FWD_PAIRS 2
#endif
constexpr int NPF = FWD_PAIRS;       // pixel pairs per forward thread
constexpr int FT = RT / (2 * NPF);   // forward threads per tile
constexpr int RGF = FT / 16;         // pair h of a thread: rows row + RGF h and row + RGF h + 8

__device__ __forceinline__ FwdPair fwd_pair_init(const gs_frame &f, int tile, int h) {
    FwdPair p;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int px = tx * GS_TILE + (threadIdx.x & 15), py = ty * GS_TILE + (threadIdx.x >> 4) + RGF * h;
    p.in0 = px < f.width && py < f.height;
    p.in1 = px < f.width && py + GS_TILE / 2 < f.height;
    p.fx = (float)px;
    p.fy = make_float2((float)py, (float)(py + GS_TILE / 2));
    p.T = f2(1.0f);
    p.c0 = p.c1 = p.c2 = p.dsum = p.osum = f2(0.0f);
    p.cnt0 = p.cnt1 = 0;
    p.done0 = !p.in0;
    p.done1 = !p.in1;
    return p;
}

__device__ __forceinline__ void fwd_pair_store(const gs_frame &f, int tile, int hp, const FwdPair &p) {
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int64_t q0 = (int64_t)(ty * GS_TILE + (threadIdx.x >> 4) + RGF * hp) * f.width + tx * GS_TILE + (threadIdx.x & 15);
#pragma unroll
    for (int h = 0; h < 2; h++) {
        if (!(h ? p.in1 : p.in0)) continue;
        const int64_t q = q0 + (int64_t)h * (GS_TILE / 2) * f.width;
        f.color[3 * q] = h ? p.c0.y : p.c0.x;
        f.color[3 * q + 1] = h ? p.c1.y : p.c1.x;
        f.color[3 * q + 2] = h ? p.c2.y : p.c2.x;
        f.depth[q] = h ? p.dsum.y : p.dsum.x;
        f.opacity[q] = h ? p.osum.y : p.osum.x;
        f.trans[q] = h ? p.T.y : p.T.x;
        f.n_contrib[q] = h ? p.cnt1 : p.cnt0;
    }
}

// The paired form of blend_range (FT threads, NPF pixel pairs each): same staging, same
// per-pixel termination, alphas bit-identical to the scalar path.

// Blends the nb staged entries (list positions b, b + 1, ...) into the thread's two pixels.
// Branch-free per-pixel bookkeeping: a pixel that is still blending takes the entry (T and its
// count advance) and, with EARLY, stops after the entry that drives T below 1e-4 -- the
// reference's semantics (R/rasterizer.py:270-291) with selects instead of divergent branches.
template <bool EARLY>
__device__ __forceinline__ void blend_chunk2(FwdPair (&px)[NPF], const FwdStage &st, int b, int nb) {
    unsigned act = 0u;
    int n[NPF][2];
    float2 T[NPF];
#pragma unroll
    for (int h = 0; h < NPF; h++) {
        act |= (px[h].done0 ? 0u : 1u << (2 * h)) | (px[h].done1 ? 0u : 2u << (2 * h));
        n[h][0] = px[h].cnt0;
        n[h][1] = px[h].cnt1;
        T[h] = px[h].T;
    }
    for (int j = 0; j < nb && act; j++) {
        const float4 A = st.a[j], B = st.b[j], C = st.c[j];
        const float dx = px[0].fx - A.x;
        const int e1 = b + j + 1;
        unsigned keep = 0u;
#pragma unroll
        for (int h = 0; h < NPF; h++) {
            const float2 dy = add2(px[h].fy, f2(-A.y));
            float2 au, ev, alpha, om;
            bool c0, c1;
            alpha2(A, B, dx, dy, au, ev, alpha, om, c0, c1);
            const bool a0 = act & (1u << (2 * h)), a1 = act & (2u << (2 * h));
            float2 w = mul2(alpha, T[h]);
            w = make_float2(a0 ? w.x : 0.0f, a1 ? w.y : 0.0f);
            px[h].c0 = fma2(f2(C.x), w, px[h].c0);
            px[h].c1 = fma2(f2(C.y), w, px[h].c1);
            px[h].c2 = fma2(f2(C.z), w, px[h].c2);
            px[h].dsum = fma2(f2(B.z), w, px[h].dsum);
            px[h].osum = add2(px[h].osum, w);
            const float2 Tn = mul2(T[h], om);
            T[h] = make_float2(a0 ? Tn.x : T[h].x, a1 ? Tn.y : T[h].y);
            n[h][0] = a0 ? e1 : n[h][0];
            n[h][1] = a1 ? e1 : n[h][1];
            if (EARLY) keep |= (Tn.x < GS_EARLY_STOP_T ? 0u : 1u << (2 * h)) | (Tn.y < GS_EARLY_STOP_T ? 0u : 2u << (2 * h));
        }
        if (EARLY) act &= keep;
    }
#pragma unroll
    for (int h = 0; h < NPF; h++) {
        px[h].T = T[h];
        px[h].done0 = !(act & (1u << (2 * h)));
        px[h].done1 = !(act & (2u << (2 * h)));
        px[h].cnt0 = n[h][0];
        px[h].cnt1 = n[h][1];
    }
}

__device__ __forceinline__ bool pairs_done(const FwdPair (&px)[NPF]) {
    bool d = true;
#pragma unroll
    for (int h = 0; h < NPF; h++) d = d && px[h].done0 && px[h].done1;
    return d;
}

// entries staged per round: FS_FIRST in the first (most blends end within a few dozen), then FS
constexpr int FS = 128, FS_FIRST = 64;
static_assert(FS <= RT && FS_FIRST <= FS, "staging rounds");

template <typename Fetch>
__device__ __forceinline__ bool blend_range2(const gs_frame &f, FwdPair (&px)[NPF], FwdStage &st, int p0, int p1,
                                             int early_stop, Fetch fetch) {
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    for (int b = p0, step = FS_FIRST; b < p1; b += step, step = FS) {
        if (__syncthreads_count(pairs_done(px)) == FT) return true;
        for (int i = threadIdx.x; i < step; i += FT) {
            const int e = b + i;
            if (e < p1) {
                const int64_t g = fetch(e);
                st.a[i] = __ldg(sp + GS_SPLAT / 4 * g);
                st.b[i] = __ldg(sp + GS_SPLAT / 4 * g + 1);
                st.c[i] = __ldg(sp + GS_SPLAT / 4 * g + 2);
            }
        }
        __syncthreads();
        const int nb = min(step, p1 - b);
        if (early_stop) blend_chunk2<true>(px, st, b, nb);
        else blend_chunk2<false>(px, st, b, nb);
    }
    return __syncthreads_count(pairs_done(px)) == FT;
}

// Blends list positions [p0, p1) of the tile front to back; fetch(p) -> Gaussian id.  The
// tile's entries are staged RT at a time in shared memory; the CTA stops once every pixel is
// done.  Returns whether every pixel is done.
template <typename Fetch>
__device__ __forceinline__ bool blend_range(const gs_frame &f, FwdPixel &px, FwdStage &st, int p0, int p1,
                                            int early_stop, Fetch fetch) {
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    // the first round stages 64 entries (most blends end within a few dozen), then RT at a time
    for (int b = p0, step = RT / 4; b < p1; b += step, step = RT) {
        if (__syncthreads_count(px.done) == RT) return true;
        const int e = b + threadIdx.x;
        if ((int)threadIdx.x < step && e < p1) {
            const int64_t g = fetch(e);
            st.a[threadIdx.x] = __ldg(sp + GS_SPLAT / 4 * g);
            st.b[threadIdx.x] = __ldg(sp + GS_SPLAT / 4 * g + 1);
            st.c[threadIdx.x] = __ldg(sp + GS_SPLAT / 4 * g + 2);
        }
        __syncthreads();
        if (!px.done) {
            const int nb = min(step, p1 - b);
            for (int j = 0; j < nb; j++) {
                const float4 A = st.a[j], B = st.b[j], C = st.c[j];
                const float dx = px.fx - A.x, dy = px.fy - A.y;
                float araw, alpha, oma, au;
                alpha_oma(B.y, C.w, quad(A.z, A.w, B.x, dx, dy, au), araw, alpha, oma);
                const float w = alpha * px.T;
                px.c0 += C.x * w;
                px.c1 += C.y * w;
                px.c2 += C.z * w;
                px.dsum += B.z * w;
                px.osum += w;
                px.T *= oma;
                if (early_stop && px.T < GS_EARLY_STOP_T) {
                    px.done = true;
                    px.cnt = b + j + 1;
                    break;
                }
            }
            if (!px.done) px.cnt = b + nb;
        }
    }
    return __syncthreads_count(px.done) == RT;
}

#ifndef FWD_MINB
#define FWD_MINB 16  // 64 registers: 16 CTAs (32 warps) per SM
#endif
__global__ void __launch_bounds__(FT, FWD_MINB) render_fwd_kernel(gs_frame f, int flags) {
    pdl_wait();
    const int early_stop = flags & GS_FWD_EARLY_STOP;
    __shared__ FwdStage st;
    __shared__ uint32_t s_words[GS_HUGE_CAP / 32];
    __shared__ int32_t s_wpre[GS_HUGE_CAP / 32];
    __shared__ int32_t s_tmp[FT / 32 > 0 ? FT / 32 : 1];
    const int tile = blockIdx.x;
    FwdPair px[NPF];
#pragma unroll
    for (int h = 0; h < NPF; h++) px[h] = fwd_pair_init(f, tile, h);
    if (blockIdx.x == 0 && threadIdx.x == 0) f.counters[GS_CNT_FWD_CLEARED] = (flags & GS_FWD_CLEAR_G2D) ? 1 : 0;
    auto store = [&]() {
        if (flags & GS_FWD_CLEAR_G2D) {
            // the engines' screen-space gradient rows (touched slots 0..nt-1) start each backward
            // at zero: cleared here as whole lines once the tile is blended, so the stores overlap
            // the other CTAs' blending, and the lines stay in L2 for the backward's atomics (the
            // chain rule only reads them)
            const int64_t words = (int64_t)(GS_G2D / 2) * f.counters[GS_CNT_TOUCHED];
            longlong2 *g2 = reinterpret_cast<longlong2 *>(f.g2d);
            for (int64_t i = (int64_t)blockIdx.x * FT + threadIdx.x; i < words; i += (int64_t)gridDim.x * FT)
                g2[i] = make_longlong2(0, 0);
        }
#pragma unroll
        for (int h = 0; h < NPF; h++) fwd_pair_store(f, tile, h, px[h]);
    };
    if (f.counters[GS_CNT_OVERFLOW]) {  // binning over capacity (tile ranges emptied): background
        store();
        return;
    }
    if (f.counters[GS_CNT_LAZY]) {
        // lazy lists: the leading screen-covering Gaussians (every one whose key is below the
        // tile's smallest bucketed key precedes the whole bucket); tiles whose blend outlives them
        // are finished by tile_finish_kernel from the stored state
        __shared__ int s_lead;
        const int na = tile_huge_setup(f, tile, s_words, s_wpre, s_tmp);
        const int nw = (min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) + 31) >> 5;
        if (threadIdx.x == 0) {
            const uint64_t mk = f.tile_minkey[tile];
            s_lead = mk == ~0ull ? na : tile_huge_rank(huge_before_key(f, mk), s_words, s_wpre, nw, na);
        }
        __syncthreads();
        const int lead = s_lead;
        const int32_t *hid = f.huge + HIDS;
        const bool all = blend_range2(f, px, st, 0, lead, early_stop,
                                      [&](int p) { return hid[tile_huge_select(p, s_words, s_wpre, nw)]; });
        const int total = f.tile_offsets[tile + 1] - f.tile_offsets[tile];
        if (!all && total > lead && threadIdx.x == 0) {
            ts_flag(f)[tile] = TL_LIST;
            ts_resume(f)[tile] = lead;
            f.counters[GS_CNT_ANYFLAG] = 1;
            ts_flagged(f)[atomicAdd(&f.counters[GS_CNT_FLAGGED], 1)] = tile;
        }
    } else {
        const int start = f.tile_offsets[tile], stop = f.tile_offsets[tile + 1];
        const int32_t *list = f.entry_splat + start;
        blend_range2(f, px, st, 0, stop - start, early_stop, [&](int p) { return list[p]; });
    }
    store();
}

// Lazy lists, continuation 1: the bucket keys of the tiles that need them (ts_flag != 0)
__global__ void __launch_bounds__(256) lazy_fill_kernel(gs_frame f) {
    pdl_wait();
    if (!f.counters[GS_CNT_LAZY] || !f.counters[GS_CNT_ANYFLAG] || f.counters[GS_CNT_OVERFLOW]) return;
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    int32_t *cur = ts_cursor(f);
    const int32_t *flag = ts_flag(f);
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += (int64_t)gridDim.x * blockDim.x) {
        const int g = f.touched_list[k];
        if (bin_rec(f)[g].kept <= 0) continue;
        const uint64_t key = depth_key(f, g);
        const int4 r = bin_rec(f)[g].rect;
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        const int64_t base = (int64_t)bin_rec(f)[g].bits;
        const SplatCull s = splat_cull(f.splat2d, g);
        for (int c = 0; c < ncand; c++) {
            const int tx = r.x + c % nx, ty = r.z + c / nx, t = ty * f.tiles_x + tx;
            bool keep;
            if (ncand <= GS_SMALL_CAND) {
                keep = (bin_rec(f)[g].bits >> c) & 1ull;
            } else if (base >= 0) {
                keep = (f.big_bits[base + (c >> 5)] >> (c & 31)) & 1u;
            } else {
                const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
                const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
                keep = tile_keep(s.mx, s.my, s.ca, s.cb, s.cc, s.qcut, x0, x1, y0, y1);
            }
            if (keep && flag[t]) f.keys_b[atomicAdd(&cur[t], 1)] = key;
        }
    }
}

// Lazy lists, continuation 2: CTA per flagged tile.  Sorts the bucket, writes the tile's merged
// list to entry_splat (the backward reads it there) and resumes the blend where the forward
// stopped (state from the stored images).
constexpr int TF_THREADS = RT;

struct FinishSmem {
    uint64_t key[SM_CAP];
    int32_t a[GS_HUGE_CAP];
    uint32_t words[GS_HUGE_CAP / 32];
    int32_t wpre_a[GS_HUGE_CAP / 32];
    uint32_t isb[(GS_HUGE_CAP + SM_CAP) / 32];
    int32_t wpre[(GS_HUGE_CAP + SM_CAP) / 32];
    int32_t tmp[TF_THREADS / 32];
    FwdStage st;
};

__device__ __forceinline__ void tile_finish_one(const gs_frame &f, FinishSmem &sm, int tile, int early_stop);

// persistent over the tiles the forward flagged (a compact list; most tiles need no
// continuation, and a grid over all tiles would mostly launch CTAs that exit at once)
__global__ void __launch_bounds__(TF_THREADS) tile_finish_kernel(gs_frame f, int early_stop) {
    pdl_wait();
    if (!f.counters[GS_CNT_LAZY] || !f.counters[GS_CNT_ANYFLAG] || f.counters[GS_CNT_OVERFLOW]) return;
    extern __shared__ uint64_t fin_raw[];
    FinishSmem &sm = *reinterpret_cast<FinishSmem *>(fin_raw);
    const int nflag = f.counters[GS_CNT_FLAGGED];
    for (int it = blockIdx.x; it < nflag; it += gridDim.x) {
        if (it != (int)blockIdx.x) __syncthreads();  // the previous tile's shared state is consumed
        tile_finish_one(f, sm, ts_flagged(f)[it], early_stop);
    }
}

__device__ __forceinline__ void tile_finish_one(const gs_frame &f, FinishSmem &sm, int tile, int early_stop) {
    const int sb = ts_boff(f)[tile], nb = ts_boff(f)[tile + 1] - sb;
    const uint64_t *B = sort_bucket<TF_THREADS>(sm.key, f.keys_b + sb, f.keys_a + sb, nb, false);
    const int na = tile_huge_setup(f, tile, sm.words, sm.wpre_a, sm.tmp);
    const int nw = (min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) + 31) >> 5;
    tile_huge_expand(sm.words, sm.wpre_a, nw, sm.a);
    int32_t *list = f.entry_splat + f.tile_offsets[tile];
    merge_tile_list<TF_THREADS>(f, list, sm.a, na, B, nb, sm.isb, sm.wpre, sm.tmp, GS_HUGE_CAP + SM_CAP);
    __syncthreads();
    FwdPixel px = fwd_pixel_init(f, tile);
    if (px.inside) {
        const int64_t q = fwd_pixel_index(f, tile);
        px.c0 = f.color[3 * q];
        px.c1 = f.color[3 * q + 1];
        px.c2 = f.color[3 * q + 2];
        px.dsum = f.depth[q];
        px.osum = f.opacity[q];
        px.T = f.trans[q];
        px.cnt = f.n_contrib[q];
        px.done = early_stop && px.T < GS_EARLY_STOP_T;
    }
    blend_range(f, px, sm.st, ts_resume(f)[tile], na + nb, early_stop, [&](int p) { return list[p]; });
    fwd_pixel_store(f, tile, px);
}

// Per-entry warp reductions (transposed butterflies: each stage halves the fields a lane carries).
// The six geometric fields (mean2d 2, conic 3, opacity) are summed in FP64: for Gaussians just
// past the near plane the chain rule cancels their mean and conic paths ~1e4-fold, and rounding
// the per-pixel partial sums to fp32 alone moved position gradients by ~2e-3 of the reference
// (tools/bwd_emulator.py); the colour / depth fields stay fp32.
//
// reduce_geo: on return lane L with (L & 3) == 0 holds the warp sum of field geo_field(L) >= 0.
__device__ __forceinline__ double reduce_geo(const float v[6]) {
    const unsigned lane = threadIdx.x & 31u;
    const bool h = lane & 16u, b3 = lane & 8u, b2 = lane & 4u;
    double u[3];
#pragma unroll
    for (int k = 0; k < 3; k++) {  // xor 16: fields {0,1,2} | {3,4,5}
        const double send = h ? (double)v[k] : (double)v[k + 3];
        const double keep = h ? (double)v[k + 3] : (double)v[k];
        u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    // xor 8: b3 = 0 keeps u0, u1; b3 = 1 keeps u2
    const double r1 = __shfl_xor_sync(0xffffffffu, b3 ? u[0] : u[2], 8);
    const double r2 = __shfl_xor_sync(0xffffffffu, u[1], 8);
    const double w0 = b3 ? u[2] + r1 : u[0] + r1;
    const double w1 = u[1] + r2;  // meaningful for b3 = 0 only
    // xor 4: b3 = 0 splits (w0 | w1); b3 = 1 lanes both hold field 2 of their half
    const double send = b3 ? w0 : (b2 ? w0 : w1);
    const double keep = b3 ? w0 : (b2 ? w1 : w0);
    double z = keep + __shfl_xor_sync(0xffffffffu, send, 4);
    z += __shfl_xor_sync(0xffffffffu, z, 2);
    z += __shfl_xor_sync(0xffffffffu, z, 1);
    return z;
}

__device__ __forceinline__ int geo_field(unsigned lane) {
    if (lane & 3u) return -1;
    const int base = (lane & 16u) ? 3 : 0;
    if (!(lane & 8u)) return base + ((lane & 4u) ? 1 : 0);
    return (lane & 4u) ? -1 : base + 2;
}

// reduce_col: the four fp32 fields (colour 3, depth); lane L with (L & 7) == 0 holds field
// col_field(L)
__device__ __forceinline__ float reduce_col(const float v[4]) {
    const unsigned lane = threadIdx.x & 31u;
    const bool h = lane & 16u, b3 = lane & 8u;
    float u[2];
#pragma unroll
    for (int k = 0; k < 2; k++) {  // xor 16: {0,1} | {2,3}
        const float send = h ? v[k] : v[k + 2];
        const float keep = h ? v[k + 2] : v[k];
        u[k] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
    }
    float z = (b3 ? u[1] : u[0]) + __shfl_xor_sync(0xffffffffu, b3 ? u[0] : u[1], 8);
    z += __shfl_xor_sync(0xffffffffu, z, 4);
    z += __shfl_xor_sync(0xffffffffu, z, 2);
    z += __shfl_xor_sync(0xffffffffu, z, 1);
    return z;
}

__device__ __forceinline__ int col_field(unsigned lane) {
    if (lane & 7u) return -1;
    return ((lane & 16u) ? 2 : 0) + ((lane & 8u) ? 1 : 0);
}


// The two pixels' replay state (R/rasterizer.py:365-410, run back to front from the final T).
struct BwdPair {
    float fx;                       // column (shared)
    float2 fy;                      // rows
    float2 T, gc0, gc1, gc2, gd, go, S0, S1, S2, Sd, So;
    int cnt0, cnt1;
};

// One entry's contribution of both pixels to the 10 screen-space gradient fields (v[k] holds
// the two pixels' terms in .x / .y): undoes the entry's 1 - alpha on T, accumulates, advances
// the suffix sums.  alpha is computed exactly as the forward computes it (same operation order:
// quad(), fast_ex2, fmaf(-op, e, 1)), so the replay divides out precisely what the blend
// multiplied in.  The quadratic and the mean gradient use the factored conic of the splat
// record: a dx + b dy = a u and b dx + c dy = beta a u + gamma dy (u = dx + beta dy).
__device__ __forceinline__ void bwd_step2(BwdPair &p, bool act0, bool act1, const float4 &A, const float4 &B,
                                          const float4 &C, float2 v[10]) {
    const float dx = p.fx - A.x;
    const float2 dy = add2(p.fy, f2(-A.y));
    const float beta = A.w, gamma = B.x, dep = B.z;
    float2 au, e, alpha, om;
    bool c0, c1;
    alpha2(A, B, dx, dy, au, e, alpha, om, c0, c1);
    const float2 rom = make_float2(fast_rcp(om.x), fast_rcp(om.y));
    const float2 Tb = mul2(p.T, rom);
    float2 w = mul2(alpha, Tb);
    w = make_float2(act0 ? w.x : 0.0f, act1 ? w.y : 0.0f);  // a finished pixel takes no part
    v[6] = fma2(w, p.gc0, v[6]);
    v[7] = fma2(w, p.gc1, v[7]);
    v[8] = fma2(w, p.gc2, v[8]);
    v[9] = fma2(w, p.gd, v[9]);
    float2 own = fma2(f2(C.x), p.gc0, p.go);
    own = fma2(f2(C.y), p.gc1, own);
    own = fma2(f2(C.z), p.gc2, own);
    own = fma2(f2(dep), p.gd, own);
    float2 suf = mul2(p.So, p.go);
    suf = fma2(p.S0, p.gc0, suf);
    suf = fma2(p.S1, p.gc1, suf);
    suf = fma2(p.S2, p.gc2, suf);
    suf = fma2(p.Sd, p.gd, suf);
    const float2 sr = mul2(suf, rom);
    const float2 dl = fma2(Tb, own, make_float2(-sr.x, -sr.y));
    // no alpha-chain gradient on the 0.99 clamp (R/rasterizer.py:399-404), none from a finished pixel
    const bool g0 = act0 && !c0, g1 = act1 && !c1;
    // ga = dl alpha; the reference's gq = -dl alpha / 2 (R/rasterizer.py:405-410) is ga / -2, and
    // gq (-2 a u) = ga a u: the power-of-two scalings are exact, so every sum is bit-identical
    const float2 dlm = make_float2(g0 ? dl.x : 0.0f, g1 ? dl.y : 0.0f);
    const float2 ga = mul2(dlm, alpha);
    const float2 gq = mul2(ga, f2(-0.5f));
    const float2 de = mul2(dlm, e);  // d alpha / d opacity = e
    v[5] = add2(v[5], de);
    v[2] = fma2(gq, f2(dx * dx), v[2]);
    v[3] = fma2(gq, mul2(f2(2.0f * dx), dy), v[3]);
    v[4] = fma2(mul2(gq, dy), dy, v[4]);
    v[0] = fma2(ga, au, v[0]);
    v[1] = fma2(ga, fma2(f2(beta), au, mul2(f2(gamma), dy)), v[1]);
    p.S0 = fma2(f2(C.x), w, p.S0);
    p.S1 = fma2(f2(C.y), w, p.S1);
    p.S2 = fma2(f2(C.z), w, p.S2);
    p.Sd = fma2(f2(dep), w, p.Sd);
    p.So = add2(p.So, w);
    p.T = make_float2(act0 ? Tb.x : p.T.x, act1 ? Tb.y : p.T.y);
}

// 64 threads per 16x16 tile, four pixels per thread (column x, rows r, r + 4, r + 8, r + 12 as
// two row pairs): the four pixels' contributions are summed in registers before the warp
// reduction, so each staged entry costs the tile two warp reductions instead of eight (one per
// 32 pixels).  Deterministic: per staged entry every warp stores its butterfly sums in its own
// shared-memory slot, the warp sums are added in warp order, and the tile partial goes to the
// Gaussian's row through fixed-point integer atomics (fx_atomic_add) -- no floating-point sum
// depends on scheduling order.
#ifndef BWD_PAIRS
#define BWD_PAIRS 2
#endif
constexpr int NP = BWD_PAIRS;       // pixel pairs per backward thread
constexpr int BT = RT / (2 * NP);   // backward threads per tile
constexpr int RG = BT / 16;         // row groups: pair h of a thread is rows row + RG h, + RG h + 8
constexpr int BW = BT / 32;         // warps per backward CTA
constexpr int BST = BT;             // entries staged per round (one per thread)

#ifndef BWD_MINB
#define BWD_MINB 1
#endif
__global__ void __launch_bounds__(BT, BWD_MINB) render_bwd_kernel(gs_frame f, int clear_depth_grads) {
    pdl_wait();
    __shared__ float4 s_a[BST];
    __shared__ float4 s_b[BST];
    __shared__ float4 s_c[BST];
    __shared__ int s_g[BST];
    __shared__ double s_geo[BW][BST][6];
    __shared__ float s_col[BW][BST][4];
    __shared__ int s_max;
    const int tile = blockIdx.x;
    const int tx = tile % f.tiles_x, ty = tile / f.tiles_x;
    const int start = f.tile_offsets[tile], stop = f.tile_offsets[tile + 1];
    const int col = threadIdx.x & 15, row = threadIdx.x >> 4;  // rows row + RG k, k < 2 NP
    if (clear_depth_grads && stop == start) {  // (GS_BWD_CLEAR_DEPTH_GRADS) an empty tile's pixels
#pragma unroll
        for (int k = 0; k < 2 * NP; k++) {
            const int x = tx * GS_TILE + col, y = ty * GS_TILE + row + RG * k;
            if (x < f.width && y < f.height) {
                const int64_t q = (int64_t)y * f.width + x;
                if (f.g_depth[q] != 0.0f) f.g_depth[q] = 0.0f;
                if (f.g_opac[q] != 0.0f) f.g_opac[q] = 0.0f;
            }
        }
    }
    if (stop == start) return;
    const unsigned lane = threadIdx.x & 31u;
    const int warp = threadIdx.x >> 5;
    const int fgeo = geo_field(lane), fcol = col_field(lane);
    // entry source: materialised list, or (lazy lists) the screen-covering Gaussians then the
    // sorted bucket
    __shared__ uint32_t s_words[GS_HUGE_CAP / 32];
    __shared__ int32_t s_wpre[GS_HUGE_CAP / 32];
    __shared__ int32_t s_tmp[BT / 32];
    const bool lazy = f.counters[GS_CNT_LAZY] && ts_flag(f)[tile] == TL_LAZY_A;
    int nw = 0;
    if (lazy) {
        tile_huge_setup(f, tile, s_words, s_wpre, s_tmp);
        nw = (min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) + 31) >> 5;
    }
    const int32_t *hid = f.huge + HIDS;
    auto fetch = [&](int p) -> int {  // list position -> Gaussian id
        // lazy, unflagged: the blend ended within the leading screen-covering Gaussians
        return lazy ? hid[tile_huge_select(p, s_words, s_wpre, nw)] : f.entry_splat[start + p];
    };
    BwdPair px[NP];  // pair h: rows row + RG h and row + RG h + 8
    if (threadIdx.x == 0) s_max = 0;
    __syncthreads();
    {
        const int x = tx * GS_TILE + col;
        int mx = 0;
#pragma unroll
        for (int h = 0; h < NP; h++) {
            const int y0 = ty * GS_TILE + row + RG * h;
            px[h].fx = (float)x;
            px[h].fy = make_float2((float)y0, (float)(y0 + GS_TILE / 2));
            float T[2] = {1.0f, 1.0f}, gc[2][3] = {}, gd[2] = {}, go[2] = {};
            int cnt[2] = {0, 0};
#pragma unroll
            for (int k = 0; k < 2; k++) {
                const int y = y0 + (GS_TILE / 2) * k;
                if (x < f.width && y < f.height) {
                    const int64_t q = (int64_t)y * f.width + x;
                    T[k] = f.trans[q];
                    cnt[k] = f.n_contrib[q];
                    gc[k][0] = f.g_color[3 * q];
                    gc[k][1] = f.g_color[3 * q + 1];
                    gc[k][2] = f.g_color[3 * q + 2];
                    gd[k] = f.g_depth[q];
                    go[k] = f.g_opac[q];
                    if (clear_depth_grads) {  // nonzero only at the view's LiDAR pixels
                        if (gd[k] != 0.0f) f.g_depth[q] = 0.0f;
                        if (go[k] != 0.0f) f.g_opac[q] = 0.0f;
                    }
                }
            }
            px[h].T = make_float2(T[0], T[1]);
            px[h].gc0 = make_float2(gc[0][0], gc[1][0]);
            px[h].gc1 = make_float2(gc[0][1], gc[1][1]);
            px[h].gc2 = make_float2(gc[0][2], gc[1][2]);
            px[h].gd = make_float2(gd[0], gd[1]);
            px[h].go = make_float2(go[0], go[1]);
            px[h].S0 = px[h].S1 = px[h].S2 = px[h].Sd = px[h].So = f2(0.0f);
            px[h].cnt0 = cnt[0];
            px[h].cnt1 = cnt[1];
            mx = max(mx, max(cnt[0], cnt[1]));
        }
        atomicMax(&s_max, mx);
    }
    __syncthreads();
    const int max_cnt = s_max;
    const float4 *sp = reinterpret_cast<const float4 *>(f.splat2d);
    for (int b_end = start + max_cnt; b_end > start; b_end -= BST) {
        const int b0 = max(start, b_end - BST);
        const int nb = b_end - b0;
        __syncthreads();
        if ((int)threadIdx.x < nb) {  // (nb <= BST == BT)
            const int i = threadIdx.x;
            const int64_t g = fetch(b0 - start + i);
            s_g[i] = splat_slot(f.splat2d, g);  // its g2d row
            s_a[i] = __ldg(sp + GS_SPLAT / 4 * g);
            s_b[i] = __ldg(sp + GS_SPLAT / 4 * g + 1);
            s_c[i] = __ldg(sp + GS_SPLAT / 4 * g + 2);
        }
        __syncthreads();
        for (int j = nb - 1; j >= 0; j--) {
            const int le = b0 + j - start;
            bool act[NP][2], any = false;
#pragma unroll
            for (int h = 0; h < NP; h++) {
                act[h][0] = le < px[h].cnt0;
                act[h][1] = le < px[h].cnt1;
                any = any || act[h][0] || act[h][1];
            }
            double sg = 0.0;
            float sc = 0.0f;
            if (__any_sync(0xffffffffu, any)) {
                const float4 A = s_a[j], B = s_b[j], C = s_c[j];
                float2 v[10];
#pragma unroll
                for (int k = 0; k < 10; k++) v[k] = f2(0.0f);
#pragma unroll
                for (int h = 0; h < NP; h++) bwd_step2(px[h], act[h][0], act[h][1], A, B, C, v);
                float vg[6], vc[4];
#pragma unroll
                for (int k = 0; k < 6; k++) vg[k] = v[k].x + v[k].y;
#pragma unroll
                for (int k = 0; k < 4; k++) vc[k] = v[6 + k].x + v[6 + k].y;
                sg = reduce_geo(vg);
                sc = reduce_col(vc);
            }
            if (fgeo >= 0) s_geo[warp][j][fgeo] = sg;
            if (fcol >= 0) s_col[warp][j][fcol] = sc;
        }
        __syncthreads();
        // the tile's partial of every staged entry: warp sums in warp order, then fixed point
        for (int idx = threadIdx.x; idx < nb * GS_G2D_FIELDS; idx += BT) {
            const int i = idx / GS_G2D_FIELDS, k = idx - i * GS_G2D_FIELDS;
            double v;
            if (k < 6) {
                v = s_geo[0][i][k];
#pragma unroll
                for (int w = 1; w < BW; w++) v += s_geo[w][i][k];
            } else {
                float c = s_col[0][i][k - 6];
#pragma unroll
                for (int w = 1; w < BW; w++) c += s_col[w][i][k - 6];
                v = c;
            }
            if (v != 0.0) fx_atomic_add(reinterpret_cast<long long *>(f.g2d) + (int64_t)s_g[i] * GS_G2D + 2 * k, v);
        }
    }
}

// zero the g2d rows of the touched slots 0..nt-1 (GS_G2D int64 = GS_G2D / 2 16-B words per row)
__global__ void zero_g2d_kernel(gs_frame f) {
    pdl_wait();
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    constexpr int W = GS_G2D / 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < W * nt; i += (int64_t)gridDim.x * blockDim.x) {
        reinterpret_cast<longlong2 *>(f.g2d)[i] = make_longlong2(0, 0);  // rows by touched slot
    }
}

}  // namespace gs

using namespace gs;

extern "C" int gs_render_fwd(const gs_frame *f, int32_t early_stop, void *stream) {
    return gs_render_fwd_ex(f, early_stop ? GS_FWD_EARLY_STOP : 0, stream);
}

extern "C" int gs_render_fwd_ex(const gs_frame *f, int32_t flags, void *stream) {
    if (flags & ~(GS_FWD_EARLY_STOP | GS_FWD_CLEAR_G2D)) {
        set_error("gs_render_fwd_ex: unknown flags");
        return GS_ERR_ARG;
    }
    const int early_stop = flags & GS_FWD_EARLY_STOP;
    const int T = f->tiles_x * f->tiles_y;
    if (T == 0) return GS_OK;
    launch_pdl(render_fwd_kernel, T, FT, 0, (cudaStream_t)stream, *f, (int)flags);
    int rc = check_launch("render_fwd_kernel");
    if (rc) return rc;
    // lazy lists: bucket fill + sorted continuation of the tiles that need them (no-ops otherwise)
    launch_pdl(lazy_fill_kernel, 4 * 148, 256, 0, (cudaStream_t)stream, *f);
    if ((rc = check_launch("lazy_fill_kernel"))) return rc;
    launch_pdl(tile_finish_kernel, (unsigned)std::min(T, 3 * 148), TF_THREADS, sizeof(FinishSmem), (cudaStream_t)stream, *f,
               early_stop);
    return check_launch("tile_finish_kernel");
}

extern "C" int gs_render_bwd(const gs_frame *f, void *stream) { return gs_render_bwd_ex(f, 0, stream); }

extern "C" int gs_render_bwd_ex(const gs_frame *f, int32_t flags, void *stream) {
    if (flags & ~(GS_BWD_ROWS_ZERO | GS_BWD_CLEAR_DEPTH_GRADS)) {
        set_error("gs_render_bwd_ex: unknown flags");
        return GS_ERR_ARG;
    }
    const int T = f->tiles_x * f->tiles_y;
    if (T == 0) return GS_OK;
    if (f->n > 0 && !(flags & GS_BWD_ROWS_ZERO)) {  // each backward starts from zero gradients (backward_2d is a pure function)
        // grid-stride over a small fixed grid: in the engine (lazy lists) every CTA exits at once
        launch_pdl(zero_g2d_kernel, 2 * 148, 256, 0, (cudaStream_t)stream, *f);
        int rc = check_launch("zero_g2d_kernel");
        if (rc) return rc;
    }
    launch_pdl(render_bwd_kernel, T, BT, 0, (cudaStream_t)stream, *f, (flags & GS_BWD_CLEAR_DEPTH_GRADS) ? 1 : 0);
    return check_launch("render_bwd_kernel");
}

namespace gs {
void init_render_attrs() {
    cudaFuncSetAttribute(tile_finish_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sizeof(FinishSmem));
}
}  // namespace gs
