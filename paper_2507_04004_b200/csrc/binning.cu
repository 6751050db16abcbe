// binning.cu -- tile binning: depth sort, exact per-tile cull, (tile|depth) entries, ranges.
//
// Replaces R/rasterizer.py:169-219 (cull_tiles) and the `touched` bookkeeping of
// _reduce_entries (:424).  The reference enumerates (splat, tile) pairs in splat order, culls
// them exactly and lexsorts by (tile, depth, splat).  Here:
//   1. the active Gaussians (>= 1 candidate tile) are sorted by fp32 depth with a stable
//      onesweep LSD radix sort over 64-bit words (depth_bits << 32 | id): stability gives the
//      id tie-break;
//   2. kept pairs are counted (exact cull, strict fp32) and emitted in depth order as 64-bit
//      words (tile << 32 | id) at scanned offsets;
//   3. a second stable onesweep sort on the tile bits only yields lexsort((id, depth, tile));
//   4. tile ranges come from adjacent-key compares.
// Every kernel reads its element count from device memory, so the sequence is graph-capturable.
#include <cstdio>

#include "common.cuh"

namespace gs {

constexpr int RS_THREADS = 256;
constexpr int RS_ITEMS = 16;
constexpr int RS_TILE = RS_THREADS * RS_ITEMS;  // 4096 keys per onesweep tile
constexpr uint32_t FLAG_AGG = 1u << 30, FLAG_INC = 2u << 30, VAL_MASK = (1u << 30) - 1u;

__device__ __forceinline__ uint32_t ld_volatile(const uint32_t *p) { return *(volatile const uint32_t *)p; }
__device__ __forceinline__ void st_atomic(uint32_t *p, uint32_t v) { atomicExch(p, v); }

__device__ __forceinline__ unsigned lanemask_lt() {
    unsigned m;
    asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
    return m;
}

// ---------------------------------------------------------------------------
// digit histograms of all requested passes in one read (filter: drop inactive words)
template <typename K>
__device__ __forceinline__ bool inactive_key(K k, int filter) {
    return filter && (uint64_t)k >> 32 == 0xffffffffull;
}

template <typename K>
__global__ void __launch_bounds__(256) radix_hist_kernel(const K *__restrict__ keys, int64_t n_host,
                                                         const int32_t *__restrict__ n_dev, int shift0, int npasses,
                                                         uint32_t *__restrict__ hist, int filter,
                                                         int32_t *__restrict__ active_out) {
    // per-warp privatised sub-histograms cut shared-atomic contention on skewed digits
    __shared__ uint32_t sh[4][4][256];
    for (int k = threadIdx.x; k < 16 * 256; k += blockDim.x) (&sh[0][0][0])[k] = 0;
    __syncthreads();
    const int sub = (threadIdx.x >> 5) & 3;
    const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    uint32_t local_active = 0;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const K k = keys[i];
        if (inactive_key(k, filter)) continue;
        local_active++;
        for (int p = 0; p < npasses; p++) atomicAdd(&sh[sub][p][(uint32_t)(k >> (shift0 + 8 * p)) & 255u], 1u);
    }
    __syncthreads();
    for (int k = threadIdx.x; k < 4 * 256; k += blockDim.x)
        (&sh[0][0][0])[k] += (&sh[1][0][0])[k] + (&sh[2][0][0])[k] + (&sh[3][0][0])[k];
    __syncthreads();
    for (int k = threadIdx.x; k < npasses * 256; k += blockDim.x) {
        uint32_t v = (&sh[0][0][0])[k];
        if (v) atomicAdd(&hist[k], v);
    }
    if (filter && active_out) {
        for (int o = 16; o > 0; o >>= 1) local_active += __shfl_xor_sync(0xffffffffu, local_active, o);
        if ((threadIdx.x & 31) == 0 && local_active) atomicAdd(active_out, (int32_t)local_active);
    }
}

// exclusive scan of each pass's 256 bins (one block per pass)
__global__ void radix_bins_kernel(uint32_t *hist) {
    __shared__ uint32_t s[256];
    uint32_t *h = hist + blockIdx.x * 256;
    uint32_t v = h[threadIdx.x];
    s[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < 256; o <<= 1) {
        uint32_t t = threadIdx.x >= o ? s[threadIdx.x - o] : 0u;
        __syncthreads();
        s[threadIdx.x] += t;
        __syncthreads();
    }
    h[threadIdx.x] = s[threadIdx.x] - v;
}

// ---------------------------------------------------------------------------
// one onesweep pass: stable counting-sort of a 4096-key tile by one 8-bit digit, decoupled
// look-back across tiles for the per-digit global offsets, scatter through shared memory.
template <typename K>
__global__ void __launch_bounds__(RS_THREADS, sizeof(K) == 4 ? 4 : 3) onesweep_kernel(const K *__restrict__ in, K *__restrict__ out,
                                                              int64_t n_host, const int32_t *__restrict__ n_dev,
                                                              int shift, const uint32_t *__restrict__ bins,
                                                              uint32_t *status, int32_t *ticket, int filter) {
    constexpr int WARPS = RS_THREADS / 32;
    // digit 256 is a dummy bucket for out-of-range and filtered items (never scattered)
    __shared__ uint32_t s_warp[WARPS][257];
    __shared__ uint32_t s_start[256];
    __shared__ uint32_t s_base[256];
    __shared__ uint32_t s_scan[WARPS];
    __shared__ K s_keys[RS_TILE];
    __shared__ int s_tile;
    __shared__ uint32_t s_total;

    const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    for (int k = threadIdx.x; k < WARPS * 257; k += RS_THREADS) (&s_warp[0][0])[k] = 0u;
    __syncthreads();
    const int tile = s_tile;
    const int64_t tbase = (int64_t)tile * RS_TILE;
    if (tbase >= n) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t wbase = tbase + (int64_t)warp * 32 * RS_ITEMS;
    const unsigned ltmask = lanemask_lt();

    K key[RS_ITEMS];
    uint32_t dig[RS_ITEMS];
    uint32_t rank[RS_ITEMS];
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const int64_t idx = wbase + i * 32 + lane;
        key[i] = idx < n ? in[idx] : (K)0;
        dig[i] = (idx < n && !inactive_key(key[i], filter)) ? ((uint32_t)(key[i] >> shift) & 255u) : 256u;
    }
    // warp-level stable ranking (items in order, lanes in order): the highest lane of each
    // peer group bumps the warp's digit counter and broadcasts the old value
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const unsigned peers = __match_any_sync(0xffffffffu, dig[i]);
        const int leader = 31 - __clz(peers);
        uint32_t before = 0;
        if (lane == leader) before = atomicAdd(&s_warp[warp][dig[i]], (uint32_t)__popc(peers));
        before = __shfl_sync(0xffffffffu, before, leader);
        rank[i] = before + __popc(peers & ltmask);
    }
    __syncthreads();
    // per-digit warp offsets and tile totals; thread t owns digit t
    const int t = threadIdx.x;
    uint32_t run = 0;
#pragma unroll
    for (int w = 0; w < WARPS; w++) {
        uint32_t c = s_warp[w][t];
        s_warp[w][t] = run;
        run += c;
    }
    uint32_t *st = status + (int64_t)tile * 256;
    if (tile == 0) st_atomic(&st[t], FLAG_INC | run);
    else st_atomic(&st[t], FLAG_AGG | run);
    // block exclusive scan of `run` over digits -> s_start
    uint32_t x = run;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_scan[warp] = x;
    __syncthreads();
    uint32_t wpre = 0;
#pragma unroll
    for (int w = 0; w < WARPS; w++)
        if (w < warp) wpre += s_scan[w];
    const uint32_t excl = wpre + x - run;
    s_start[t] = excl;
    if (t == 255) s_total = excl + run;
    // decoupled look-back over preceding tiles
    uint32_t prefix = 0;
    if (tile > 0) {
        int j = tile - 1;
        while (j >= 0) {
            uint32_t s = ld_volatile(&status[(int64_t)j * 256 + t]);
            uint32_t flag = s & ~VAL_MASK;
            if (flag == 0u) continue;
            prefix += s & VAL_MASK;
            if (flag == FLAG_INC) break;
            j--;
        }
        st_atomic(&st[t], FLAG_INC | (prefix + run));
    }
    s_base[t] = bins[t] + prefix - excl;
    __syncthreads();
#pragma unroll
    for (int i = 0; i < RS_ITEMS; i++) {
        const uint32_t d = dig[i];
        if (d < 256u) s_keys[s_start[d] + s_warp[warp][d] + rank[i]] = key[i];
    }
    __syncthreads();
    const uint32_t total = s_total;
    for (uint32_t j = threadIdx.x; j < total; j += RS_THREADS) {
        const K k = s_keys[j];
        const uint32_t d = (uint32_t)(k >> shift) & 255u;
        out[s_base[d] + j] = k;
    }
}

// ---------------------------------------------------------------------------
// single-pass exclusive scan (decoupled look-back) of int32 counts; total -> *total_out
constexpr int SC_ITEMS = 16;
constexpr int SC_TILE = RS_THREADS * SC_ITEMS;

__global__ void __launch_bounds__(RS_THREADS) scan_kernel(const int32_t *__restrict__ vals,
                                                          const uint64_t *__restrict__ perm, int32_t *data,
                                                          int64_t n_host, const int32_t *n_dev,
                                                          uint32_t *status, int32_t *ticket, int32_t *total_out,
                                                          int64_t capacity, int32_t *overflow, int32_t *eff_out) {
    __shared__ int s_tile;
    __shared__ uint32_t s_warp[RS_THREADS / 32];
    __shared__ uint32_t s_prefix;
    const int64_t n = n_dev ? (int64_t)*n_dev : n_host;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1);
    __syncthreads();
    const int tile = s_tile;
    const int64_t tbase = (int64_t)tile * SC_TILE;
    if (tbase >= n && !(tile == 0 && n == 0)) return;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t v[SC_ITEMS];
    uint32_t sum = 0;
    const int64_t mybase = tbase + (int64_t)threadIdx.x * SC_ITEMS;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; i++) {
        // value of rank mybase+i: kept count of the Gaussian at that depth rank (huge
        // Gaussians, encoded negative, emit nothing into the sort)
        v[i] = (mybase + i < n) ? (uint32_t)max(vals[(uint32_t)perm[mybase + i]], 0) : 0u;
        sum += v[i];
    }
    uint32_t x = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    uint32_t wpre = 0, agg = 0;
    for (int w = 0; w < RS_THREADS / 32; w++) {
        if (w < warp) wpre += s_warp[w];
        agg += s_warp[w];
    }
    if (threadIdx.x == 0) {
        uint32_t prefix = 0;
        if (tile == 0) {
            st_atomic(&status[0], FLAG_INC | agg);
        } else {
            st_atomic(&status[tile], FLAG_AGG | agg);
            int j = tile - 1;
            while (j >= 0) {
                uint32_t s = ld_volatile(&status[j]);
                uint32_t flag = s & ~VAL_MASK;
                if (flag == 0u) continue;
                prefix += s & VAL_MASK;
                if (flag == FLAG_INC) break;
                j--;
            }
            st_atomic(&status[tile], FLAG_INC | (prefix + agg));
        }
        s_prefix = prefix;
        if (tbase + SC_TILE >= n) {  // last tile
            const int64_t tot = (int64_t)(prefix + agg);
            *total_out = (int32_t)tot;
            if (tot > capacity) *overflow = 1;
            *eff_out = tot > capacity ? 0 : (int32_t)tot;
        }
    }
    __syncthreads();
    uint32_t run = s_prefix + wpre + x - sum;
#pragma unroll
    for (int i = 0; i < SC_ITEMS; i++) {
        if (mybase + i < n) data[mybase + i] = (int32_t)run;
        run += v[i];
    }
}

// ---------------------------------------------------------------------------
// emit kept pairs as (tile << 32 | id) at the scanned offsets, one thread per touched
// Gaussian in depth order.  The cull bits of the first 64 candidates come from preprocess;
// candidates beyond 64 are re-culled here (same strict decision function).
// entry word: 64-bit (tile << 32 | id), or 32-bit (tile << rank_bits | depth rank) when both fit
__device__ __forceinline__ void put_entry(void *out, int64_t pos, int rank_bits, int tile, uint32_t g, int64_t k) {
    if (rank_bits) reinterpret_cast<uint32_t *>(out)[pos] = ((uint32_t)tile << rank_bits) | (uint32_t)k;
    else reinterpret_cast<uint64_t *>(out)[pos] = ((uint64_t)(uint32_t)tile << 32) | (uint64_t)g;
}

__global__ void __launch_bounds__(256) emit_kernel(gs_frame f, const uint64_t *__restrict__ sorted, void *out,
                                                   int cull, int rank_bits) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t n_sorted = f.counters[GS_CNT_ACTIVE];
    if (k >= n_sorted || f.counters[GS_CNT_OVERFLOW]) return;
    const uint32_t g = (uint32_t)sorted[k];
    const int kept = f.kept[g];
    if (kept < 0) return;  // screen-covering: binned per tile by huge_count/merge
    int4 r = reinterpret_cast<const int4 *>(f.rect)[g];
    if (!cull) r = make_int4(0, f.tiles_x - 1, 0, f.tiles_y - 1);
    const int nx = r.y - r.x + 1;
    const int ncand = nx * (r.w - r.z + 1);
    if (cull && ncand > GS_SMALL_CAND) {  // large footprint: emitted warp-wide by emit_big_kernel
        f.big_emit[atomicAdd(&f.counters[GS_CNT_BIG_EMIT], 1)] = (int32_t)k;
        return;
    }
    const uint64_t bits = f.keep_bits[g];
    int64_t off = f.counts[k];
    for (int c = 0; c < ncand; c++) {
        const int tx = r.x + c % nx, ty = r.z + c / nx;
        if (!cull || ((bits >> c) & 1ull)) put_entry(out, off++, rank_bits, ty * f.tiles_x + tx, g, k);
    }
}

// warp per large-footprint Gaussian: lanes stride over candidates; ballot prefix gives the
// in-order slot (candidates in ty-major order, as the thread path writes them)
__global__ void __launch_bounds__(256) emit_big_kernel(gs_frame f, const uint64_t *__restrict__ sorted, void *out,
                                                       int rank_bits) {
    // one CTA per large-footprint Gaussian; 256 candidates per round, block-wide ordered slots
    __shared__ int s_warp[8];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (f.counters[GS_CNT_OVERFLOW]) return;
    const int64_t nb = f.counters[GS_CNT_BIG_EMIT];
    const unsigned ltmask = lanemask_lt();
    for (int64_t b = blockIdx.x; b < nb; b += gridDim.x) {
        const int64_t k = f.big_emit[b];
        const uint32_t g = (uint32_t)sorted[k];
        const float4 s0 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g];
        const float4 s1 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g + 1];
        const int4 r = reinterpret_cast<const int4 *>(f.rect)[g];
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        const int64_t base = (int64_t)f.keep_bits[g];  // cull bitmap from big_bands_kernel (-1: none)
        int64_t off = f.counts[k];
        for (int c0 = 0; c0 < ncand; c0 += 256) {
            const int c = c0 + threadIdx.x;
            const int tx = r.x + c % nx, ty = r.z + c / nx;
            bool keep = false;
            if (c < ncand) {
                if (base >= 0) keep = (f.big_bits[base + (c >> 5)] >> (c & 31)) & 1u;
                else {
                    const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
                    const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
                    keep = tile_keep(s0.x, s0.y, s0.z, s0.w, s1.x, s1.w, x0, x1, y0, y1);
                }
            }
            const unsigned bal = __ballot_sync(0xffffffffu, keep);
            if (lane == 0) s_warp[warp] = __popc(bal);
            __syncthreads();
            int before = 0, total = 0;
#pragma unroll
            for (int w = 0; w < 8; w++) {
                const int v = s_warp[w];
                before += w < warp ? v : 0;
                total += v;
            }
            if (keep) put_entry(out, off + before + __popc(bal & ltmask), rank_bits, ty * f.tiles_x + tx, g, k);
            off += total;
            __syncthreads();
        }
    }
}

// per-tile ranges of the tile-sorted (non-huge) entry words: small_off[t] = first word with
// tile >= t (adjacent-word compares)
template <typename K>
__global__ void ranges_kernel(gs_frame f, const K *__restrict__ sorted, int rank_bits) {
    const int64_t E = f.counters[GS_CNT_SMALL_E];
    const int32_t T = f.tiles_x * f.tiles_y;
    int32_t *small_off = f.tile_scratch;
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int tshift = rank_bits ? rank_bits : 32;
    if (E == 0) {
        for (int64_t t = e; t <= T; t += (int64_t)gridDim.x * blockDim.x) small_off[t] = 0;
        return;
    }
    for (int64_t i = e; i < E; i += (int64_t)gridDim.x * blockDim.x) {
        const int32_t tile = (int32_t)((uint64_t)sorted[i] >> tshift);
        const int32_t prev = i == 0 ? -1 : (int32_t)((uint64_t)sorted[i - 1] >> tshift);
        for (int32_t t = prev + 1; t <= tile; t++) small_off[t] = (int32_t)i;
        if (i == E - 1)
            for (int32_t t = tile + 1; t <= T; t++) small_off[t] = (int32_t)E;
    }
}

// ---------------------------------------------------------------------------
// screen-covering ("huge") Gaussians: binned per tile from their cull bitmaps in depth order,
// then merged with the tile's sorted entries.  They never enter the emit + sort.

// Huge records (depth order), 8 ints each: id, depth rank, slot; then their ids alone (depth
// order), then the per-chunk counts of the ordered compaction
constexpr int HREC = 8;
constexpr int HIDS = HREC * GS_HUGE_CAP;
constexpr int HCNT0 = HIDS + GS_HUGE_CAP;
constexpr int HCHUNK = 1024;

// ordered compaction of the huge Gaussians from the depth-sorted list, pass 1: counts per chunk
__global__ void __launch_bounds__(HCHUNK) huge_flag_count_kernel(gs_frame f, const uint64_t *__restrict__ sorted) {
    __shared__ int s;
    if (f.counters[GS_CNT_HUGE] == 0) return;
    if (threadIdx.x == 0) s = 0;
    __syncthreads();
    const int64_t k = (int64_t)blockIdx.x * HCHUNK + threadIdx.x;
    const bool h = k < f.counters[GS_CNT_ACTIVE] && f.kept[(uint32_t)sorted[k]] < 0;
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if ((threadIdx.x & 31) == 0 && m) atomicAdd(&s, __popc(m));
    __syncthreads();
    if (threadIdx.x == 0) f.huge[HCNT0 + blockIdx.x] = s;
}

// pass 2: each chunk sums its predecessors and writes its huge records in order
__global__ void __launch_bounds__(HCHUNK) huge_write_kernel(gs_frame f, const uint64_t *__restrict__ sorted) {
    __shared__ int s_warp[HCHUNK / 32];
    __shared__ int s_base;
    if (f.counters[GS_CNT_HUGE] == 0) return;
    const int32_t *chunk_cnt = f.huge + HCNT0;
    if (threadIdx.x == 0) s_base = 0;
    __syncthreads();
    int acc = 0;
    for (int c = threadIdx.x; c < (int)blockIdx.x; c += HCHUNK) acc += chunk_cnt[c];
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0 && acc) atomicAdd(&s_base, acc);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int64_t k = (int64_t)blockIdx.x * HCHUNK + threadIdx.x;
    uint32_t g = 0;
    bool h = false;
    if (k < f.counters[GS_CNT_ACTIVE]) {
        g = (uint32_t)sorted[k];
        h = f.kept[g] < 0;
    }
    const unsigned m = __ballot_sync(0xffffffffu, h);
    if (lane == 0) s_warp[warp] = __popc(m);
    __syncthreads();
    int pos = s_base;
    for (int w = 0; w < warp; w++) pos += s_warp[w];
    pos += __popc(m & ((1u << lane) - 1u));
    // merge key of every depth rank: the huge Gaussians ahead of it
    if (k < f.counters[GS_CNT_ACTIVE]) f.huge_before[k] = pos;
    if (h && pos < GS_HUGE_CAP) {
        int4 *rec = reinterpret_cast<int4 *>(f.huge + HREC * pos);
        rec[0] = make_int4((int)g, (int)k, -f.kept[g] - 1, 0);  // id, depth rank, huge slot
        f.huge[HIDS + pos] = (int)g;
    }
    if (threadIdx.x == 0) {
        int tot = 0;
        for (int w = 0; w < HCHUNK / 32; w++) tot += s_warp[w];
        if (tot) atomicAdd(&f.counters[GS_CNT_HUGE_N], tot);
    }
}

// Per-tile masks in depth order: bit j of huge_mask[t][w] <-> huge record 32w + j keeps tile t
// (a 32 x 32 bit transpose per warp of huge_mask_t rows, which the big_* cull kernels wrote by slot),
// plus the per-tile huge counts.
__global__ void __launch_bounds__(256) huge_transpose_kernel(gs_frame f) {
    const int T = f.tiles_x * f.tiles_y, tw = (T + 31) >> 5;
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const int lane = threadIdx.x & 31;
    const int w = blockIdx.y * 8 + (threadIdx.x >> 5);  // 32 records in depth order
    if (32 * w >= nrec) return;
    const int u = blockIdx.x;  // 32 tiles
    const int i = 32 * w + lane;
    uint32_t v = 0u;
    if (i < nrec) v = f.huge_mask_t[(int64_t)f.huge[HREC * i + 2] * tw + u];
    uint32_t mine = 0u;
#pragma unroll
    for (int j = 0; j < 32; j++) {
        const uint32_t b = __ballot_sync(0xffffffffu, (v >> j) & 1u);
        if (lane == j) mine = b;
    }
    const int t = 32 * u + lane;
    if (t < T) {
        f.huge_mask[(int64_t)t * (GS_HUGE_CAP / 32) + w] = mine;
        if (mine) atomicAdd(&f.tile_scratch[T + 1 + t], __popc(mine));
    }
}

// one CTA: tile_offsets = exclusive scan of (sorted entries + huge entries) per tile; E total
__global__ void __launch_bounds__(1024) tile_scan_kernel(gs_frame f) {
    __shared__ int32_t s_warp[32];
    __shared__ int32_t s_carry;
    const int T = f.tiles_x * f.tiles_y;
    const int32_t *small_off = f.tile_scratch, *hcount = f.tile_scratch + T + 1;
    const bool use_huge = min(f.counters[GS_CNT_HUGE], GS_HUGE_CAP) > 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x == 0) s_carry = 0;
    __syncthreads();
    for (int t0 = 0; t0 < T; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const int v = t < T ? (small_off[t + 1] - small_off[t]) + (use_huge ? hcount[t] : 0) : 0;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) s_warp[warp] = x;
        __syncthreads();
        int before = s_carry, total = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            before += w < warp ? s_warp[w] : 0;
            total += s_warp[w];
        }
        if (t < T) f.tile_offsets[t] = before + x - v;
        __syncthreads();
        if (threadIdx.x == 0) s_carry += total;
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t E = s_carry;
        f.tile_offsets[T] = (int32_t)E;
        f.counters[GS_CNT_ENTRIES] = (int32_t)E;
        const bool over = f.counters[GS_CNT_OVERFLOW] || E > f.entry_capacity;
        if (over) f.counters[GS_CNT_OVERFLOW] = 1;
        f.counters[GS_CNT_ENTRIES_EFF] = over ? 0 : (int32_t)E;
    }
}

// CTA per tile: merge the tile's huge Gaussians (depth order: the set bits of its mask words)
// with its tile-sorted entries (depth order) and write entry_splat.  Keys: a huge record's
// index i, a sorted entry's huge_before h (huge records ahead of its depth rank), so record i
// precedes the entry iff i < h.  On an overflow every range is emptied.
constexpr int MERGE_B = 2048;

template <typename K>
__global__ void __launch_bounds__(256) merge_kernel(gs_frame f, const K *__restrict__ sorted, int rank_bits,
                                                    const uint64_t *__restrict__ depth_sorted) {
    __shared__ int32_t s_a[GS_HUGE_CAP];
    __shared__ uint32_t s_isb[(GS_HUGE_CAP + MERGE_B) / 32];
    __shared__ int32_t s_wpre[(GS_HUGE_CAP + MERGE_B) / 32];
    __shared__ int s_warp[8];
    const int T = f.tiles_x * f.tiles_y;
    const int t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (f.counters[GS_CNT_OVERFLOW]) {
        if (tid == 0) f.tile_offsets[t] = 0;
        if (t == 0 && tid == 1) f.tile_offsets[T] = 0;
        return;
    }
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const int off = f.tile_offsets[t];
    const int sb = f.tile_scratch[t], nb = f.tile_scratch[t + 1] - sb;
    const uint32_t rmask = rank_bits ? (1u << rank_bits) - 1u : 0u;
    int32_t *out = f.entry_splat + off;
    auto b_id = [&](int j) -> int {
        const K w = sorted[sb + j];
        return rank_bits ? (int)(uint32_t)depth_sorted[(uint32_t)w & rmask] : (int)(uint32_t)w;
    };
    // A: expand the depth-ordered mask words (thread per word)
    const int nw = (nrec + 31) >> 5;
    uint32_t v = tid < nw ? f.huge_mask[(int64_t)t * (GS_HUGE_CAP / 32) + tid] : 0u;
    const int c = __popc(v);
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_warp[warp] = x;
    __syncthreads();
    int na = 0, pos = x - c;
#pragma unroll
    for (int w = 0; w < 8; w++) {
        const int sw = s_warp[w];
        pos += w < warp ? sw : 0;
        na += sw;
    }
    if (tid < nw) s_wpre[tid] = pos;
    __syncthreads();
    // expand: a warp per word, lane j <-> bit j (coalesced shared stores)
    for (int w = warp; w < nw; w += 8) {
        const uint32_t word = f.huge_mask[(int64_t)t * (GS_HUGE_CAP / 32) + w];
        if ((word >> lane) & 1u) s_a[s_wpre[w] + __popc(word & ((1u << lane) - 1u))] = 32 * w + lane;
    }
    if (na == 0) {  // no huge Gaussian in this tile: the sorted entries as they are
        for (int j = tid; j < nb; j += 256) out[j] = b_id(j);
        return;
    }
    const int total = na + nb;
    const int32_t *hid = f.huge + HIDS;
    if (nb <= MERGE_B) {
        // B element j lands at j + #{A preceding it} (binary search in A); its slot is marked in
        // a bitmap.  Every other output d is A element d - #{B slots before d}.  Both write
        // passes are coalesced.
        const int tw = (total + 31) >> 5;
        for (int w = tid; w < tw; w += 256) s_isb[w] = 0u;
        __syncthreads();
        for (int j = tid; j < nb; j += 256) {
            const int h = f.huge_before[(uint32_t)sorted[sb + j] & rmask];
            int lo = 0, hi = na;
            while (lo < hi) {
                const int mid = (lo + hi) >> 1;
                if (s_a[mid] < h) lo = mid + 1;
                else hi = mid;
            }
            const int d = j + lo;
            out[d] = b_id(j);
            atomicOr(&s_isb[d >> 5], 1u << (d & 31));
        }
        __syncthreads();
        // exclusive prefix of the B-slot popcounts per word (tw <= 192 words)
        const int cnt = tid < tw ? __popc(s_isb[tid]) : 0;
        int xx = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xx, o);
            if (lane >= o) xx += y;
        }
        if (lane == 31) s_warp[warp] = xx;
        __syncthreads();
        int pre = xx - cnt;
        for (int w = 0; w < warp; w++) pre += s_warp[w];
        if (tid < tw) s_wpre[tid] = pre;
        __syncthreads();
        for (int d = tid; d < total; d += 256) {
            const uint32_t word = s_isb[d >> 5];
            if ((word >> (d & 31)) & 1u) continue;
            const int a = d - (s_wpre[d >> 5] + __popc(word & ((1u << (d & 31)) - 1u)));
            out[d] = hid[s_a[a]];
        }
        return;
    }
    // many sorted entries: merge path, each thread merges a run of ceil(total / 256) outputs
    __syncthreads();
    auto bh = [&](int j) -> int { return f.huge_before[(uint32_t)sorted[sb + j] & rmask]; };
    const int L = (total + 255) / 256;
    const int d0 = min(tid * L, total), d1 = min(d0 + L, total);
    if (d0 >= d1) return;
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {  // a = number of A among the first d0 outputs
        const int mid = (lo + hi) >> 1;
        if (s_a[mid] < bh(d0 - 1 - mid)) lo = mid + 1;
        else hi = mid;
    }
    int aa = lo, bb = d0 - lo;
    int hb = bb < nb ? bh(bb) : 0;
    for (int d = d0; d < d1; d++) {
        if (bb >= nb || (aa < na && s_a[aa] < hb)) {
            out[d] = hid[s_a[aa]];
            aa++;
        } else {
            out[d] = b_id(bb);
            bb++;
            if (bb < nb) hb = bh(bb);
        }
    }
}

// cull=False: every valid Gaussian lands in every tile (R/rasterizer.py:195-199)
__global__ void nocull_kernel(gs_frame f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool v = false;
    if (i < f.n) {
        v = f.valid[i] != 0;
        const float d = f.splat2d[12 * i + 6];
        f.keys_a[i] = v ? (((uint64_t)__float_as_uint(d) << 32) | (uint64_t)i) : ((0xffffffffull << 32) | (uint64_t)i);
        f.kept[i] = v ? f.tiles_x * f.tiles_y : 0;
        f.touched[i] = v;
    }
    warp_append(v, (int32_t)i, &f.counters[GS_CNT_TOUCHED], f.touched_list);
}

template <typename K>
static int sort_pass(const gs_frame *f, const K *in, K *out, int64_t n_host, const int32_t *n_dev, int shift,
                     const uint32_t *bins, int pass_slot, int filter, cudaStream_t st) {
    const int64_t tiles = (n_host + RS_TILE - 1) / RS_TILE;
    if (tiles == 0) return GS_OK;
    uint32_t *status = f->sort_status + (int64_t)pass_slot * (f->status_words / 8);
    onesweep_kernel<K><<<(unsigned)tiles, RS_THREADS, 0, st>>>(in, out, n_host, n_dev, shift, bins, status,
                                                                f->counters + GS_CNT_TICKET0 + pass_slot, filter);
    return check_launch("onesweep_kernel");
}

// stable LSD sort of the entry words on the tile field; returns the buffer holding the result
template <typename K>
static int tile_sort(const gs_frame *f, K *a, K *b, int shift0, int tpasses, cudaStream_t st, K **result) {
    const int32_t *n_ent = f->counters + GS_CNT_SMALL_E;
    const int64_t cap = f->entry_capacity;
    radix_hist_kernel<K><<<4 * 148, 256, 0, st>>>(a, cap, n_ent, shift0, tpasses, f->sort_hist + 4 * 256, 0, nullptr);
    int rc = check_launch("radix_hist_kernel");
    if (rc) return rc;
    radix_bins_kernel<<<tpasses, 256, 0, st>>>(f->sort_hist + 4 * 256);
    K *src = a, *dst = b;
    for (int p = 0; p < tpasses; p++) {
        if ((rc = sort_pass<K>(f, src, dst, cap, n_ent, shift0 + 8 * p, f->sort_hist + (4 + p) * 256, 4 + p, 0, st)))
            return rc;
        K *tmp = src;
        src = dst;
        dst = tmp;
    }
    *result = src;
    return GS_OK;
}

void init_binning_attrs() {
    // the onesweep tiles want the full shared-memory carveout (occupancy is smem-limited)
    cudaFuncSetAttribute(onesweep_kernel<uint64_t>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(onesweep_kernel<uint32_t>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
}

}  // namespace gs

using namespace gs;

extern "C" int gs_bin(const gs_frame *f, int32_t cull, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = f->n;
    const int32_t T = f->tiles_x * f->tiles_y;
    int rc;
    // reset the binning counters (touched and huge belong to preprocess), histograms and
    // look-back state
    cudaMemsetAsync(f->counters + GS_CNT_ACTIVE, 0, sizeof(int32_t) * 2, st);
    cudaMemsetAsync(f->counters + GS_CNT_OVERFLOW, 0, sizeof(int32_t) * (GS_CNT_SLOTS - GS_CNT_OVERFLOW), st);
    cudaMemsetAsync(f->counters + GS_CNT_SMALL_E, 0, sizeof(int32_t) * 2, st);  // SMALL_E, HUGE_N
    cudaMemsetAsync(f->sort_hist, 0, sizeof(uint32_t) * 8 * 256, st);
    cudaMemsetAsync(f->sort_status, 0, sizeof(uint32_t) * f->status_words, st);
    cudaMemsetAsync(f->scan_status, 0, sizeof(uint32_t) * f->scan_words, st);
    cudaMemsetAsync(f->tile_scratch + T + 1, 0, sizeof(int32_t) * T, st);  // per-tile huge counts
    if (n == 0) {
        cudaMemsetAsync(f->tile_offsets, 0, sizeof(int32_t) * (T + 1), st);
        return check_launch("gs_bin");
    }
    if (!cull) {  // every valid Gaussian in every tile: no huge binning, all through the sort
        cudaMemsetAsync(f->counters + GS_CNT_TOUCHED, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->counters + GS_CNT_HUGE, 0, sizeof(int32_t) * 2, st);
        nocull_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*f);
        if ((rc = check_launch("nocull_kernel"))) return rc;
    }
    const int hist_blocks = 4 * 148;
    // 1) depth sort of the touched Gaussians (4 passes over the 32 depth bits, the first pass
    //    drops untouched ones)
    radix_hist_kernel<uint64_t><<<hist_blocks, 256, 0, st>>>(f->keys_a, n, nullptr, 32, 4, f->sort_hist, 1,
                                                             f->counters + GS_CNT_ACTIVE);
    if ((rc = check_launch("radix_hist_kernel"))) return rc;
    radix_bins_kernel<<<4, 256, 0, st>>>(f->sort_hist);
    const int32_t *n_act = f->counters + GS_CNT_ACTIVE;
    if ((rc = sort_pass(f, f->keys_a, f->keys_b, n, nullptr, 32, f->sort_hist + 0 * 256, 0, 1, st))) return rc;
    if ((rc = sort_pass(f, f->keys_b, f->keys_a, n, n_act, 40, f->sort_hist + 1 * 256, 1, 0, st))) return rc;
    if ((rc = sort_pass(f, f->keys_a, f->keys_b, n, n_act, 48, f->sort_hist + 2 * 256, 2, 0, st))) return rc;
    if ((rc = sort_pass(f, f->keys_b, f->keys_a, n, n_act, 56, f->sort_hist + 3 * 256, 3, 0, st))) return rc;
    // 2) offsets of the sorted (non-huge) entries: exclusive scan of kept counts in depth order
    {
        const int64_t tiles = (n + SC_TILE - 1) / SC_TILE;
        scan_kernel<<<(unsigned)(tiles > 0 ? tiles : 1), RS_THREADS, 0, st>>>(
            f->kept, f->keys_a, f->counts, n, n_act, (uint32_t *)f->scan_status, f->counters + GS_CNT_TICKET0 + 7,
            f->counters + GS_CNT_ENTRIES, f->entry_capacity, f->counters + GS_CNT_OVERFLOW,
            f->counters + GS_CNT_SMALL_E);
        if ((rc = check_launch("scan_kernel"))) return rc;
    }
    // entry words: 32-bit (tile << rank_bits | depth rank) when tile and rank bits fit, so the
    // tile sort moves half the bytes; 64-bit (tile << 32 | id) otherwise
    int tile_bits = 0, rank_bits = 0;
    const bool compact = compact_words(n, T, &tile_bits, &rank_bits);
    const int tpasses = tile_bits <= 8 ? 1 : (tile_bits <= 16 ? 2 : 3);
    const int rb = compact ? rank_bits : 0;
    emit_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*f, f->keys_a, f->keys_b, cull, rb);
    if ((rc = check_launch("emit_kernel"))) return rc;
    emit_big_kernel<<<8 * 148, 256, 0, st>>>(*f, f->keys_a, f->keys_b, rb);
    if ((rc = check_launch("emit_big_kernel"))) return rc;
    {
        const unsigned chunks = (unsigned)((n + HCHUNK - 1) / HCHUNK);
        huge_flag_count_kernel<<<chunks, HCHUNK, 0, st>>>(*f, f->keys_a);
        if ((rc = check_launch("huge_flag_count_kernel"))) return rc;
        huge_write_kernel<<<chunks, HCHUNK, 0, st>>>(*f, f->keys_a);
        if ((rc = check_launch("huge_write_kernel"))) return rc;
        huge_transpose_kernel<<<dim3((unsigned)((T + 31) / 32), GS_HUGE_CAP / 256), 256, 0, st>>>(*f);
        if ((rc = check_launch("huge_transpose_kernel"))) return rc;
    }
    // 3) stable sort of the emitted entries on the tile field, their per-tile ranges
    uint32_t *res32 = nullptr;
    uint64_t *res64 = nullptr;
    if (compact) {
        uint32_t *a = reinterpret_cast<uint32_t *>(f->keys_b), *b = a + f->entry_capacity;
        if ((rc = tile_sort<uint32_t>(f, a, b, rank_bits, tpasses, st, &res32))) return rc;
        ranges_kernel<uint32_t><<<4 * 148, 256, 0, st>>>(*f, res32, rank_bits);
    } else {
        if ((rc = tile_sort<uint64_t>(f, f->keys_b, f->keys_a, 32, tpasses, st, &res64))) return rc;
        ranges_kernel<uint64_t><<<4 * 148, 256, 0, st>>>(*f, res64, 0);
    }
    if ((rc = check_launch("ranges_kernel"))) return rc;
    // 4) huge Gaussians per tile, tile offsets, merged entry lists
    tile_scan_kernel<<<1, 1024, 0, st>>>(*f);
    if ((rc = check_launch("tile_scan_kernel"))) return rc;
    if (compact) merge_kernel<uint32_t><<<T, 256, 0, st>>>(*f, res32, rank_bits, f->keys_a);
    else merge_kernel<uint64_t><<<T, 256, 0, st>>>(*f, res64, 0, f->keys_a);
    return check_launch("merge_kernel");
}
