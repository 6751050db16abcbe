// binning.cu -- tile binning: per-tile buckets sorted by depth, ranges, merged entry lists.
//
// Replaces R/rasterizer.py:169-219 (cull_tiles) and the `touched` bookkeeping of
// _reduce_entries (:424).  The reference enumerates (splat, tile) pairs in splat order, culls
// them exactly and lexsorts by (tile, depth, splat).  The exact cull itself runs in
// preprocess.cu (kept counts, cull bitmaps, huge-slot masks); here, with the 64-bit key
// (depth_f32_bits << 32 | id) -- a total order equal to lexsort((id, depth)) inside a tile:
//   1. per-tile counts of the kept pairs of the non-screen-covering Gaussians, taken where the
//      cull decides them (preprocess_kernel, big_finish_kernel; bucket_count for cull=False);
//   2. huge_sort: the screen-covering ("huge") Gaussians, already binned per tile by bitmap,
//      are sorted by key in one CTA (records in depth order);
//   3. huge_transpose: their per-tile masks in that order, per-tile counts;
//   4. tile_scan: tile ranges (bucket + huge counts), bucket offsets, E;
//   5. bucket_fill: every kept pair's key lands in its tile's bucket (atomic cursors);
//   6. tile_sort_merge: CTA per tile sorts its bucket in shared memory (bitonic; oversized
//      buckets merge-sorted in global memory) and merges it with the tile's huge list.
// No global sort: the buckets average a few hundred keys, the huge list a few thousand.
// Every kernel reads its element counts from device memory, so the sequence is graph-capturable.
#include <cstdio>

#include "common.cuh"

namespace gs {

// Huge records (depth order), 8 ints each: id, depth bits, slot; then their ids alone, then
// their 64-bit keys
constexpr int HREC = 8;
constexpr int HIDS = HREC * GS_HUGE_CAP;
constexpr int HKEYS = HIDS + GS_HUGE_CAP;  // int offset of the uint64 key array (8-B aligned)

__device__ __forceinline__ uint64_t depth_key(const gs_frame &f, int g) {
    return ((uint64_t)__float_as_uint(f.splat2d[12 * (int64_t)g + 6]) << 32) | (uint32_t)g;
}

// Calls fn(tile) for every kept tile of a non-huge touched Gaussian, in candidate order
// (ty-major, then tx, R/rasterizer.py:113-122).
template <typename F>
__device__ __forceinline__ void for_kept_tiles(const gs_frame &f, int g, F fn) {
    const int4 r = reinterpret_cast<const int4 *>(f.rect)[g];
    const int nx = r.y - r.x + 1;
    const int ncand = nx > 0 ? nx * (r.w - r.z + 1) : 0;
    if (ncand <= GS_SMALL_CAND) {  // cull bits from preprocess_kernel
        const uint64_t bits = f.keep_bits[g];
        for (int c = 0; c < ncand; c++)
            if ((bits >> c) & 1ull) fn((r.z + c / nx) * f.tiles_x + r.x + c % nx);
        return;
    }
    // large footprint: bitmap of the big_* cull kernels, or the exact test again on overflow
    const int64_t base = (int64_t)f.keep_bits[g];
    const float4 s0 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g];
    const float4 s1 = reinterpret_cast<const float4 *>(f.splat2d)[3 * g + 1];
    for (int c = 0; c < ncand; c++) {
        const int tx = r.x + c % nx, ty = r.z + c / nx;
        bool keep;
        if (base >= 0) {
            keep = (f.big_bits[base + (c >> 5)] >> (c & 31)) & 1u;
        } else {
            const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
            const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
            keep = tile_keep(s0.x, s0.y, s0.z, s0.w, s1.x, s1.w, x0, x1, y0, y1);
        }
        if (keep) fn(ty * f.tiles_x + tx);
    }
}

// cull=False: every valid Gaussian lands in every tile (R/rasterizer.py:195-199)
__global__ void nocull_kernel(gs_frame f) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool v = false;
    if (i < f.n) {
        v = f.valid[i] != 0;
        f.kept[i] = v ? f.tiles_x * f.tiles_y : 0;
        f.touched[i] = v;
    }
    warp_append(v, (int32_t)i, &f.counters[GS_CNT_TOUCHED], f.touched_list);
}

// 1) per-tile bucket counts for cull=False (every tile holds every valid Gaussian); with the
// cull they are counted where the cull decides (preprocess_kernel, big_finish_kernel)
__global__ void __launch_bounds__(256) bucket_count_kernel(gs_frame f) {
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    const int T = f.tiles_x * f.tiles_y;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x)
        f.tile_scratch[t] = (int32_t)nt;
}

// 2) the huge Gaussians with >= 1 kept tile, sorted by key in one CTA: records in depth order
constexpr int HS_THREADS = 1024;

__global__ void __launch_bounds__(HS_THREADS) huge_sort_kernel(gs_frame f) {
    __shared__ uint64_t s_key[GS_HUGE_CAP];
    // the keys were staged (unordered) by big_finish_kernel
    uint64_t *keys = reinterpret_cast<uint64_t *>(f.huge + HKEYS);
    const int nh = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    for (int i = threadIdx.x; i < nh; i += HS_THREADS) s_key[i] = keys[i];
    int np = 1;
    while (np < nh) np <<= 1;
    for (int i = nh + threadIdx.x; i < np; i += HS_THREADS) s_key[i] = ~0ull;
    __syncthreads();
    for (int k = 2; k <= np; k <<= 1)
        for (int j = k >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += HS_THREADS) {
                const int l = i ^ j;
                if (l > i) {
                    const uint64_t a = s_key[i], c = s_key[l];
                    if ((a > c) == ((i & k) == 0)) {
                        s_key[i] = c;
                        s_key[l] = a;
                    }
                }
            }
            __syncthreads();
        }
    for (int i = threadIdx.x; i < nh; i += HS_THREADS) {
        const uint64_t key = s_key[i];
        const int g = (int)(uint32_t)key;
        reinterpret_cast<int4 *>(f.huge + HREC * i)[0] = make_int4(g, (int)(key >> 32), -f.kept[g] - 1, 0);
        f.huge[HIDS + i] = g;
        keys[i] = key;
    }
}

// 3) per-tile masks in depth order: bit j of huge_mask[t][w] <-> huge record 32w + j keeps tile
// t (a 32 x 32 bit transpose per warp of huge_mask_t rows, which the big_* cull kernels wrote
// by slot), plus the per-tile huge counts (tile_scratch[T+1 ..))
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

// 4) one CTA: tile_offsets = exclusive scan of (bucket + huge) counts; bucket offsets (both
// as the fill cursors, tile_scratch[0..T], and kept, tile_scratch[2T+2 ..]); E
__global__ void __launch_bounds__(1024) tile_scan_kernel(gs_frame f) {
    __shared__ int32_t s_warp[2][32];
    __shared__ int32_t s_carry[2];
    const int T = f.tiles_x * f.tiles_y;
    int32_t *cur = f.tile_scratch, *hcount = f.tile_scratch + T + 1, *boff = f.tile_scratch + 2 * (T + 1);
    const bool use_huge = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) > 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 2) s_carry[threadIdx.x] = 0;
    __syncthreads();
    for (int t0 = 0; t0 < T; t0 += blockDim.x) {
        const int t = t0 + threadIdx.x;
        const int vb = t < T ? cur[t] : 0;
        const int v = vb + (t < T && use_huge ? hcount[t] : 0);
        int x = v, xb = vb;
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o), yb = __shfl_up_sync(0xffffffffu, xb, o);
            if (lane >= o) {
                x += y;
                xb += yb;
            }
        }
        if (lane == 31) {
            s_warp[0][warp] = x;
            s_warp[1][warp] = xb;
        }
        __syncthreads();
        int before = s_carry[0], bb = s_carry[1], total = 0, totb = 0;
        for (int w = 0; w < (int)(blockDim.x >> 5); w++) {
            before += w < warp ? s_warp[0][w] : 0;
            bb += w < warp ? s_warp[1][w] : 0;
            total += s_warp[0][w];
            totb += s_warp[1][w];
        }
        if (t < T) {
            f.tile_offsets[t] = before + x - v;
            cur[t] = bb + xb - vb;
            boff[t] = bb + xb - vb;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            s_carry[0] += total;
            s_carry[1] += totb;
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const int64_t E = s_carry[0];
        f.tile_offsets[T] = (int32_t)E;
        boff[T] = s_carry[1];
        f.counters[GS_CNT_ENTRIES] = (int32_t)E;
        f.counters[GS_CNT_SMALL_E] = s_carry[1];
        const bool over = E > f.entry_capacity;
        if (over) f.counters[GS_CNT_OVERFLOW] = 1;
        f.counters[GS_CNT_ENTRIES_EFF] = over ? 0 : (int32_t)E;
    }
}

// 5) every bucketed pair's key into its tile's bucket (keys_b), unordered
__global__ void __launch_bounds__(256) bucket_fill_kernel(gs_frame f, int cull) {
    if (f.counters[GS_CNT_OVERFLOW]) return;
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    int32_t *cur = f.tile_scratch;
    uint64_t *bucket = f.keys_b;
    if (!cull) {  // every tile holds every valid Gaussian: bucket t = the touched list
        const int T = f.tiles_x * f.tiles_y;
        const int32_t *boff = f.tile_scratch + 2 * (T + 1);
        for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nt * T;
             i += (int64_t)gridDim.x * blockDim.x)
            bucket[boff[i / nt] + (i % nt)] = depth_key(f, f.touched_list[i % nt]);
        return;
    }
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nt; k += (int64_t)gridDim.x * blockDim.x) {
        const int g = f.touched_list[k];
        if (f.kept[g] <= 0) continue;
        const uint64_t key = depth_key(f, g);
        const int4 r = reinterpret_cast<const int4 *>(f.rect)[g];
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        if (ncand <= GS_SMALL_CAND) {
            // all slot reservations in flight before the first store
            const uint64_t bits = f.keep_bits[g];
            int pos[GS_SMALL_CAND];
#pragma unroll
            for (int c = 0; c < GS_SMALL_CAND; c++)
                if ((bits >> c) & 1ull) pos[c] = atomicAdd(&cur[(r.z + c / nx) * f.tiles_x + r.x + c % nx], 1);
#pragma unroll
            for (int c = 0; c < GS_SMALL_CAND; c++)
                if ((bits >> c) & 1ull) bucket[pos[c]] = key;
        } else {
            for_kept_tiles(f, g, [&](int t) { bucket[atomicAdd(&cur[t], 1)] = key; });
        }
    }
}

// 6) CTA per tile: sort the bucket, merge it with the tile's huge list, write entry_splat.
// A = the tile's huge records (record indices, ascending = depth order), B = the sorted bucket;
// B_j is preceded by exactly the records with key < key_j, hb_j of them in total, so record i
// precedes B_j iff i < hb_j.
constexpr int SM_THREADS = 256;
constexpr int SM_CAP = 4096;  // bucket keys sorted in shared memory at once

struct SortMergeSmem {
    uint64_t key[SM_CAP];
    int32_t a[GS_HUGE_CAP];
    uint32_t isb[(GS_HUGE_CAP + SM_CAP) / 32];
    int32_t wpre[(GS_HUGE_CAP + SM_CAP) / 32];
    int warp[SM_THREADS / 32];
};

__device__ __forceinline__ void bitonic_smem(uint64_t *k, int np) {
    for (int s = 2; s <= np; s <<= 1)
        for (int j = s >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += SM_THREADS) {
                const int l = i ^ j;
                if (l > i) {
                    const uint64_t a = k[i], c = k[l];
                    if ((a > c) == ((i & s) == 0)) {
                        k[i] = c;
                        k[l] = a;
                    }
                }
            }
            __syncthreads();
        }
}

// sorted B in shared memory (nb <= SM_CAP), or in global memory (returned) otherwise
__device__ const uint64_t *sort_bucket(SortMergeSmem &sm, uint64_t *src, uint64_t *tmp, int nb) {
    if (nb <= SM_CAP) {
        int np = 1;
        while (np < nb) np <<= 1;
        for (int i = threadIdx.x; i < np; i += SM_THREADS) sm.key[i] = i < nb ? src[i] : ~0ull;
        __syncthreads();
        bitonic_smem(sm.key, np);
        return sm.key;
    }
    // oversized bucket: sorted runs of SM_CAP in shared memory, then pairwise merges in global
    // memory (each element's output slot = its rank in its run + its rank in the other run)
    for (int c0 = 0; c0 < nb; c0 += SM_CAP) {
        const int m = min(SM_CAP, nb - c0);
        int np = 1;
        while (np < m) np <<= 1;
        for (int i = threadIdx.x; i < np; i += SM_THREADS) sm.key[i] = i < m ? src[c0 + i] : ~0ull;
        __syncthreads();
        bitonic_smem(sm.key, np);
        for (int i = threadIdx.x; i < m; i += SM_THREADS) src[c0 + i] = sm.key[i];
        __syncthreads();
    }
    for (int w = SM_CAP; w < nb; w <<= 1) {
        for (int i = threadIdx.x; i < nb; i += SM_THREADS) {
            const int lo = (i / (2 * w)) * (2 * w), mid = min(lo + w, nb), hi = min(lo + 2 * w, nb);
            const uint64_t v = src[i];
            const bool in_a = i < mid;
            int a = in_a ? mid : lo, b = in_a ? hi : mid;  // rank in the other run
            while (a < b) {
                const int m = (a + b) >> 1;
                if (src[m] < v) a = m + 1;
                else b = m;
            }
            tmp[lo + (i - (in_a ? lo : mid)) + (a - (in_a ? mid : lo))] = v;
        }
        __syncthreads();
        uint64_t *t = src;
        src = tmp;
        tmp = t;
    }
    return src;
}

__global__ void __launch_bounds__(SM_THREADS) tile_sort_merge_kernel(gs_frame f) {
    extern __shared__ uint64_t sm_raw[];
    SortMergeSmem &sm = *reinterpret_cast<SortMergeSmem *>(sm_raw);
    const int T = f.tiles_x * f.tiles_y;
    const int t = blockIdx.x;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    if (f.counters[GS_CNT_OVERFLOW]) {
        if (tid == 0) f.tile_offsets[t] = 0;
        if (t == 0 && tid == 1) f.tile_offsets[T] = 0;
        return;
    }
    const int32_t *boff = f.tile_scratch + 2 * (T + 1);
    const int sb = boff[t], nb = boff[t + 1] - sb;
    int32_t *out = f.entry_splat + f.tile_offsets[t];
    const uint64_t *B = sort_bucket(sm, f.keys_b + sb, f.keys_a + sb, nb);
    // A: expand the depth-ordered mask words (prefix of the per-word popcounts, then a warp per
    // word, lane j <-> bit j)
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const int nw = (nrec + 31) >> 5;
    const uint32_t *mask = f.huge_mask + (int64_t)t * (GS_HUGE_CAP / 32);
    const int c = tid < nw ? __popc(mask[tid]) : 0;
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) sm.warp[warp] = x;
    __syncthreads();
    int na = 0, pos = x - c;
#pragma unroll
    for (int w = 0; w < SM_THREADS / 32; w++) {
        const int sw = sm.warp[w];
        pos += w < warp ? sw : 0;
        na += sw;
    }
    if (tid < nw) sm.wpre[tid] = pos;
    __syncthreads();
    for (int w = warp; w < nw; w += SM_THREADS / 32) {
        const uint32_t word = mask[w];
        if ((word >> lane) & 1u) sm.a[sm.wpre[w] + __popc(word & ((1u << lane) - 1u))] = 32 * w + lane;
    }
    if (na == 0) {  // no huge Gaussian in this tile: the sorted bucket as it is
        for (int j = tid; j < nb; j += SM_THREADS) out[j] = (int32_t)(uint32_t)B[j];
        return;
    }
    __syncthreads();  // sm.a complete
    const uint64_t *hkeys = reinterpret_cast<const uint64_t *>(f.huge + HKEYS);
    const int32_t *hid = f.huge + HIDS;
    auto huge_before = [&](uint64_t key) -> int {  // records with a smaller key
        int lo = 0, hi = nrec;
        while (lo < hi) {
            const int m = (lo + hi) >> 1;
            if (hkeys[m] < key) lo = m + 1;
            else hi = m;
        }
        return lo;
    };
    const int total = na + nb;
    // the common case: every huge Gaussian of the tile is in front of every bucketed one
    // (screen-covering Gaussians hug the near plane): the merged list is a concatenation
    if (nb == 0 || hkeys[sm.a[na - 1]] < B[0]) {
        for (int d = tid; d < total; d += SM_THREADS) out[d] = d < na ? hid[sm.a[d]] : (int32_t)(uint32_t)B[d - na];
        return;
    }
    if (nb <= SM_CAP) {
        // B_j lands at j + #{A preceding it}; its slot is marked in a bitmap.  Every other output
        // d is A element d - #{B slots before d}.  Both write passes are coalesced.
        const int tw = (total + 31) >> 5;
        for (int w = tid; w < tw; w += SM_THREADS) sm.isb[w] = 0u;
        __syncthreads();
        for (int j = tid; j < nb; j += SM_THREADS) {
            const int h = huge_before(B[j]);
            int lo = 0, hi = na;
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (sm.a[m] < h) lo = m + 1;
                else hi = m;
            }
            const int d = j + lo;
            out[d] = (int32_t)(uint32_t)B[j];
            atomicOr(&sm.isb[d >> 5], 1u << (d & 31));
        }
        __syncthreads();
        const int cnt = tid < tw ? __popc(sm.isb[tid]) : 0;
        int xx = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, xx, o);
            if (lane >= o) xx += y;
        }
        if (lane == 31) sm.warp[warp] = xx;
        __syncthreads();
        int pre = xx - cnt;
        for (int w = 0; w < warp; w++) pre += sm.warp[w];
        if (tid < tw) sm.wpre[tid] = pre;
        __syncthreads();
        for (int d = tid; d < total; d += SM_THREADS) {
            const uint32_t word = sm.isb[d >> 5];
            if ((word >> (d & 31)) & 1u) continue;
            const int a = d - (sm.wpre[d >> 5] + __popc(word & ((1u << (d & 31)) - 1u)));
            out[d] = hid[sm.a[a]];
        }
        return;
    }
    // oversized bucket: merge path, each thread merges a run of ceil(total / 256) outputs
    __syncthreads();
    const int L = (total + SM_THREADS - 1) / SM_THREADS;
    const int d0 = min(tid * L, total), d1 = min(d0 + L, total);
    if (d0 >= d1) return;
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {  // a = number of A among the first d0 outputs
        const int m = (lo + hi) >> 1;
        if (sm.a[m] < huge_before(B[d0 - 1 - m])) lo = m + 1;
        else hi = m;
    }
    int aa = lo, bb = d0 - lo;
    int hb = bb < nb ? huge_before(B[bb]) : 0;
    for (int d = d0; d < d1; d++) {
        if (bb >= nb || (aa < na && sm.a[aa] < hb)) {
            out[d] = hid[sm.a[aa]];
            aa++;
        } else {
            out[d] = (int32_t)(uint32_t)B[bb];
            bb++;
            if (bb < nb) hb = huge_before(B[bb]);
        }
    }
}

void init_binning_attrs() {
    cudaFuncSetAttribute(tile_sort_merge_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)sizeof(SortMergeSmem));
}

}  // namespace gs

using namespace gs;

extern "C" int gs_bin(const gs_frame *f, int32_t cull, void *stream) {
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t n = f->n;
    const int32_t T = f->tiles_x * f->tiles_y;
    int rc;
    // reset the binning counters (touched, big and huge belong to preprocess) and the per-tile
    // counts
    cudaMemsetAsync(f->counters + GS_CNT_ENTRIES, 0, sizeof(int32_t), st);
    cudaMemsetAsync(f->counters + GS_CNT_OVERFLOW, 0, sizeof(int32_t) * 2, st);  // OVERFLOW, ENTRIES_EFF
    cudaMemsetAsync(f->counters + GS_CNT_SMALL_E, 0, sizeof(int32_t), st);
    if (n == 0) {
        cudaMemsetAsync(f->tile_offsets, 0, sizeof(int32_t) * (T + 1), st);
        return check_launch("gs_bin");
    }
    if (!cull) {  // every valid Gaussian in every tile: no huge binning
        cudaMemsetAsync(f->counters + GS_CNT_TOUCHED, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->counters + GS_CNT_HUGE, 0, sizeof(int32_t) * 2, st);
        cudaMemsetAsync(f->counters + GS_CNT_HUGE_N, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->tile_scratch + T + 1, 0, sizeof(int32_t) * ((size_t)T + 1), st);  // no huge
        nocull_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(*f);
        if ((rc = check_launch("nocull_kernel"))) return rc;
        bucket_count_kernel<<<4 * 148, 256, 0, st>>>(*f);
        if ((rc = check_launch("bucket_count_kernel"))) return rc;
    }
    if (cull) {  // the bucket counts come from the cull (preprocess, big_finish)
        huge_sort_kernel<<<1, HS_THREADS, 0, st>>>(*f);
        if ((rc = check_launch("huge_sort_kernel"))) return rc;
        huge_transpose_kernel<<<dim3((unsigned)((T + 31) / 32), GS_HUGE_CAP / 256), 256, 0, st>>>(*f);
        if ((rc = check_launch("huge_transpose_kernel"))) return rc;
    }
    tile_scan_kernel<<<1, 1024, 0, st>>>(*f);
    if ((rc = check_launch("tile_scan_kernel"))) return rc;
    bucket_fill_kernel<<<4 * 148, 256, 0, st>>>(*f, cull);
    if ((rc = check_launch("bucket_fill_kernel"))) return rc;
    tile_sort_merge_kernel<<<T, SM_THREADS, sizeof(SortMergeSmem), st>>>(*f);
    return check_launch("tile_sort_merge_kernel");
}
