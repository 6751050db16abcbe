// binning.cu -- tile binning: per-tile buckets sorted by depth, ranges, merged entry lists.
//
// Replaces R/rasterizer.py:169-219 (cull_tiles) and the `touched` bookkeeping of
// _reduce_entries (:424).  The reference enumerates (splat, tile) pairs in splat order, culls
// them exactly and lexsorts by (tile, depth, splat).  The exact cull itself runs in
// preprocess.cu (kept counts, cull bitmaps, huge-slot masks); here, with the 64-bit key
// (depth_f32_bits << 32 | id) -- a total order equal to lexsort((id, depth)) inside a tile:
//   1. per-tile counts of the kept pairs of the non-screen-covering Gaussians, taken where the
//      cull decides them (preprocess_kernel, big_cull_kernel; bucket_count for cull=False);
//   2. huge_sort: the screen-covering ("huge") Gaussians, already binned per tile by bitmap,
//      are rank-sorted by key (records in depth order);
//   3. huge_transpose: their per-tile masks in that order, per-tile counts;
//   4. tile_scan: tile ranges (bucket + huge counts), bucket offsets, E;
//   5. bucket_fill: every kept pair's key lands in its tile's bucket (atomic cursors);
//   6. tile_sort_merge: CTA per tile sorts its bucket in shared memory (bitonic; oversized
//      buckets merge-sorted in global memory) and merges it with the tile's huge list.
// No global sort: the buckets average a few hundred keys, the huge list a few thousand.
// Every kernel reads its element counts from device memory, so the sequence is graph-capturable.
#include <cstdio>

#include "tilelist.cuh"

namespace gs {

// Calls fn(tile) for every kept tile of a non-huge touched Gaussian, in candidate order
// (ty-major, then tx, R/rasterizer.py:113-122).
template <typename F>
__device__ __forceinline__ void for_kept_tiles(const gs_frame &f, int g, F fn) {
    const int4 r = bin_rec(f)[g].rect;
    const int nx = r.y - r.x + 1;
    const int ncand = nx > 0 ? nx * (r.w - r.z + 1) : 0;
    if (ncand <= GS_SMALL_CAND) {  // cull bits from preprocess_kernel
        const uint64_t bits = bin_rec(f)[g].bits;
        for (int c = 0; c < ncand; c++)
            if ((bits >> c) & 1ull) fn((r.z + c / nx) * f.tiles_x + r.x + c % nx);
        return;
    }
    // large footprint: bitmap of the big_* cull kernels, or the exact test again on overflow
    const int64_t base = (int64_t)bin_rec(f)[g].bits;
    const SplatCull s = splat_cull(f.splat2d, g);
    for (int c = 0; c < ncand; c++) {
        const int tx = r.x + c % nx, ty = r.z + c / nx;
        bool keep;
        if (base >= 0) {
            keep = (f.big_bits[base + (c >> 5)] >> (c & 31)) & 1u;
        } else {
            const int x0 = tx * GS_TILE, y0 = ty * GS_TILE;
            const int x1 = min(x0 + GS_TILE - 1, f.width - 1), y1 = min(y0 + GS_TILE - 1, f.height - 1);
            keep = tile_keep(s.mx, s.my, s.ca, s.cb, s.cc, s.qcut, x0, x1, y0, y1);
        }
        if (keep) fn(ty * f.tiles_x + tx);
    }
}

// cull=False: every valid Gaussian lands in every tile (R/rasterizer.py:195-199)
__global__ void nocull_kernel(gs_frame f) {
    pdl_wait();
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    bool v = false;
    if (i < f.n) {
        v = f.valid[i] != 0;
        bin_rec(f)[i].kept = v ? f.tiles_x * f.tiles_y : 0;
        f.touched[i] = v;
    }
    touched_append(f, v, (int32_t)i);
}

// 1) per-tile bucket counts for cull=False (every tile holds every valid Gaussian); with the
// cull they are counted where the cull decides (preprocess_kernel, big_cull_kernel)
__global__ void __launch_bounds__(256) bucket_count_kernel(gs_frame f) {
    pdl_wait();
    const int64_t nt = f.counters[GS_CNT_TOUCHED];
    const int T = f.tiles_x * f.tiles_y;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x)
        f.tile_scratch[t] = (int32_t)nt;
}

// 2) the huge Gaussians with >= 1 kept tile, in key order: a rank sort spread over the GPU.  Keys
// are unique (the id is in the low word), so a key's rank -- the number of smaller keys -- is its
// slot.  CTA c ranks keys [HS_KEYS c, HS_KEYS (c+1)): its HS_GROUPS thread groups each count
// over one slice of all keys (staged in shared memory), the partial counts are summed in shared
// memory and every record is written straight to its slot.  No atomics, no global sync.
#ifndef HS_KEYS_N
#define HS_KEYS_N 16
#endif
constexpr int HS_KEYS = HS_KEYS_N;
#ifndef HS_GROUPS_N
#define HS_GROUPS_N 64
#endif
constexpr int HS_GROUPS = HS_GROUPS_N;
constexpr int HS_THREADS = HS_KEYS * HS_GROUPS;

__global__ void __launch_bounds__(HS_THREADS) huge_sort_kernel(gs_frame f) {
    pdl_wait();
    __shared__ uint64_t s_key[GS_HUGE_CAP];
    __shared__ int s_part[HS_GROUPS][HS_KEYS];
    const int nh = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const int i0 = blockIdx.x * HS_KEYS;
    if (i0 >= nh) return;
    const uint64_t *staged = reinterpret_cast<const uint64_t *>(f.huge + HSTAGE);
    for (int i = threadIdx.x; i < nh; i += HS_THREADS) s_key[i] = staged[i];
    __syncthreads();
    const int k = threadIdx.x % HS_KEYS, grp = threadIdx.x / HS_KEYS;
    const int i = i0 + k;
    const uint64_t mine = i < nh ? s_key[i] : 0ull;
    const int per = (nh + HS_GROUPS - 1) / HS_GROUPS;
    const int j0 = grp * per, j1 = min(nh, j0 + per);
    int cnt = 0;
#pragma unroll 8
    for (int j = j0; j < j1; j++) cnt += s_key[j] < mine;  // same j across the warp: broadcast
    s_part[grp][k] = cnt;
    __syncthreads();
    if (grp == 0 && i < nh) {
        int rank = 0;
#pragma unroll
        for (int q = 0; q < HS_GROUPS; q++) rank += s_part[q][k];
        const int g = (int)(uint32_t)mine;
        reinterpret_cast<int4 *>(f.huge + HREC * rank)[0] = make_int4(g, (int)(mine >> 32), -bin_rec(f)[g].kept - 1, 0);
        f.huge[HIDS + rank] = g;
        reinterpret_cast<uint64_t *>(f.huge + HKEYS)[rank] = mine;
    }
}

// 3) per-tile masks in depth order: bit j of huge_mask[t][w] <-> huge record 32w + j keeps tile
// t (a 32 x 32 bit transpose per warp of huge_mask_t rows, which big_cull_kernel wrote
// by slot), plus the per-tile huge counts (tile_scratch[T+1 ..))
__global__ void __launch_bounds__(256) huge_transpose_kernel(gs_frame f) {
    pdl_wait();
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
        if (mine) atomicAdd(&ts_huge(f)[t], __popc(mine));
    }
}

// 4) one CTA: tile_offsets = exclusive scan of (bucket + huge) counts; bucket offsets (both
// as the fill cursors, tile_scratch[0..T], and kept, tile_scratch[2T+2 ..]); E.  Passes of
// TS_THREADS * TS_PER tiles: coalesced loads into shared memory, a sequential scan of TS_PER
// consecutive tiles per thread, one block scan of the per-thread sums, results back through
// shared memory and coalesced stores (a thread storing its own consecutive tiles would scatter
// every warp store over 32 sectors).
constexpr int TS_THREADS = 1024, TS_PER = 4;

__global__ void __launch_bounds__(TS_THREADS) tile_scan_kernel(gs_frame f, int lazy) {
    pdl_wait();
    __shared__ int32_t s_b[TS_THREADS * TS_PER], s_h[TS_THREADS * TS_PER];
    __shared__ int32_t s_warp[2][32];
    __shared__ int32_t s_pre[2][33];
    __shared__ int32_t s_carry[2];
    const int T = f.tiles_x * f.tiles_y;
    int32_t *cur = f.tile_scratch, *hcount = f.tile_scratch + T + 1, *boff = f.tile_scratch + 2 * (T + 1);
    int32_t *flag = ts_flag(f);
    const bool use_huge = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) > 0;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (threadIdx.x < 2) s_carry[threadIdx.x] = 0;
    constexpr int PASS = TS_THREADS * TS_PER;
    for (int t0 = 0; t0 < T; t0 += PASS) {
#pragma unroll
        for (int q = 0; q < TS_PER; q++) {  // coalesced loads
            const int i = q * TS_THREADS + threadIdx.x, t = t0 + i;
            s_b[i] = t < T ? cur[t] : 0;
            s_h[i] = (t < T && use_huge) ? hcount[t] : 0;
        }
        __syncthreads();
        int vb[TS_PER], vh[TS_PER], sx = 0, sb = 0;
#pragma unroll
        for (int q = 0; q < TS_PER; q++) {
            vb[q] = s_b[threadIdx.x * TS_PER + q];
            vh[q] = s_h[threadIdx.x * TS_PER + q];
            sx += vb[q] + vh[q];
            sb += vb[q];
        }
        int x = sx, xb = sb;  // inclusive warp scan of the per-thread sums
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
        if (warp == 0) {  // exclusive scan of the 32 warp totals by one warp
            const int w0 = s_warp[0][lane], w1 = s_warp[1][lane];
            int a0 = w0, a1 = w1;
            for (int o = 1; o < 32; o <<= 1) {
                const int y0 = __shfl_up_sync(0xffffffffu, a0, o), y1 = __shfl_up_sync(0xffffffffu, a1, o);
                if (lane >= o) {
                    a0 += y0;
                    a1 += y1;
                }
            }
            s_pre[0][lane] = a0 - w0;
            s_pre[1][lane] = a1 - w1;
            if (lane == 31) {
                s_pre[0][32] = a0;
                s_pre[1][32] = a1;
            }
        }
        __syncthreads();
        int run = s_carry[0] + s_pre[0][warp] + x - sx, runb = s_carry[1] + s_pre[1][warp] + xb - sb;
#pragma unroll
        for (int q = 0; q < TS_PER; q++) {  // exclusive prefixes back into shared memory
            s_b[threadIdx.x * TS_PER + q] = runb;
            s_h[threadIdx.x * TS_PER + q] = run;
            run += vb[q] + vh[q];
            runb += vb[q];
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < TS_PER; q++) {  // coalesced stores
            const int i = q * TS_THREADS + threadIdx.x, t = t0 + i;
            if (t < T) {
                f.tile_offsets[t] = s_h[i];
                cur[t] = s_b[i];
                boff[t] = s_b[i];
                flag[t] = TL_LAZY_A;  // lazy lists: the forward flags the tiles it cannot finish
            }
        }
        if (threadIdx.x == 0) {
            s_carry[0] += s_pre[0][32];
            s_carry[1] += s_pre[1][32];
        }
        __syncthreads();
    }
    const int64_t E = s_carry[0];
    const bool over = E > f.entry_capacity;
    if (threadIdx.x == 0) {
        f.tile_offsets[T] = over ? 0 : (int32_t)E;
        boff[T] = s_carry[1];
        f.counters[GS_CNT_ENTRIES] = (int32_t)E;
        f.counters[GS_CNT_SMALL_E] = s_carry[1];
        f.counters[GS_CNT_OVERFLOW] = over ? 1 : 0;
        f.counters[GS_CNT_ENTRIES_EFF] = over ? 0 : (int32_t)E;
        f.counters[GS_CNT_LAZY] = lazy;
        f.counters[GS_CNT_ANYFLAG] = 0;
        f.counters[GS_CNT_FLAGGED] = 0;
    }
    // over capacity: every tile range is emptied, so no later kernel (lazy or materialised lists,
    // forward, backward) can index entry_splat / keys past the capacity; the caller re-lays out
    // the workspace and repeats the frame
    if (over)
        for (int t = threadIdx.x; t < T; t += TS_THREADS) f.tile_offsets[t] = 0;
}

// 5) every bucketed pair's key into its tile's bucket (keys_b), unordered
__global__ void __launch_bounds__(256) bucket_fill_kernel(gs_frame f, int cull) {
    pdl_wait();
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
        if (bin_rec(f)[g].kept <= 0) continue;
        const uint64_t key = depth_key(f, g);
        const int4 r = bin_rec(f)[g].rect;
        const int nx = r.y - r.x + 1, ncand = nx * (r.w - r.z + 1);
        if (ncand <= GS_SMALL_CAND) {
            // all slot reservations in flight before the first store
            const uint64_t bits = bin_rec(f)[g].bits;
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

// 6) CTA per tile (materialised lists): sort the bucket, merge it with the tile's huge list,
// write entry_splat
constexpr int SM_THREADS = 256;

struct SortMergeSmem {
    uint64_t key[SM_CAP];
    int32_t a[GS_HUGE_CAP];
    uint32_t words[GS_HUGE_CAP / 32];
    int32_t wpre_a[GS_HUGE_CAP / 32];
    uint32_t isb[(GS_HUGE_CAP + SM_CAP) / 32];
    int32_t wpre[(GS_HUGE_CAP + SM_CAP) / 32];
    int32_t tmp[SM_THREADS / 32];
};

__global__ void __launch_bounds__(SM_THREADS) tile_sort_merge_kernel(gs_frame f) {
    pdl_wait();
    extern __shared__ uint64_t sm_raw[];
    SortMergeSmem &sm = *reinterpret_cast<SortMergeSmem *>(sm_raw);
    const int T = f.tiles_x * f.tiles_y;
    const int t = blockIdx.x;
    if (f.counters[GS_CNT_OVERFLOW]) {
        if (threadIdx.x == 0) f.tile_offsets[t] = 0;
        if (t == 0 && threadIdx.x == 1) f.tile_offsets[T] = 0;
        return;
    }
    const int sb = ts_boff(f)[t], nb = ts_boff(f)[t + 1] - sb;
    const uint64_t *B = sort_bucket<SM_THREADS>(sm.key, f.keys_b + sb, f.keys_a + sb, nb, false);
    const int na = tile_huge_setup(f, t, sm.words, sm.wpre_a, sm.tmp);
    const int nw = (min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP) + 31) >> 5;
    tile_huge_expand(sm.words, sm.wpre_a, nw, sm.a);
    merge_tile_list<SM_THREADS>(f, f.entry_splat + f.tile_offsets[t], sm.a, na, B, nb, sm.isb, sm.wpre, sm.tmp,
                                GS_HUGE_CAP + SM_CAP);
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
    const bool lazy = cull == GS_BIN_LAZY;
    int rc;
    if (cull < 0 || cull > GS_BIN_LAZY) {
        set_error("gs_bin: cull must be 0, 1 or GS_BIN_LAZY");
        return GS_ERR_ARG;
    }
    // reset the binning counters (touched, big and huge belong to preprocess) and the per-tile
    // counts
    // (tile_scan_kernel assigns the binning counters -- entries, small entries, overflow -- so a
    // repeated binning of one preprocess starts from its own values)
    if (n == 0) {
        cudaMemsetAsync(f->counters + GS_CNT_ENTRIES, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->counters + GS_CNT_OVERFLOW, 0, sizeof(int32_t) * 2, st);  // OVERFLOW, ENTRIES_EFF
        cudaMemsetAsync(f->counters + GS_CNT_SMALL_E, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->tile_offsets, 0, sizeof(int32_t) * (T + 1), st);
        return check_launch("gs_bin");
    }
    if (!cull) {  // every valid Gaussian in every tile: no huge binning
        cudaMemsetAsync(f->counters + GS_CNT_TOUCHED, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->counters + GS_CNT_HUGE, 0, sizeof(int32_t) * 2, st);
        cudaMemsetAsync(f->counters + GS_CNT_HUGE_N, 0, sizeof(int32_t), st);
        cudaMemsetAsync(f->tile_scratch + T + 1, 0, sizeof(int32_t) * ((size_t)T + 1), st);  // no huge
        launch_pdl(nocull_kernel, (unsigned)((n + 255) / 256), 256, 0, st, *f);
        if ((rc = check_launch("nocull_kernel"))) return rc;
        launch_pdl(bucket_count_kernel, 4 * 148, 256, 0, st, *f);
        if ((rc = check_launch("bucket_count_kernel"))) return rc;
    }
    if (cull) {  // the bucket counts come from the cull (preprocess, big_cull)
        launch_pdl(huge_sort_kernel, GS_HUGE_CAP / HS_KEYS, HS_THREADS, 0, st, *f);
        if ((rc = check_launch("huge_sort_kernel"))) return rc;
        launch_pdl(huge_transpose_kernel, dim3((unsigned)((T + 31) / 32), GS_HUGE_CAP / 256), 256, 0, st, *f);
        if ((rc = check_launch("huge_transpose_kernel"))) return rc;
    }
    launch_pdl(tile_scan_kernel, 1, TS_THREADS, 0, st, *f, lazy ? 1 : 0);
    if ((rc = check_launch("tile_scan_kernel"))) return rc;
    if (lazy) return GS_OK;  // buckets filled, sorted and merged on demand by gs_render_fwd
    launch_pdl(bucket_fill_kernel, 4 * 148, 256, 0, st, *f, cull);
    if ((rc = check_launch("bucket_fill_kernel"))) return rc;
    launch_pdl(tile_sort_merge_kernel, T, SM_THREADS, sizeof(SortMergeSmem), st, *f);
    return check_launch("tile_sort_merge_kernel");
}
