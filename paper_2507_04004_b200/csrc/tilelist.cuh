// tilelist.cuh -- per-tile entry lists shared by the binning and the blend (sm_100a).
//
// A tile's list (R/rasterizer.py:213-219 order: depth, then id) is the merge of
//   A: its screen-covering ("huge") Gaussians -- bits of the depth-ordered per-tile masks
//      (huge_mask[t][w], bit j <-> huge record 32w + j; records sorted by key), and
//   B: its bucket of the other kept Gaussians' keys (depth_f32_bits << 32 | id), sorted per
//      tile on demand.
// Record i precedes bucket key k iff hkeys[i] < k.  When every A key is smaller than every B
// key (the usual case: screen-covering Gaussians hug the near plane) the list is A then B.
#pragma once
#include "common.cuh"

namespace gs {


// tile_scratch segments (each tiles + 1 ints)
__device__ __forceinline__ int32_t *ts_cursor(const gs_frame &f) { return f.tile_scratch; }
__device__ __forceinline__ int32_t *ts_huge(const gs_frame &f) { return f.tile_scratch + (f.tiles_x * f.tiles_y + 1); }
__device__ __forceinline__ int32_t *ts_boff(const gs_frame &f) { return f.tile_scratch + 2 * (f.tiles_x * f.tiles_y + 1); }
__device__ __forceinline__ int32_t *ts_flag(const gs_frame &f) { return f.tile_scratch + 3 * (f.tiles_x * f.tiles_y + 1); }
__device__ __forceinline__ int32_t *ts_resume(const gs_frame &f) { return f.tile_scratch + 4 * (f.tiles_x * f.tiles_y + 1); }
// lazy lists: the ids of the tiles flagged for the continuation (GS_CNT_FLAGGED of them)
__device__ __forceinline__ int32_t *ts_flagged(const gs_frame &f) { return f.tile_scratch + 5 * (f.tiles_x * f.tiles_y + 1); }

// per-tile list state of lazy binning (ts_flag): the forward blends the leading run of
// screen-covering Gaussians (those ahead of every bucketed key); a tile whose blend outlives
// it gets its full merged list in entry_splat and is resumed at ts_resume by tile_finish_kernel
enum { TL_LAZY_A = 0, TL_LIST = 1 };

__device__ __forceinline__ const uint64_t *huge_keys(const gs_frame &f) {
    return reinterpret_cast<const uint64_t *>(f.huge + HKEYS);
}

__device__ __forceinline__ uint64_t depth_key(const gs_frame &f, int g) {
    return ((uint64_t)__float_as_uint(splat_depth(f.splat2d, g)) << 32) | (uint32_t)g;
}

// ---------------------------------------------------------------------------------------------
// records with a key below `key` (binary search over the sorted huge keys)
__device__ __forceinline__ int huge_before_key(const gs_frame &f, uint64_t key) {
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const uint64_t *hkeys = huge_keys(f);
    int lo = 0, hi = nrec;
    while (lo < hi) {
        const int m = (lo + hi) >> 1;
        if (hkeys[m] < key) lo = m + 1;
        else hi = m;
    }
    return lo;
}

// A elements of the tile with record index < h (rank in the setup words)
__device__ __forceinline__ int tile_huge_rank(int h, const uint32_t *s_words, const int32_t *s_wpre, int nw, int na) {
    const int w = h >> 5;
    if (w >= nw) return na;
    return s_wpre[w] + __popc(s_words[w] & ((1u << (h & 31)) - 1u));
}

// A of a tile: the depth-ordered mask words and their exclusive popcount prefix in shared
// memory (collective over the CTA; returns |A|).  s_tmp: >= blockDim.x / 32 ints.
__device__ __forceinline__ int tile_huge_setup(const gs_frame &f, int t, uint32_t *s_words, int32_t *s_wpre,
                                               int32_t *s_tmp) {
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const int nw = (nrec + 31) >> 5;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nwarps = blockDim.x >> 5;
    // thread tid holds words [K tid, K tid + K) (K = 1 for CTAs of >= GS_HUGE_CAP / 32 threads;
    // a 64-thread backward CTA needs K = 2 once there are more than 2048 records)
    constexpr int KMAX = 4;  // CTAs of >= GS_HUGE_CAP / 128 = 32 threads
    const int K = (GS_HUGE_CAP / 32 + blockDim.x - 1) / blockDim.x;
    const uint32_t *row = f.huge_mask + (int64_t)t * (GS_HUGE_CAP / 32);
    uint32_t wv[KMAX];
    int c = 0;
#pragma unroll
    for (int k = 0; k < KMAX; k++) {
        const int w = K * tid + k;
        wv[k] = (k < K && w < nw) ? row[w] : 0u;
        c += __popc(wv[k]);
    }
    int x = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) s_tmp[warp] = x;
    __syncthreads();
    int na = 0, pos = x - c;
    for (int w = 0; w < nwarps; w++) {
        const int sw = s_tmp[w];
        pos += w < warp ? sw : 0;
        na += sw;
    }
#pragma unroll
    for (int k = 0; k < KMAX; k++) {
        const int w = K * tid + k;
        if (k < K && w < nw) {
            s_words[w] = wv[k];
            s_wpre[w] = pos;
            pos += __popc(wv[k]);
        }
    }
    __syncthreads();
    return na;
}

// record index of A's p-th element (p < |A|): the word holding it by binary search over the
// prefix, then the bit by __fns
__device__ __forceinline__ int tile_huge_select(int p, const uint32_t *s_words, const int32_t *s_wpre, int nw) {
    int lo = 0, hi = nw - 1;  // largest w with s_wpre[w] <= p
    while (lo < hi) {
        const int m = (lo + hi + 1) >> 1;
        if (s_wpre[m] <= p) lo = m;
        else hi = m - 1;
    }
    return 32 * lo + (int)__fns(s_words[lo], 0, p - s_wpre[lo] + 1);
}

// ---------------------------------------------------------------------------------------------
// bucket sort (bitonic in shared memory; oversized buckets: sorted runs merged in global memory)
constexpr int SM_CAP = 4096;  // bucket keys sorted in shared memory at once

template <int NT>
__device__ __forceinline__ void bitonic_smem(uint64_t *k, int np) {
    for (int s = 2; s <= np; s <<= 1)
        for (int j = s >> 1; j > 0; j >>= 1) {
            for (int i = threadIdx.x; i < np; i += NT) {
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

// Sorts src[0, nb) in place (tmp: nb scratch keys); skey: SM_CAP shared keys.  Returns a pointer
// to the sorted keys: skey when nb <= SM_CAP (src is then also written back if writeback),
// else src.
template <int NT>
__device__ const uint64_t *sort_bucket(uint64_t *skey, uint64_t *src, uint64_t *tmp, int nb, bool writeback) {
    if (nb <= SM_CAP) {
        int np = 1;
        while (np < nb) np <<= 1;
        for (int i = threadIdx.x; i < np; i += NT) skey[i] = i < nb ? src[i] : ~0ull;
        __syncthreads();
        bitonic_smem<NT>(skey, np);
        if (writeback)
            for (int i = threadIdx.x; i < nb; i += NT) src[i] = skey[i];
        return skey;
    }
    for (int c0 = 0; c0 < nb; c0 += SM_CAP) {
        const int m = min(SM_CAP, nb - c0);
        int np = 1;
        while (np < m) np <<= 1;
        for (int i = threadIdx.x; i < np; i += NT) skey[i] = i < m ? src[c0 + i] : ~0ull;
        __syncthreads();
        bitonic_smem<NT>(skey, np);
        for (int i = threadIdx.x; i < m; i += NT) src[c0 + i] = skey[i];
        __syncthreads();
    }
    uint64_t *cur = src, *other = tmp;
    for (int w = SM_CAP; w < nb; w <<= 1) {
        for (int i = threadIdx.x; i < nb; i += NT) {
            const int lo = (i / (2 * w)) * (2 * w), mid = min(lo + w, nb), hi = min(lo + 2 * w, nb);
            const uint64_t v = cur[i];
            const bool in_a = i < mid;
            int a = in_a ? mid : lo, b = in_a ? hi : mid;  // rank in the other run
            while (a < b) {
                const int m = (a + b) >> 1;
                if (cur[m] < v) a = m + 1;
                else b = m;
            }
            other[lo + (i - (in_a ? lo : mid)) + (a - (in_a ? mid : lo))] = v;
        }
        __syncthreads();
        uint64_t *tt = cur;
        cur = other;
        other = tt;
    }
    if (cur != src) {  // the sorted keys end in src
        for (int i = threadIdx.x; i < nb; i += NT) src[i] = cur[i];
        __syncthreads();
    }
    return src;
}

// ---------------------------------------------------------------------------------------------
// Merged list of a tile into out[0, na + nb): A = s_a[0, na) (record indices, ascending), B =
// sorted keys.  Scratch: isb / wpre >= (na + nb) / 32 + 1 words each, s_tmp >= warps ints.
template <int NT>
__device__ void merge_tile_list(const gs_frame &f, int32_t *out, const int32_t *s_a, int na, const uint64_t *B,
                                int nb, uint32_t *isb, int32_t *wpre, int32_t *s_tmp, int cap_bits) {
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int nrec = min(f.counters[GS_CNT_HUGE_N], GS_HUGE_CAP);
    const uint64_t *hkeys = huge_keys(f);
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
    if (na == 0) {
        for (int j = tid; j < nb; j += NT) out[j] = (int32_t)(uint32_t)B[j];
        return;
    }
    if (nb == 0 || hkeys[s_a[na - 1]] < B[0]) {  // concatenation
        const int32_t *hid2 = hid;
        for (int d = tid; d < total; d += NT) out[d] = d < na ? hid2[s_a[d]] : (int32_t)(uint32_t)B[d - na];
        return;
    }
    if (total <= cap_bits) {
        // B_j lands at j + #{A preceding it}; its slot is marked in a bitmap.  Every other output
        // d is A element d - #{B slots before d}.  Both write passes are coalesced.
        const int tw = (total + 31) >> 5;
        for (int w = tid; w < tw; w += NT) isb[w] = 0u;
        __syncthreads();
        for (int j = tid; j < nb; j += NT) {
            const int h = huge_before(B[j]);
            int lo = 0, hi = na;
            while (lo < hi) {
                const int m = (lo + hi) >> 1;
                if (s_a[m] < h) lo = m + 1;
                else hi = m;
            }
            const int d = j + lo;
            out[d] = (int32_t)(uint32_t)B[j];
            atomicOr(&isb[d >> 5], 1u << (d & 31));
        }
        __syncthreads();
        for (int w0 = 0; w0 < tw; w0 += NT) {  // exclusive prefix of the B-slot popcounts
            const int w = w0 + tid;
            const int cnt = w < tw ? __popc(isb[w]) : 0;
            int xx = cnt;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, xx, o);
                if (lane >= o) xx += y;
            }
            if (lane == 31) s_tmp[warp] = xx;
            __syncthreads();
            int pre = xx - cnt + (w0 > 0 ? wpre[w0 - 1] + __popc(isb[w0 - 1]) : 0);
            for (int ww = 0; ww < warp; ww++) pre += s_tmp[ww];
            if (w < tw) wpre[w] = pre;
            __syncthreads();
        }
        for (int d = tid; d < total; d += NT) {
            const uint32_t word = isb[d >> 5];
            if ((word >> (d & 31)) & 1u) continue;
            const int a = d - (wpre[d >> 5] + __popc(word & ((1u << (d & 31)) - 1u)));
            out[d] = hid[s_a[a]];
        }
        return;
    }
    // large lists: merge path, each thread merges a run of ceil(total / NT) outputs
    const int L = (total + NT - 1) / NT;
    const int d0 = min(tid * L, total), d1 = min(d0 + L, total);
    if (d0 >= d1) return;
    int lo = max(0, d0 - nb), hi = min(d0, na);
    while (lo < hi) {  // a = number of A among the first d0 outputs
        const int m = (lo + hi) >> 1;
        if (s_a[m] < huge_before(B[d0 - 1 - m])) lo = m + 1;
        else hi = m;
    }
    int aa = lo, bb = d0 - lo;
    int hb = bb < nb ? huge_before(B[bb]) : 0;
    for (int d = d0; d < d1; d++) {
        if (bb >= nb || (aa < na && s_a[aa] < hb)) {
            out[d] = hid[s_a[aa]];
            aa++;
        } else {
            out[d] = (int32_t)(uint32_t)B[bb];
            bb++;
            if (bb < nb) hb = huge_before(B[bb]);
        }
    }
}

// A expanded into s_a (record indices, ascending) from the setup words; collective
__device__ __forceinline__ void tile_huge_expand(const uint32_t *s_words, const int32_t *s_wpre, int nw, int32_t *s_a) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int w = warp; w < nw; w += nwarps) {
        const uint32_t word = s_words[w];
        if ((word >> lane) & 1u) s_a[s_wpre[w] + __popc(word & ((1u << lane) - 1u))] = 32 * w + lane;
    }
    __syncthreads();
}

}  // namespace gs
