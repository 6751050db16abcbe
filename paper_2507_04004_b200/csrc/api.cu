#include <algorithm>
// api.cu -- workspace layout, camera setup and error reporting of the C ABI (include/gslic.h).
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <mutex>

#include "common.cuh"

namespace gs {

static thread_local char g_err[512] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof g_err, fmt, ap);
    va_end(ap);
}

int check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        set_error("%s: %s", what, cudaGetErrorString(e));
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

int64_t loss_parts_needed(int32_t width, int32_t height);  // loss.cu
void init_loss_attrs();                                     // loss.cu
void init_chain_attrs();                                    // adam.cu
void init_binning_attrs();                                  // binning.cu
void init_render_attrs();                                   // render.cu
void init_preprocess_attrs();                               // preprocess.cu

// kernel attributes (dynamic shared-memory opt-in) are set once per process, outside any
// stream capture, the first time a workspace is laid out
static void init_attrs_once() {
    static std::once_flag flag;
    std::call_once(flag, [] {
        init_loss_attrs();
        init_chain_attrs();
        init_binning_attrs();
        init_render_attrs();
        init_preprocess_attrs();
    });
}

struct Carver {
    size_t off = 0;
    unsigned char *base = nullptr;
    template <class T>
    T *take(size_t count) {
        off = (off + 255) & ~(size_t)255;
        T *p = base ? reinterpret_cast<T *>(base + off) : nullptr;
        off += sizeof(T) * count;
        return p;
    }
};

static void carve(Carver &c, int64_t n, int32_t w, int32_t h, int64_t cap, gs_frame &f) {
    const int64_t nn = n > 0 ? n : 1;
    const int32_t tx = (w + GS_TILE - 1) / GS_TILE, ty = (h + GS_TILE - 1) / GS_TILE;
    const int64_t P = (int64_t)w * h;
    f.n = n;
    f.entry_capacity = cap;
    f.width = w;
    f.height = h;
    f.tiles_x = tx;
    f.tiles_y = ty;
    f.splat2d = c.take<float>((int64_t)GS_SPLAT * nn);
    f.cov2d = c.take<float>(4 * nn);
    f.rect = c.take<int32_t>(8 * nn);  // BinRec (common.cuh): rect, keep bits, kept
    f.valid = c.take<uint8_t>(nn);
    f.touched = c.take<uint8_t>(nn);
    f.touched_list = c.take<int32_t>(nn);
    f.g2d = c.take<int64_t>((int64_t)GS_G2D * nn);
    f.grad_rows = c.take<float>((int64_t)GS_ROW * nn);
    f.bias_corr = c.take<float>(2 * nn);
    f.keep_bits = nullptr;  // in the BinRec records
    f.kept = nullptr;
    f.big_list = c.take<int32_t>(nn);
    f.big_slot = c.take<int32_t>(nn);
    f.cull_queue_cap = nn > (1 << 20) ? nn : (1 << 20);
    f.cull_queue = c.take<int32_t>(2 * f.cull_queue_cap);
    // huge records (8 ints each), their ids and 64-bit keys in depth order, then the unsorted
    // staged keys
    f.huge = c.take<int32_t>(13 * GS_HUGE_CAP);
    f.huge_mask = c.take<uint32_t>(((int64_t)tx * ty) * (GS_HUGE_CAP / 32));
    f.huge_mask_t = c.take<uint32_t>((int64_t)GS_HUGE_CAP * (((int64_t)tx * ty + 31) / 32));
    f.tile_scratch = c.take<int32_t>(6 * ((int64_t)tx * ty + 1));  // segments: tilelist.cuh
    f.tile_minkey = c.take<uint64_t>((int64_t)tx * ty + 1);
    f.big_bits_words = 4 * nn > (1 << 20) ? 4 * nn : (1 << 20);
    f.big_bits = c.take<uint32_t>(f.big_bits_words);
    f.keys_a = c.take<uint64_t>(cap > 0 ? cap : 1);
    f.keys_b = c.take<uint64_t>(cap > 0 ? cap : 1);
    f.entry_splat = c.take<int32_t>(cap > 0 ? cap : 1);
    f.tile_offsets = c.take<int32_t>((int64_t)tx * ty + 1);
    f.counters = c.take<int32_t>(GS_CNT_SLOTS * 2);
    f.color = c.take<float>(3 * P);
    f.depth = c.take<float>(P);
    f.opacity = c.take<float>(P);
    f.trans = c.take<float>(P);
    f.n_contrib = c.take<int32_t>(P);
    f.g_color = c.take<float>(3 * P);
    f.g_depth = c.take<float>(P);
    f.g_opac = c.take<float>(P);
    f.loss_blocks = loss_parts_needed(w, h);
    // loss partials (3 doubles per block) followed by the two 11-tap reflection tables
    f.loss_parts = c.take<double>(3 * f.loss_blocks + (int64_t)11 * (w + h) + 1);
    // total, photometric, depth, dssim, running sum, -, ring position, -, then the per-iteration
    // loss ring (GS_LOSS_ACCUMULATE)
    f.loss = c.take<double>(8 + 5 * GS_LOSS_RING);  // + the counter snapshot ring (gslic.h)
    f.pose_acc = c.take<int64_t>(16);
    f.ssim_g = c.take<float>(12 * P);
}

}  // namespace gs

using namespace gs;

extern "C" size_t gs_workspace_size(int64_t n, int32_t width, int32_t height, int64_t entry_capacity) {
    Carver c;
    gs_frame f;
    carve(c, n, width, height, entry_capacity, f);
    return (c.off + 255) & ~(size_t)255;
}

extern "C" int gs_frame_layout(int64_t n, int32_t width, int32_t height, int64_t entry_capacity, void *ws,
                               size_t ws_bytes, gs_frame *out) {
    if (!out || n < 0 || width <= 0 || height <= 0 || entry_capacity < 0) {
        set_error("gs_frame_layout: bad dimensions (n=%lld, %dx%d, cap=%lld)", (long long)n, width, height,
                  (long long)entry_capacity);
        return GS_ERR_DIMS;
    }
    if (n >= (1ll << 31) || entry_capacity >= (1ll << 30)) {
        set_error("gs_frame_layout: n or entry_capacity exceeds the 32-bit index range");
        return GS_ERR_DIMS;
    }
    if ((int64_t)((width + GS_TILE - 1) / GS_TILE) * ((height + GS_TILE - 1) / GS_TILE) > GS_MAX_TILES) {
        set_error("gs_frame_layout: %dx%d exceeds GS_MAX_TILES (%d) tiles", width, height, GS_MAX_TILES);
        return GS_ERR_DIMS;
    }
    const size_t need = gs_workspace_size(n, width, height, entry_capacity);
    if (!ws || ws_bytes < need || ((uintptr_t)ws & 255u)) {
        set_error("gs_frame_layout: workspace too small or misaligned (%zu < %zu)", ws_bytes, need);
        return GS_ERR_WORKSPACE;
    }
    init_attrs_once();
    Carver c;
    c.base = static_cast<unsigned char *>(ws);
    memset(out, 0, sizeof *out);
    carve(c, n, width, height, entry_capacity, *out);
    return GS_OK;
}

extern "C" void gs_camera_init(gs_camera *cam) {
    const float *R = cam->rot_cw, *t = cam->trans_cw;
    for (int c = 0; c < 3; c++) cam->center[c] = -(R[c] * t[0] + R[3 + c] * t[1] + R[6 + c] * t[2]);
}

extern "C" const char *gs_last_error(void) { return g_err; }

extern "C" int gs_version(void) { return 1; }
