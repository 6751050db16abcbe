// p2p.cu -- the multi-GPU batch step's gradient allreduce fused with the sparse Adam update,
// over peer memory (R/rasterizer.py:707-725 for the update).
//
// Every rank of a keyframe batch has accumulated its views' parameter-gradient rows (grads, n x
// GS_ROW, by Gaussian id) and all ranks hold the same union of touched ids (idx[0..u), id
// order).  One persistent kernel per rank replaces "NCCL allreduce, then Adam":
//   prologue  rank r publishes gready[r] = epoch (its grads are complete: stream order);
//   phase A   reduce-scatter: rank r owns union rows [u r / N, u (r+1) / N); once every peer's
//             gready has reached the epoch it sums those rows over the ranks' grads, read
//             straight from peer memory, in rank order (the same bits on every rank), into its
//             packed buffer, then publishes rdone[r] = epoch (the last CTA to finish, after a
//             system-scope fence);
//   phase B   all-gather fused with Adam: for each shard s, once rdone[s] has reached the epoch,
//             every rank reads the reduced rows of shard s from rank s's packed buffer and
//             applies the update to its own replica (params, m, v, t), clearing its gradient row
//             and touched flag.  The replicas stay bitwise identical.
// Wire bytes per rank: 2 (N-1)/N x 240 B x u, as a ring allreduce, with no staging copy and no
// separate Adam pass.  Ordering across steps needs no extra barrier: a rank reads a peer's grads
// (phase A, step e) only after that peer's prologue of step e, and clears its own rows (phase B)
// only after every rank's rdone of step e, i.e. after all reads of them.
// The grid is persistent and fully resident (phase B waits on this rank's own phase A).  Waits
// are bounded: a peer that never arrives sets *err and the kernel finishes (wrong but no hang).
#include <cuda.h>

#include <algorithm>
#include <cstring>

#include "common.cuh"

namespace gs {

constexpr int P2P_MAX = 8;
constexpr int P2P_THREADS = 256;

struct P2PArgs {
    const float *grads[P2P_MAX];               // each rank's gradient rows (n x GS_ROW)
    const float *packed[P2P_MAX];              // each rank's reduced shard rows (union order x 60)
    unsigned long long *gready[P2P_MAX];       // each rank's "grads of this epoch complete"
    unsigned long long *rdone[P2P_MAX];        // each rank's "shard of this epoch reduced"
};

__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long *p) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_sys(unsigned long long *p, unsigned long long v) {
    asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// thread 0 waits for *flag >= epoch (bounded), then the CTA proceeds
__device__ __forceinline__ void cta_wait_flag(const unsigned long long *flag, unsigned long long epoch, int *err) {
    if (threadIdx.x == 0) {
        unsigned polls = 0;
        while (ld_acquire_sys(flag) < epoch) {
            if (++polls > (1u << 24)) {  // ~seconds: a peer is gone
                atomicExch(err, 1);
                break;
            }
            __nanosleep(128);
        }
    }
    __syncthreads();
}

__global__ void __launch_bounds__(P2P_THREADS) p2p_reduce_adam_kernel(
    P2PArgs a, int rank, int world, unsigned long long epoch, int64_t u, const int32_t *__restrict__ idx,
    float *__restrict__ params, float *__restrict__ am, float *__restrict__ av, int32_t *__restrict__ at,
    const float *__restrict__ lr_cols, float *__restrict__ grads, uint8_t *__restrict__ touched,
    unsigned *__restrict__ ticket, float *__restrict__ keep, int *__restrict__ err) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {  // this rank's grads are complete (stream order)
        __threadfence_system();
        st_release_sys(a.gready[rank], epoch);
    }
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, gstride = (int64_t)gridDim.x * blockDim.x;
    // phase A: this rank's shard, summed over the ranks in rank order
    for (int k = 0; k < world; k++) cta_wait_flag(a.gready[k], epoch, err);
    {
        const int64_t lo = u * rank / world, hi = u * (rank + 1) / world;
        float4 *out = reinterpret_cast<float4 *>(const_cast<float *>(a.packed[rank]));
        for (int64_t q = lo * 15 + gtid; q < hi * 15; q += gstride) {
            const int64_t i = q / 15;
            const int c4 = (int)(q - i * 15);
            const int64_t off = (int64_t)idx[i] * (GS_ROW / 4) + c4;
            float4 s = __ldcg(reinterpret_cast<const float4 *>(a.grads[0]) + off);
            for (int k = 1; k < world; k++) {
                const float4 g = __ldcg(reinterpret_cast<const float4 *>(a.grads[k]) + off);
                s.x += g.x;
                s.y += g.y;
                s.z += g.z;
                s.w += g.w;
            }
            out[q] = s;
        }
    }
    __threadfence_system();
    __syncthreads();
    if (threadIdx.x == 0) {
        if (atomicAdd(ticket, 1u) == gridDim.x - 1) {  // the last CTA: the shard is reduced
            *ticket = 0u;
            __threadfence_system();
            st_release_sys(a.rdone[rank], epoch);
        }
    }
    // phase B: every shard, from its owner's packed rows, into this replica (as adam_packed_kernel)
    for (int j = 0; j < world; j++) {
        const int s = (rank + 1 + j) % world;  // the own shard last: peers' are usually ready first
        cta_wait_flag(a.rdone[s], epoch, err);
        const int64_t lo = u * s / world, hi = u * (s + 1) / world;
        const float4 *src = reinterpret_cast<const float4 *>(a.packed[s]);
        for (int64_t q = lo * 16 + gtid; q < hi * 16; q += gstride) {
            const int64_t i = q >> 4;
            const int c4 = (int)(q & 15);
            const int64_t row = idx[i];
            const int tn = at[row] + 1;  // read by the row's 16 lanes before its lane 15 writes it
            __syncwarp(0xffffu << (threadIdx.x & 16u));
            const float bc1 = (float)(1.0 / (1.0 - pow(0.9, (double)tn))),
                        bc2 = (float)(1.0 / (1.0 - pow(0.999, (double)tn)));
            if (c4 == 15) {  // columns 60-63: padding; this lane bumps the step and clears the flag
                at[row] = tn;
                touched[row] = 0;
                continue;
            }
            const int64_t off = row * GS_ROW + 4 * c4;
            const float4 g4 = __ldcg(src + i * 15 + c4);
            if (keep) reinterpret_cast<float4 *>(keep)[i * 15 + c4] = g4;
            *reinterpret_cast<float4 *>(grads + off) = make_float4(0.f, 0.f, 0.f, 0.f);
            const float4 P = *reinterpret_cast<const float4 *>(params + off);
            float4 m4 = *reinterpret_cast<const float4 *>(am + off);
            float4 v4 = *reinterpret_cast<const float4 *>(av + off);
            const float4 lr = __ldg(reinterpret_cast<const float4 *>(lr_cols) + c4);
            float4 p4;
            p4.x = adam_one(P.x, m4.x, v4.x, g4.x, lr.x, bc1, bc2);
            p4.y = adam_one(P.y, m4.y, v4.y, g4.y, lr.y, bc1, bc2);
            p4.z = adam_one(P.z, m4.z, v4.z, g4.z, lr.z, bc1, bc2);
            p4.w = c4 == 14 ? P.w : adam_one(P.w, m4.w, v4.w, g4.w, lr.w, bc1, bc2);  // column 59: padding
            *reinterpret_cast<float4 *>(am + off) = m4;
            *reinterpret_cast<float4 *>(av + off) = v4;
            *reinterpret_cast<float4 *>(params + off) = p4;
        }
    }
}

}  // namespace gs

using namespace gs;

extern "C" int gs_ipc_export(const void *ptr, uint8_t *handle, int64_t *offset) {
    if (!ptr || !handle || !offset) {
        set_error("gs_ipc_export: null argument");
        return GS_ERR_ARG;
    }
    // the allocation's base (IPC handles name whole cudaMalloc allocations; torch's caching
    // allocator hands out pieces of them): the driver's cuMemGetAddressRange through the runtime's
    // entry-point table, so the library carries no link-time libcuda dependency
    using range_fn = CUresult (*)(CUdeviceptr *, size_t *, CUdeviceptr);
    static range_fn get_range = nullptr;
    if (!get_range) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess || !fn) {
            set_error("gs_ipc_export: cuMemGetAddressRange unavailable");
            return GS_ERR_CUDA;
        }
        get_range = reinterpret_cast<range_fn>(fn);
    }
    CUdeviceptr base = 0;
    size_t size = 0;
    if (get_range(&base, &size, (CUdeviceptr)ptr) != CUDA_SUCCESS) {
        set_error("gs_ipc_export: not a device allocation");
        return GS_ERR_ARG;
    }
    cudaIpcMemHandle_t h;
    const cudaError_t e = cudaIpcGetMemHandle(&h, reinterpret_cast<void *>(base));
    if (e != cudaSuccess) {
        set_error("gs_ipc_export: %s", cudaGetErrorString(e));
        return GS_ERR_CUDA;
    }
    memcpy(handle, &h, sizeof(h));
    *offset = (int64_t)((CUdeviceptr)ptr - base);
    return GS_OK;
}

extern "C" int gs_ipc_import(const uint8_t *handle, int64_t offset, void **ptr, void **base) {
    if (!handle || !ptr || !base || offset < 0) {
        set_error("gs_ipc_import: bad arguments");
        return GS_ERR_ARG;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    void *b = nullptr;
    const cudaError_t e = cudaIpcOpenMemHandle(&b, h, cudaIpcMemLazyEnablePeerAccess);
    if (e != cudaSuccess) {
        set_error("gs_ipc_import: %s", cudaGetErrorString(e));
        return GS_ERR_CUDA;
    }
    *base = b;
    *ptr = static_cast<char *>(b) + offset;
    return GS_OK;
}

extern "C" int gs_ipc_close(void *base) {
    const cudaError_t e = cudaIpcCloseMemHandle(base);
    if (e != cudaSuccess) {
        set_error("gs_ipc_close: %s", cudaGetErrorString(e));
        return GS_ERR_CUDA;
    }
    return GS_OK;
}

extern "C" int gs_p2p_reduce_adam(int32_t world, int32_t rank, const float *const *grads, const float *const *packed,
                                  uint64_t *const *gready, uint64_t *const *rdone, uint64_t epoch, int64_t u,
                                  const int32_t *idx, float *params, float *adam_m, float *adam_v, int32_t *adam_t,
                                  const float *lr_cols, float *my_grads, uint8_t *touched, uint32_t *ticket,
                                  float *keep, int32_t *err, void *stream) {
    if (world < 1 || world > P2P_MAX || rank < 0 || rank >= world || !grads || !packed || !gready || !rdone ||
        !idx || !params || !adam_m || !adam_v || !adam_t || !lr_cols || !my_grads || !touched || !ticket || !err ||
        u < 0 || epoch == 0) {
        set_error("gs_p2p_reduce_adam: bad arguments");
        return GS_ERR_ARG;
    }
    P2PArgs a = {};
    for (int k = 0; k < world; k++) {
        if (!grads[k] || !packed[k] || !gready[k] || !rdone[k]) {
            set_error("gs_p2p_reduce_adam: missing peer pointer %d", k);
            return GS_ERR_ARG;
        }
        a.grads[k] = grads[k];
        a.packed[k] = packed[k];
        a.gready[k] = reinterpret_cast<unsigned long long *>(gready[k]);
        a.rdone[k] = reinterpret_cast<unsigned long long *>(rdone[k]);
    }
    // persistent and fully resident: phase B waits on this grid's own phase A
    static const int per_sm = [] {  // (thread-safe static initialisation)
        int b = 0;
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, p2p_reduce_adam_kernel, P2P_THREADS, 0);
        return b < 1 ? 1 : b;
    }();
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned blocks = (unsigned)std::min(per_sm * sms, 4 * sms);
    // a plain launch (no programmatic overlap): every CTA of the grid must become resident
    p2p_reduce_adam_kernel<<<blocks, P2P_THREADS, 0, (cudaStream_t)stream>>>(
        a, rank, world, (unsigned long long)epoch, u, idx, params, adam_m, adam_v, adam_t, lr_cols, my_grads, touched,
        reinterpret_cast<unsigned *>(ticket), keep, reinterpret_cast<int *>(err));
    return check_launch("p2p_reduce_adam_kernel");
}
