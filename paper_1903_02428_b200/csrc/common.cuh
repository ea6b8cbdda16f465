// common.cuh -- shared device helpers for libpygs (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>

#include "pyg_gs.h"

namespace pyg {

// ---------------------------------------------------------------- host side
extern std::atomic<uint64_t> g_launches;
void set_error(const char* fmt, ...);
pyg_status_t fail(pyg_status_t st, const char* fmt, ...);
pyg_status_t cuda_check(cudaError_t e, const char* what);

#define PYG_LAUNCHED() ::pyg::g_launches.fetch_add(1, std::memory_order_relaxed)
#define PYG_CUDA(call)                                              \
    do {                                                            \
        cudaError_t _e = (call);                                    \
        if (_e != cudaSuccess) return ::pyg::cuda_check(_e, #call); \
    } while (0)
#define PYG_TRY(call)                         \
    do {                                      \
        pyg_status_t _s = (call);             \
        if (_s != PYG_OK) return _s;          \
    } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }
__host__ __device__ inline int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Carve aligned sub-buffers out of a caller workspace.
struct Carver {
    char* base;
    size_t cap, off = 0;
    Carver(void* b, size_t c) : base(static_cast<char*>(b)), cap(c) {}
    template <class T>
    T* take(size_t n) {
        off = align_up(off, 256);
        T* p = reinterpret_cast<T*>(base ? base + off : nullptr);
        off += n * sizeof(T);
        return p;
    }
    bool ok() const { return off <= cap; }
    // the uncarved tail (for a callee that carves its own buffers)
    void* rest() const { return base ? base + align_up(off, 256) : nullptr; }
    size_t rest_bytes() const { return cap > align_up(off, 256) ? cap - align_up(off, 256) : 0; }
};

// Tuning / test knobs from the environment, read ONCE per process (pyg_refresh_env re-reads them;
// tests flip PYG_SEG_TMA between cases).  Defaults are the measured best settings.
struct Knobs {
    int seg_tma = -1;     // PYG_SEG_TMA: -1 auto, 0 off, 1 whenever eligible
    int tma_hubs = 1;     // PYG_TMA_HUBS: 0 keeps split hub rows on the LDG kernel
    int tma_warp_kb = 4;  // PYG_TMA_WARP_KB: ring bytes per warp of the TMA gather4 kernel
    int tma_warps = 8;    // PYG_TMA_WARPS
    int seg_bulk = -1;    // PYG_SEG_BULK: row-staged bulk-copy kernel -- 1 on wherever eligible, else off
    int bulk_warp_kb = 8; // PYG_BULK_WARP_KB: ring bytes per warp of the bulk-copy kernel
    int gat_warp_kb = 10; // PYG_GAT_WARP_KB: ring bytes per warp of the one-pass GAT backward
    int gat_sm_kb = 160;  // PYG_GAT_SM_KB: its shared memory per SM (the rest stays L1)
    int gat_warps = 8;    // PYG_GAT_WARPS: warps per CTA of the GAT TMA kernels (8, 4 or 2)
    int gat_fused = 1;    // PYG_GAT_FUSED: 0 keeps the GAT forward on softmax + aggregation (two kernels)
    int gat_fwd_warp_kb = 5;   // PYG_GAT_FWD_WARP_KB: ring bytes per warp of the one-pass GAT forward
    int gat_fwd_sm_kb = 160;   // PYG_GAT_FWD_SM_KB
    int coo_tile = 1;     // PYG_COO_TILE: 0 keeps every atomic launch on the generic coo_kernel
    int coo_compact = 1;  // PYG_COO_COMPACT: L2 column tiles through packed scratch -- 1 auto (large spans), 2 always, 0 never
    int coo_chunk = 128;  // PYG_COO_CHUNK: edges per warp of the tile kernel
    int coo_l2_mb = 72;   // PYG_COO_L2_MB: L2 budget of the atomic path's column tiles (0: no tiling)
    int coo_l2_mb_max = 96;  // PYG_COO_L2_MB_MAX: the same for MAX (keys mostly read, not written)
};
const Knobs& knobs();

// Device-side validation flag (pinned, mapped) -- PYG_VALIDATE paths.
int* validate_flag_dev();
void validate_begin();  // clear this thread's flag before launching checking kernels
pyg_status_t validate_flag_check(cudaStream_t s, const char* what);
pyg_status_t validate_index(const int64_t* idx, int64_t n, int64_t lo, int64_t hi,
                            cudaStream_t s);

// ---------------------------------------------------------------- device side
template <int V>
struct VecT;
template <>
struct VecT<1> { using T = float; };
template <>
struct VecT<2> { using T = float2; };
template <>
struct VecT<4> { using T = float4; };

template <int V>
__device__ __forceinline__ void ldv(float (&r)[V], const float* p) {
    if constexpr (V == 4) {
        float4 t = __ldg(reinterpret_cast<const float4*>(p));
        r[0] = t.x; r[1] = t.y; r[2] = t.z; r[3] = t.w;
    } else if constexpr (V == 2) {
        float2 t = __ldg(reinterpret_cast<const float2*>(p));
        r[0] = t.x; r[1] = t.y;
    } else {
        r[0] = __ldg(p);
    }
}

// store `n` (<= V) leading floats of r at p (vector store when n == V)
template <int V>
__device__ __forceinline__ void stv(float* p, const float (&r)[V], int n) {
    if (n == V) {
        if constexpr (V == 4) {
            *reinterpret_cast<float4*>(p) = make_float4(r[0], r[1], r[2], r[3]);
        } else if constexpr (V == 2) {
            *reinterpret_cast<float2*>(p) = make_float2(r[0], r[1]);
        } else {
            p[0] = r[0];
        }
    } else {
#pragma unroll
        for (int t = 0; t < V; ++t)
            if (t < n) p[t] = r[t];
    }
}

// vector atomic add (RED, no return) of n (<= V) floats
template <int V>
__device__ __forceinline__ void redv(float* p, const float (&r)[V], int n) {
    if (n == V) {
        if constexpr (V == 4) {
            atomicAdd(reinterpret_cast<float4*>(p), make_float4(r[0], r[1], r[2], r[3]));
        } else if constexpr (V == 2) {
            atomicAdd(reinterpret_cast<float2*>(p), make_float2(r[0], r[1]));
        } else {
            atomicAdd(p, r[0]);
        }
    } else {
#pragma unroll
        for (int t = 0; t < V; ++t)
            if (t < n) atomicAdd(p + t, r[t]);
    }
}

// Order-preserving map float -> uint32 (after -0 -> +0) and the packed
// 64-bit max key (value high, inverted edge id low => ties -> lowest id).
__device__ __forceinline__ uint32_t f2ord(float v) {
    uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);
    return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
    uint32_t u = (o & 0x80000000u) ? (o & 0x7fffffffu) : ~o;
    return __uint_as_float(u);
}
__device__ __forceinline__ unsigned long long max_key(float v, uint32_t k) {
    return (static_cast<unsigned long long>(f2ord(v)) << 32) |
           static_cast<unsigned long long>(0xffffffffu - k);
}

}  // namespace pyg
