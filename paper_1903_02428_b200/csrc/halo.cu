// halo.cu -- the sparse source exchange of the dst-range partition (north_star (3): "for sparse
// cross-partition edges, by a halo exchange of only the referenced rows").
//
// Rank p owns targets [own_lo, own_hi) (a slice of the global plan) and the X rows of the same
// range.  Its in-edges reference some source rows owned by other ranks: the halo.  At plan time
// (once per graph, "pre-processing"):
//   1. mark every source referenced by the slice's positions;
//   2. the halo = marked sources outside [own_lo, own_hi), in ascending global id (hence grouped
//      by owner rank, the order an all-to-all delivers them in);
//   3. map: own source j -> j - own_lo, halo source halo_ids[h] -> own_rows + h;
//   4. a copy of the slice whose `col` holds the mapped ids, so the unchanged segment kernels
//      gather from the rank-local buffer X_loc = [own shard (own_rows rows) ; halo rows].
// Per call, the owner packs the rows each peer asked for (pyg_gather_rows) and one NCCL
// all-to-all delivers them into X_loc's halo block; the propagate then runs on X_loc.
#include <cub/cub.cuh>

#include "kernels.cuh"

namespace pyg {

namespace {

int grid_for(int64_t work, int threads = 256) {
    int64_t b = cdiv(work, threads);
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

#define GRID_STRIDE(t, total) \
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (total); t += (int64_t)gridDim.x * blockDim.x)

__global__ void mark_kernel(const int32_t* __restrict__ col, int64_t plo, int64_t n, int32_t* mark) {
    GRID_STRIDE(t, n) mark[col[plo + t]] = 1;  // benign race: every writer stores 1
}

__global__ void halo_flag_kernel(int32_t* mark, int64_t n_src, int64_t own_lo, int64_t own_hi) {
    GRID_STRIDE(j, n_src) if (j >= own_lo && j < own_hi) mark[j] = 0;
}

__global__ void halo_map_kernel(const int32_t* __restrict__ flag, const int32_t* __restrict__ hpos, int64_t n_src,
                                int64_t own_lo, int64_t own_hi, int64_t own_rows, int32_t* map, int64_t* halo_ids) {
    GRID_STRIDE(j, n_src) {
        int32_t m = -1;
        if (j >= own_lo && j < own_hi) {
            m = (int32_t)(j - own_lo);
        } else if (flag[j]) {
            m = (int32_t)(own_rows + hpos[j]);
            halo_ids[hpos[j]] = j;
        }
        map[j] = m;
    }
}

__global__ void remap_kernel(const int32_t* __restrict__ col, const int32_t* __restrict__ map, int64_t plo, int64_t n,
                             int32_t* col2) {
    GRID_STRIDE(t, n) col2[t] = map[col[plo + t]];
}

// out[r] = x[rows[r]]: one warp per row, 16-byte vectors when rows and strides allow
template <int V>
__global__ void gather_rows_kernel(const float* __restrict__ x, int64_t ldx, int F, const int64_t* __restrict__ rows,
                                   int64_t n, float* __restrict__ out, int64_t ldo) {
    const int lane = threadIdx.x & 31;
    const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = w0; r < n; r += nw) {
        const float* src = x + rows[r] * ldx;
        float* dst = out + r * ldo;
        if constexpr (V == 4) {
            const int nv = F >> 2;
            for (int c = lane; c < nv; c += 32)
                reinterpret_cast<float4*>(dst)[c] = __ldg(reinterpret_cast<const float4*>(src) + c);
            for (int c = 4 * nv + lane; c < F; c += 32) dst[c] = __ldg(src + c);
        } else {
            for (int c = lane; c < F; c += 32) dst[c] = __ldg(src + c);
        }
    }
}

struct HaloLayout {
    int32_t *mark, *hpos, *map, *col2;
    void* cub_tmp;
    size_t cub_bytes;
};

size_t halo_layout(void* ws, size_t bytes, int64_t n_src, int64_t e_slice, HaloLayout& L) {
    Carver cv(ws, bytes);
    const size_t n = (size_t)std::max<int64_t>(n_src, 1);
    L.col2 = cv.take<int32_t>((size_t)std::max<int64_t>(e_slice, 1));  // kept: the halo plan's col
    L.mark = cv.take<int32_t>(n);
    L.hpos = cv.take<int32_t>(n);
    L.map = cv.take<int32_t>(n);
    L.cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, L.cub_bytes, L.mark, L.hpos, (int)n);
    L.cub_tmp = cv.take<char>(L.cub_bytes);
    return cv.off;
}

pyg_status_t slice_positions(const pyg_plan* p, int64_t* plo, int64_t* phi) {
    int64_t v[2] = {0, 0};
    if (p->n_rows > 0) {
        PYG_CUDA(cudaMemcpy(&v[0], p->rowptr, 8, cudaMemcpyDeviceToHost));
        PYG_CUDA(cudaMemcpy(&v[1], p->rowptr + p->n_rows, 8, cudaMemcpyDeviceToHost));
    }
    *plo = v[0];
    *phi = v[1];
    return PYG_OK;
}

}  // namespace

pyg_status_t halo_workspace_impl(const pyg_plan* p, int64_t n_src, size_t* bytes) {
    int64_t plo = 0, phi = 0;
    PYG_TRY(slice_positions(p, &plo, &phi));
    HaloLayout L;
    *bytes = halo_layout(nullptr, 0, n_src, phi - plo, L) + 256;
    return PYG_OK;
}

pyg_status_t halo_build_impl(const pyg_plan* p, int64_t n_src, int64_t own_lo, int64_t own_hi, int64_t own_rows,
                             void* ws, size_t bytes, pyg_plan** out, int64_t* halo_ids, int64_t* n_halo,
                             cudaStream_t s) {
    int64_t plo = 0, phi = 0;
    PYG_TRY(slice_positions(p, &plo, &phi));
    const int64_t e = phi - plo;
    HaloLayout L;
    const size_t need = halo_layout(ws, bytes, n_src, e, L);
    if (!ws || need > bytes) return fail(PYG_ERR_NO_MEMORY, "halo workspace too small (%zu < %zu)", bytes, need);
    int64_t nh = 0;
    if (n_src > 0) {
        PYG_CUDA(cudaMemsetAsync(L.mark, 0, (size_t)n_src * 4, s));
        if (e > 0) {
            mark_kernel<<<grid_for(e), 256, 0, s>>>(p->col, plo, e, L.mark);
            PYG_LAUNCHED();
            PYG_CUDA(cudaGetLastError());
        }
        halo_flag_kernel<<<grid_for(n_src), 256, 0, s>>>(L.mark, n_src, own_lo, own_hi);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
        size_t cb = L.cub_bytes;
        PYG_CUDA(cub::DeviceScan::ExclusiveSum(L.cub_tmp, cb, L.mark, L.hpos, (int)n_src, s));
        PYG_LAUNCHED();
        int32_t last[2] = {0, 0};
        PYG_CUDA(cudaMemcpyAsync(&last[0], L.hpos + n_src - 1, 4, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaMemcpyAsync(&last[1], L.mark + n_src - 1, 4, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        nh = (int64_t)last[0] + last[1];
        if (own_rows + nh > 0x7ffffffeLL) return fail(PYG_ERR_UNSUPPORTED, "halo: own_rows + n_halo must be < 2^31");
        halo_map_kernel<<<grid_for(n_src), 256, 0, s>>>(L.mark, L.hpos, n_src, own_lo, own_hi, own_rows, L.map,
                                                         halo_ids);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
        if (e > 0) {
            remap_kernel<<<grid_for(e), 256, 0, s>>>(p->col, L.map, plo, e, L.col2);
            PYG_LAUNCHED();
            PYG_CUDA(cudaGetLastError());
        }
    }
    PYG_CUDA(cudaStreamSynchronize(s));
    pyg_plan* q = new pyg_plan(*p);
    q->col = L.col2 - plo;  // indexed by absolute sorted position, like the parent's arrays
    q->n_cols = own_rows + nh;
    *n_halo = nh;
    *out = q;
    return PYG_OK;
}

pyg_status_t gather_rows_impl(const float* x, int64_t ldx, int64_t F, const int64_t* rows, int64_t n, float* out,
                              int64_t ldo, cudaStream_t s) {
    if (n <= 0 || F <= 0) return PYG_OK;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 148 * 16));
    const bool v4 = (ldx % 4 == 0) && (ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
                    ((reinterpret_cast<uintptr_t>(out) & 15) == 0);
    if (v4) gather_rows_kernel<4><<<blocks, 256, 0, s>>>(x, ldx, (int)F, rows, n, out, ldo);
    else gather_rows_kernel<1><<<blocks, 256, 0, s>>>(x, ldx, (int)F, rows, n, out, ldo);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg

// ---- halo push over peer memory (NVLink P2P stores) ------------------------------------------
// The owner writes the rows each peer asked for straight into the peer's X_loc halo block through
// a CUDA-IPC mapping of that buffer: the gather of the rows and their transfer are one kernel, with
// no staging buffer and no NCCL call (the peer-store alternative to pack + all-to-all).
namespace pyg {

namespace {

constexpr int kMaxPeers = 16;

struct PushArgs {
    const float* x;
    int64_t ldx;
    int F;
    const int64_t* rows;      // local row ids, grouped by destination peer
    int n_peers;
    int64_t ptr[kMaxPeers + 1];   // rows[ptr[q] .. ptr[q+1]) go to peer q
    float* dst[kMaxPeers];        // peer q's X_loc (mapped)
    int64_t dst_row[kMaxPeers];   // first halo row of this owner's block at peer q
    int64_t ldd;
    int vec;
};

__global__ void halo_push_kernel(PushArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t total = a.ptr[a.n_peers];
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < total; i += nw) {
        int q = 0;
        while (q + 1 < a.n_peers && i >= a.ptr[q + 1]) ++q;  // <= 16 peers
        const float* src = a.x + a.rows[i] * a.ldx;
        float* d = a.dst[q] + (a.dst_row[q] + (i - a.ptr[q])) * a.ldd;
        if (a.vec) {
            const int nv = a.F >> 2;
            for (int c = lane; c < nv; c += 32)
                reinterpret_cast<float4*>(d)[c] = __ldg(reinterpret_cast<const float4*>(src) + c);
            for (int c = 4 * nv + lane; c < a.F; c += 32) d[c] = __ldg(src + c);
        } else {
            for (int c = lane; c < a.F; c += 32) d[c] = __ldg(src + c);
        }
    }
}

}  // namespace

pyg_status_t halo_push_impl(const float* x, int64_t ldx, int64_t F, const int64_t* rows, const int64_t* ptr,
                            void* const* dst, const int64_t* dst_row, int64_t ldd, int n_peers, cudaStream_t s) {
    if (n_peers > kMaxPeers) return fail(PYG_ERR_UNSUPPORTED, "halo_push: at most %d peers", kMaxPeers);
    PushArgs a;
    a.x = x; a.ldx = ldx; a.F = (int)F; a.rows = rows; a.n_peers = n_peers; a.ldd = ldd;
    bool aligned = (ldx % 4 == 0) && (ldd % 4 == 0) && !(reinterpret_cast<uintptr_t>(x) & 15);
    for (int q = 0; q <= n_peers; ++q) a.ptr[q] = ptr[q];
    for (int q = 0; q < n_peers; ++q) {
        a.dst[q] = static_cast<float*>(dst[q]);
        a.dst_row[q] = dst_row[q];
        if (reinterpret_cast<uintptr_t>(dst[q]) & 15) aligned = false;
    }
    a.vec = aligned;
    const int64_t total = ptr[n_peers];
    if (total <= 0 || F <= 0) return PYG_OK;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 8), 148 * 16));
    halo_push_kernel<<<blocks, 256, 0, s>>>(a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

namespace {
struct FlagArgs {
    uint32_t* f[kMaxPeers];
    int n;
    uint32_t value;
};
// every earlier write of this stream (the push kernel's peer stores) is made visible system-wide,
// then each flag (a peer's, mapped over NVLink, or local) is released with `value`
__global__ void peer_signal_kernel(FlagArgs a) {
    const int i = threadIdx.x;
    if (i >= a.n) return;
    __threadfence_system();
    asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(a.f[i]), "r"(a.value) : "memory");
}
// spin (with backoff) until every flag reaches `value` (wrap-safe comparison), acquire semantics
__global__ void peer_wait_kernel(FlagArgs a) {
    const int i = threadIdx.x;
    if (i < a.n) {
        uint32_t v = 0;
        unsigned ns = 32;
        for (;;) {
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(a.f[i]) : "memory");
            if ((int32_t)(v - a.value) >= 0) break;
            __nanosleep(ns);
            if (ns < 4096) ns <<= 1;
        }
    }
    __syncwarp();
}
}  // namespace

pyg_status_t peer_flags_impl(uint32_t* const* flags, int n, uint32_t value, int wait, cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    if (n > kMaxPeers) return fail(PYG_ERR_UNSUPPORTED, "peer flags: at most %d", kMaxPeers);
    FlagArgs a;
    for (int i = 0; i < n; ++i) a.f[i] = flags[i];
    a.n = n;
    a.value = value;
    if (wait) peer_wait_kernel<<<1, 32, 0, s>>>(a);
    else peer_signal_kernel<<<1, 32, 0, s>>>(a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg

// ---- CUDA IPC for the peer-store halo ---------------------------------------------------------
#include <cuda.h>

#include <cstring>
#include <map>
#include <mutex>
#include <string>

namespace pyg {

namespace {
typedef CUresult (*AddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
AddrRangeFn addr_range_fn() {
    static AddrRangeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<AddrRangeFn>(p);
    });
    return fn;
}
}  // namespace

pyg_status_t ipc_handle_impl(const void* ptr, void* handle, int64_t* offset) {
    if (!addr_range_fn()) return fail(PYG_ERR_CUDA, "cuMemGetAddressRange unavailable");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (addr_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
        return fail(PYG_ERR_INVALID_ARGUMENT, "ipc_handle: not a device allocation");
    cudaIpcMemHandle_t h;
    PYG_CUDA(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)));
    static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
    memcpy(handle, &h, 64);
    *offset = (int64_t)(reinterpret_cast<CUdeviceptr>(ptr) - base);
    return PYG_OK;
}

// A peer allocation can hold several of its buffers (torch's caching allocator packs tensors into
// one cudaMalloc segment) while CUDA maps an IPC handle once per context: mappings are shared and
// reference-counted per allocation.
namespace {
struct IpcMap {
    std::mutex mu;
    std::map<std::string, std::pair<void*, int>> by_handle;  // handle bytes -> (base, refs)
    std::map<void*, std::string> by_base;
};
IpcMap& ipc_map() {
    static IpcMap m;
    return m;
}
}  // namespace

pyg_status_t ipc_open_impl(const void* handle, int64_t offset, void** ptr) {
    IpcMap& m = ipc_map();
    std::lock_guard<std::mutex> g(m.mu);
    const std::string key(static_cast<const char*>(handle), 64);
    auto it = m.by_handle.find(key);
    if (it == m.by_handle.end()) {
        cudaIpcMemHandle_t h;
        memcpy(&h, handle, 64);
        void* base = nullptr;
        PYG_CUDA(cudaIpcOpenMemHandle(&base, h, cudaIpcMemLazyEnablePeerAccess));
        it = m.by_handle.emplace(key, std::make_pair(base, 0)).first;
        m.by_base[base] = key;
    }
    it->second.second += 1;
    *ptr = static_cast<char*>(it->second.first) + offset;
    return PYG_OK;
}

pyg_status_t ipc_close_impl(void* ptr, int64_t offset) {
    IpcMap& m = ipc_map();
    std::lock_guard<std::mutex> g(m.mu);
    void* base = static_cast<char*>(ptr) - offset;
    auto b = m.by_base.find(base);
    if (b == m.by_base.end()) return fail(PYG_ERR_INVALID_ARGUMENT, "ipc_close: not an open mapping");
    auto it = m.by_handle.find(b->second);
    if (--it->second.second == 0) {
        m.by_handle.erase(it);
        m.by_base.erase(b);
        PYG_CUDA(cudaIpcCloseMemHandle(base));
    }
    return PYG_OK;
}

}  // namespace pyg
