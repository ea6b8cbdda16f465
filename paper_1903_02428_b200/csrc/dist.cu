// dist.cu -- the multi-GPU layer of the C ABI (north_star (3); SURVEY.md §8(b) pyg_dist_init /
// pyg_dist_propagate, §8(e)): destination-range partitioning with the source exchange over NCCL
// (NVLink 5 / NVSwitch), forward and backward.
//
// Rank p owns the targets [lo_p, hi_p) -- equal shards of `per` rows -- and every in-edge of them,
// so the BOX of Eq. (1) is local: no cross-GPU reduction, results equal to one GPU
// (bitwise for max / argmax, and for sum / mean too: every row keeps its edge order).  The only
// exchange is the source rows:
//   * all-gather (dense: Reddit references essentially every row from every partition):
//     ncclAllGather of the X shards, or -- for source-blocked plans -- one ncclBroadcast per owner on
//     a side stream with the owner's source blocks (a pass view) run as soon as its rows land;
//   * halo (sparse cross-partition edges, R-MAT): only the referenced remote rows, packed by
//     pyg_gather_rows and delivered by grouped ncclSend / ncclRecv behind the own shard.
// Backward ("both for forward and backward passes"): the rank's local edges, transposed
// (rows = sources in the rank's source index space), give partial dL/dX for every source they
// reference (segment-reduce; MAX routes through argmax) -> ncclReduceScatter to the owners
// (all-gather mode) or the reverse halo: the halo rows' partials are sent back to their owners and
// added in rank order by a segment-reduce over a plan of the received rows (deterministic).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2 -- the one torch already loaded, if any),
// so the library loads without it; a missing NCCL or a failing NCCL call returns PYG_ERR_NCCL.
// Dist plans own their device buffers (cudaMalloc at build, cudaFree at destroy).
#include <dlfcn.h>
#include <nccl.h>

#include <cub/cub.cuh>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

namespace pyg {
namespace {

struct NcclApi {
    bool loaded = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        // $PYG_NCCL_LIB names the library exactly (no fallback); else the soname torch loaded
        const char* env = getenv("PYG_NCCL_LIB");
        void* h = nullptr;
        if (env && *env) {
            h = dlopen(env, RTLD_NOW | RTLD_GLOBAL);
        } else {
            for (const char* n : {"libnccl.so.2", "libnccl.so"})
                if ((h = dlopen(n, RTLD_NOW | RTLD_GLOBAL))) break;
        }
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("cannot load NCCL: ") + (e ? e : "dlopen failed");
            return;
        }
#define PYG_SYM(field, name)                                                   \
    api.field = reinterpret_cast<decltype(api.field)>(dlsym(h, name));        \
    if (!api.field) {                                                          \
        api.why = std::string("NCCL symbol missing: ") + name;                 \
        return;                                                                \
    }
        PYG_SYM(GetUniqueId, "ncclGetUniqueId")
        PYG_SYM(CommInitRank, "ncclCommInitRank")
        PYG_SYM(CommDestroy, "ncclCommDestroy")
        PYG_SYM(GetErrorString, "ncclGetErrorString")
        PYG_SYM(AllGather, "ncclAllGather")
        PYG_SYM(ReduceScatter, "ncclReduceScatter")
        PYG_SYM(AllReduce, "ncclAllReduce")
        PYG_SYM(Broadcast, "ncclBroadcast")
        PYG_SYM(Send, "ncclSend")
        PYG_SYM(Recv, "ncclRecv")
        PYG_SYM(GroupStart, "ncclGroupStart")
        PYG_SYM(GroupEnd, "ncclGroupEnd")
#undef PYG_SYM
        api.loaded = true;
    });
    return api;
}

#define PYG_NCCL(call)                                                                                  \
    do {                                                                                                \
        ncclResult_t _r = (call);                                                                       \
        if (_r != ncclSuccess) return fail(PYG_ERR_NCCL, "NCCL error %d (%s) in %s", (int)_r,          \
                                           nccl().GetErrorString ? nccl().GetErrorString(_r) : "?", #call); \
    } while (0)

int grid_for(int64_t work, int threads = 256) {
    int64_t b = cdiv(work, threads);
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

#define GRID_STRIDE(t, total) \
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < (total); t += (int64_t)gridDim.x * blockDim.x)

__global__ void local_flag_kernel(const int64_t* __restrict__ dst, int64_t E, int64_t lo, int64_t hi, char* flag) {
    GRID_STRIDE(k, E) flag[k] = (dst[k] >= lo && dst[k] < hi) ? 1 : 0;
}

// local edge j (global id eid[j], ascending): (source in the rank's source index space, local target)
__global__ void local_edges_kernel(const int64_t* __restrict__ ei, int64_t E, const int64_t* __restrict__ eid,
                                   int64_t n_loc, int64_t lo, int64_t hi, int64_t per, const int64_t* __restrict__ halo,
                                   int64_t n_halo, int64_t* src_out, int64_t* dst_out) {
    GRID_STRIDE(j, n_loc) {
        const int64_t k = eid[j];
        int64_t s = ei[k];
        if (halo) {  // rank-local ids: own rows first, then the halo rows in ascending global id
            if (s >= lo && s < hi) {
                s -= lo;
            } else {
                int64_t a = 0, b = n_halo;
                while (a < b) {
                    const int64_t m = (a + b) >> 1;
                    if (halo[m] < s) a = m + 1; else b = m;
                }
                s = per + a;
            }
        }
        src_out[j] = s;
        dst_out[j] = ei[E + k] - lo;
    }
}

__global__ void compose_perm_kernel(const int32_t* __restrict__ perm, const int64_t* __restrict__ eid, int64_t n,
                                    int32_t* out) {
    GRID_STRIDE(p, n) out[p] = (int32_t)eid[perm[p]];
}

__global__ void sub_kernel(int64_t* v, int64_t n, int64_t off) {
    GRID_STRIDE(t, n) v[t] -= off;
}

// MAX backward: partial[src(arg[i][c])][c] += w * g[i][c]; src via the local edge list (sorted by
// global edge id).  Each (i, c) feeds one source; only multi-argmax sources sum several terms.
__global__ void dist_max_route_kernel(const float* __restrict__ g, int64_t ldg, const int64_t* __restrict__ arg,
                                      int64_t lda, int F, int64_t n, const int64_t* __restrict__ eid,
                                      const int64_t* __restrict__ src, int64_t n_loc, const float* __restrict__ w,
                                      int64_t E, float* part, int64_t ldp) {
    GRID_STRIDE(t, n * F) {
        const int64_t i = t / F;
        const int c = (int)(t - i * F);
        const int64_t k = arg[i * lda + c];
        if (k < 0 || k >= E) continue;
        int64_t a = 0, b = n_loc;
        while (a < b) {
            const int64_t m = (a + b) >> 1;
            if (eid[m] < k) a = m + 1; else b = m;
        }
        if (a >= n_loc || eid[a] != k) continue;  // not a local edge (cannot happen for own rows)
        const float gv = g[i * ldg + c];
        atomicAdd(part + src[a] * ldp + c, w ? w[k] * gv : gv);
    }
}

}  // namespace
}  // namespace pyg

using namespace pyg;

struct pyg_dist {
    ncclComm_t comm = nullptr;
    int rank = 0, world = 1, device = 0;
    cudaStream_t side = nullptr;  // broadcasts of the overlapped all-gather
};

struct pyg_dist_plan {
    pyg_dist* d = nullptr;
    int64_t n = 0, E = 0, F = 0, ld = 0, per = 0, lo = 0, hi = 0, n_own = 0, col_block = 0;
    int exchange = 0;
    int64_t n_halo = 0, n_send = 0, n_loc = 0, n_src_space = 0;
    pyg_plan_t* plan_full = nullptr;  // global forward plan (every rank builds it)
    pyg_plan_t* slice = nullptr;      // rows [lo, hi)
    pyg_plan_t* halo_plan = nullptr;  // slice with rank-local gathered ids (halo mode)
    std::vector<pyg_plan_t*> views;   // per-owner pass views (overlapped all-gather)
    pyg_plan_t* planT = nullptr;      // local edges transposed (rows = sources, rank source space)
    pyg_plan* planT_g = nullptr;      // the same with GLOBAL edge ids as perm (weights by edge id)
    pyg_plan_t* rev_plan = nullptr;   // scatter plan of the reverse-halo rows over own rows
    float* xbuf = nullptr;            // [per * world | per + n_halo] x ld
    float* sendbuf = nullptr;         // halo pack [n_send x ld]
    int64_t* send_rows = nullptr;     // [n_send] local rows of the own shard, grouped by peer
    int64_t* halo_ids = nullptr;      // [n_halo]
    float* part = nullptr;            // backward partials [n_src_space x ld]
    float* rs_out = nullptr;          // reduce-scatter output [per x ld]
    float* rbuf = nullptr;            // reverse-halo receive [n_send x ld]
    int64_t* eid_loc = nullptr;       // [n_loc] global ids of the local edges, ascending
    int64_t* ledges = nullptr;        // [2 x n_loc] (source in rank space, local target)
    int32_t* perm_g = nullptr;        // [n_loc]
    int32_t* deg_loc = nullptr;       // [n_own] in-degree of own targets
    void* ws = nullptr;               // propagate / backward scratch
    size_t ws_bytes = 0;
    std::vector<int64_t> send_counts, recv_counts, soff, roff;  // rows per peer
    std::vector<void*> allocs;
    std::vector<cudaEvent_t> events;
    ~pyg_dist_plan() {
        for (auto* v : views) pyg_plan_destroy(v);
        if (rev_plan) pyg_plan_destroy(rev_plan);
        delete planT_g;
        if (planT) pyg_plan_destroy(planT);
        if (halo_plan) pyg_plan_destroy(halo_plan);
        if (slice) pyg_plan_destroy(slice);
        if (plan_full) pyg_plan_destroy(plan_full);
        for (auto e : events) cudaEventDestroy(e);
        for (void* p : allocs) cudaFree(p);
    }
    void release(void* p) {
        for (auto& q : allocs)
            if (q == p) {
                cudaFree(q);
                q = allocs.back();
                allocs.pop_back();
                return;
            }
    }
    template <class T>
    pyg_status_t alloc(T** p, size_t n) {
        void* q = nullptr;
        if (n == 0) n = 1;
        PYG_CUDA(cudaMalloc(&q, n * sizeof(T)));
        allocs.push_back(q);
        *p = static_cast<T*>(q);
        return PYG_OK;
    }
};

#define REQUIRE(cond, st, ...)                     \
    do {                                           \
        if (!(cond)) return fail(st, __VA_ARGS__); \
    } while (0)

namespace {

pyg_status_t build_plan(pyg_dist_plan* P, const int64_t* row, const int64_t* col, int64_t E, int64_t n_rows,
                        int64_t n_cols, int64_t col_block, pyg_plan_t** out, cudaStream_t s) {
    size_t nb = 0;
    PYG_TRY(pyg_plan_workspace_size(E, n_rows, n_cols, col_block, &nb));
    char* ws = nullptr;
    PYG_TRY(P->alloc(&ws, nb));
    return pyg_plan_build(row, col, E, n_rows, n_cols, col_block, 0, ws, nb, out, s);
}

// grouped send / recv of int64 rows: sc[q] / rc[q] elements to / from peer q
pyg_status_t exchange_i64(pyg_dist* d, const int64_t* send, const std::vector<int64_t>& sc, int64_t* recv,
                          const std::vector<int64_t>& rc, cudaStream_t s) {
    PYG_NCCL(nccl().GroupStart());
    int64_t so = 0, ro = 0;
    for (int q = 0; q < d->world; ++q) {
        if (sc[q] > 0) PYG_NCCL(nccl().Send(send + so, (size_t)sc[q], ncclInt64, q, d->comm, s));
        if (rc[q] > 0) PYG_NCCL(nccl().Recv(recv + ro, (size_t)rc[q], ncclInt64, q, d->comm, s));
        so += sc[q];
        ro += rc[q];
    }
    PYG_NCCL(nccl().GroupEnd());
    return PYG_OK;
}

}  // namespace

extern "C" {

pyg_status_t pyg_dist_unique_id(void* id) {
    REQUIRE(id, PYG_ERR_INVALID_ARGUMENT, "dist_unique_id: null");
    NcclApi& api = nccl();
    REQUIRE(api.loaded, PYG_ERR_NCCL, "NCCL unavailable: %s", api.why.c_str());
    ncclUniqueId u;
    PYG_NCCL(api.GetUniqueId(&u));
    memcpy(id, &u, sizeof u);
    return PYG_OK;
}

pyg_status_t pyg_dist_init(const void* nccl_unique_id, int rank, int world, pyg_dist_t** comm) {
    REQUIRE(nccl_unique_id && comm, PYG_ERR_INVALID_ARGUMENT, "dist_init: null");
    REQUIRE(world >= 1 && rank >= 0 && rank < world, PYG_ERR_INVALID_ARGUMENT, "dist_init: rank %d / world %d", rank,
            world);
    *comm = nullptr;
    NcclApi& api = nccl();
    REQUIRE(api.loaded, PYG_ERR_NCCL, "NCCL unavailable: %s", api.why.c_str());
    ncclUniqueId u;
    memcpy(&u, nccl_unique_id, sizeof u);
    auto* d = new pyg_dist();
    d->rank = rank;
    d->world = world;
    cudaError_t e = cudaGetDevice(&d->device);
    if (e != cudaSuccess) {
        delete d;
        return cuda_check(e, "cudaGetDevice");
    }
    ncclResult_t r = api.CommInitRank(&d->comm, world, u, rank);
    if (r != ncclSuccess) {
        delete d;
        return fail(PYG_ERR_NCCL, "ncclCommInitRank: %s", api.GetErrorString(r));
    }
    e = cudaStreamCreateWithFlags(&d->side, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        api.CommDestroy(d->comm);
        delete d;
        return cuda_check(e, "cudaStreamCreate");
    }
    *comm = d;
    return PYG_OK;
}

void pyg_dist_finalize(pyg_dist_t* d) {
    if (!d) return;
    if (d->side) cudaStreamDestroy(d->side);
    if (d->comm && nccl().loaded) nccl().CommDestroy(d->comm);
    delete d;
}

pyg_status_t pyg_dist_plan_build(pyg_dist_t* d, const int64_t* edge_index, int64_t E, int64_t n, int64_t F,
                                 int64_t ld, int64_t col_block, int exchange, pyg_dist_plan_t** out, void* stream) {
    REQUIRE(d && out, PYG_ERR_INVALID_ARGUMENT, "dist_plan_build: null");
    REQUIRE(E >= 0 && n >= 0 && F >= 0 && col_block >= 0, PYG_ERR_INVALID_ARGUMENT, "dist_plan_build: negative size");
    REQUIRE(E == 0 || edge_index, PYG_ERR_INVALID_ARGUMENT, "dist_plan_build: null edge_index");
    REQUIRE(ld >= F && ld % 4 == 0, PYG_ERR_DIMENSION, "dist_plan_build: ld must be >= F and a multiple of 4");
    REQUIRE(exchange >= PYG_EXCHANGE_AUTO && exchange <= PYG_EXCHANGE_HALO, PYG_ERR_INVALID_ARGUMENT,
            "dist_plan_build: bad exchange");
    REQUIRE(!(exchange == PYG_EXCHANGE_HALO && col_block > 0), PYG_ERR_UNSUPPORTED,
            "dist_plan_build: the halo exchange needs an unblocked plan (col_block = 0)");
    REQUIRE(n <= 0x7ffffffeLL && E <= 0x7ffffffeLL, PYG_ERR_UNSUPPORTED, "dist_plan_build: sizes must be < 2^31");
    *out = nullptr;
    cudaStream_t s = as_stream(stream);
    auto P = std::make_unique<pyg_dist_plan>();
    P->d = d;
    P->n = n;
    P->E = E;
    P->F = F;
    P->ld = ld;
    const int W = d->world, R = d->rank;
    // partition: equal shards; source-blocked plans align the shards with the blocks (per = k * cb)
    int64_t per = cdiv(n, W);
    if (col_block > 0) {
        const int64_t k = std::max<int64_t>(1, cdiv(per, col_block));
        col_block = std::max<int64_t>(1, cdiv(per, k));
        per = k * col_block;
    }
    P->per = per;
    P->col_block = col_block;
    P->lo = std::min<int64_t>((int64_t)R * per, n);
    P->hi = std::min<int64_t>((int64_t)(R + 1) * per, n);
    P->n_own = P->hi - P->lo;
    PYG_TRY(build_plan(P.get(), edge_index + E, edge_index, E, n, n, col_block, &P->plan_full, s));
    PYG_TRY(pyg_plan_slice(P->plan_full, P->lo, P->hi, &P->slice));

    // halo (unblocked plans): the referenced remote rows
    std::vector<int64_t> h_halo;
    if (col_block == 0 && W > 1 && exchange != PYG_EXCHANGE_ALLGATHER) {
        size_t hb = 0;
        PYG_TRY(pyg_halo_workspace_size(P->slice, n, &hb));
        char* hws = nullptr;
        PYG_TRY(P->alloc(&hws, hb));
        int64_t* hids = nullptr;
        PYG_TRY(P->alloc(&hids, (size_t)std::max<int64_t>(n, 1)));
        int64_t nh = 0;
        PYG_TRY(pyg_halo_build(P->slice, n, P->lo, P->hi, per, hws, hb, &P->halo_plan, hids, &nh, stream));
        // largest halo over the ranks decides AUTO (the same choice on every rank)
        int64_t* dmax = nullptr;
        PYG_TRY(P->alloc(&dmax, 1));
        PYG_CUDA(cudaMemcpyAsync(dmax, &nh, 8, cudaMemcpyHostToDevice, s));
        PYG_NCCL(nccl().AllReduce(dmax, dmax, 1, ncclInt64, ncclMax, d->comm, s));
        int64_t nh_max = 0;
        PYG_CUDA(cudaMemcpyAsync(&nh_max, dmax, 8, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        const bool use = exchange == PYG_EXCHANGE_HALO || (double)nh_max < 0.5 * (double)(W - 1) * (double)per;
        if (use) {
            P->exchange = PYG_EXCHANGE_HALO;
            P->n_halo = nh;
            P->halo_ids = hids;
            h_halo.resize((size_t)nh);
            if (nh > 0) PYG_CUDA(cudaMemcpyAsync(h_halo.data(), hids, 8 * (size_t)nh, cudaMemcpyDeviceToHost, s));
            PYG_CUDA(cudaStreamSynchronize(s));
        } else {
            pyg_plan_destroy(P->halo_plan);
            P->halo_plan = nullptr;
        }
    }
    if (P->exchange != PYG_EXCHANGE_HALO) P->exchange = PYG_EXCHANGE_ALLGATHER;
    const bool halo = P->exchange == PYG_EXCHANGE_HALO;
    P->send_counts.assign(W, 0);
    P->recv_counts.assign(W, 0);
    P->soff.assign(W + 1, 0);
    P->roff.assign(W + 1, 0);
    if (halo) {
        // request exchange (plan time): recv_counts[q] halo rows come from owner q, in ascending id
        for (int64_t id : h_halo) P->recv_counts[(size_t)(id / per)] += 1;
        int64_t *c_send = nullptr, *c_recv = nullptr;
        PYG_TRY(P->alloc(&c_send, W));
        PYG_TRY(P->alloc(&c_recv, W));
        PYG_CUDA(cudaMemcpyAsync(c_send, P->recv_counts.data(), 8 * W, cudaMemcpyHostToDevice, s));
        std::vector<int64_t> ones(W, 1);
        PYG_TRY(exchange_i64(d, c_send, ones, c_recv, ones, s));
        PYG_CUDA(cudaMemcpyAsync(P->send_counts.data(), c_recv, 8 * W, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        for (int q = 0; q < W; ++q) {
            P->soff[q + 1] = P->soff[q] + P->send_counts[q];
            P->roff[q + 1] = P->roff[q] + P->recv_counts[q];
        }
        P->n_send = P->soff[W];
        PYG_TRY(P->alloc(&P->send_rows, (size_t)P->n_send));
        PYG_TRY(exchange_i64(d, P->halo_ids, P->recv_counts, P->send_rows, P->send_counts, s));
        if (P->n_send > 0) {
            sub_kernel<<<grid_for(P->n_send), 256, 0, s>>>(P->send_rows, P->n_send, P->lo);
            PYG_LAUNCHED();
        }
        PYG_TRY(P->alloc(&P->sendbuf, (size_t)P->n_send * ld));
        PYG_TRY(P->alloc(&P->rbuf, (size_t)P->n_send * ld));
        PYG_TRY(P->alloc(&P->xbuf, (size_t)(per + P->n_halo) * ld));
        PYG_CUDA(cudaMemsetAsync(P->xbuf, 0, (size_t)(per + P->n_halo) * ld * 4, s));
        P->n_src_space = per + P->n_halo;
        // reverse halo: a scatter plan of the received rows over the own rows (stable: peer order)
        PYG_TRY(build_plan(P.get(), P->send_rows, nullptr, P->n_send, P->n_own, 0, 0, &P->rev_plan, s));
    } else {
        PYG_TRY(P->alloc(&P->xbuf, (size_t)per * W * ld));
        PYG_CUDA(cudaMemsetAsync(P->xbuf, 0, (size_t)per * W * ld * 4, s));
        PYG_TRY(P->alloc(&P->rs_out, (size_t)per * ld));
        P->n_src_space = per * W;
        if (col_block > 0 && W > 1) {  // per-owner pass views for the overlapped all-gather
            pyg_plan_view_t v;
            PYG_TRY(pyg_plan_view(P->slice, &v));
            const int64_t k = per / col_block;
            for (int q = 0; q < W; ++q) {
                pyg_plan_t* view = nullptr;
                const int64_t b0 = q * k, b1 = std::min<int64_t>((q + 1) * k, v.n_col_blocks);
                if (b0 < b1) PYG_TRY(pyg_plan_passes(P->slice, b0, b1, &view));
                P->views.push_back(view);
                cudaEvent_t ev;
                PYG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
                P->events.push_back(ev);
            }
            cudaEvent_t ev;
            PYG_CUDA(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
            P->events.push_back(ev);  // "shard ready" on the caller's stream
        }
    }
    // local edges (targets in [lo, hi)) in ascending global id, and their transposed plan
    {
        char* flag = nullptr;
        PYG_TRY(P->alloc(&flag, (size_t)E));
        int64_t* eid = nullptr;
        PYG_TRY(P->alloc(&eid, (size_t)E));
        int64_t* nsel = nullptr;
        PYG_TRY(P->alloc(&nsel, 1));
        if (E > 0) {
            local_flag_kernel<<<grid_for(E), 256, 0, s>>>(edge_index + E, E, P->lo, P->hi, flag);
            PYG_LAUNCHED();
        }
        size_t tb = 0;
        cub::CountingInputIterator<int64_t> it(0);
        PYG_CUDA(cub::DeviceSelect::Flagged(nullptr, tb, it, flag, eid, nsel, (int)E, s));
        char* tmp = nullptr;
        PYG_TRY(P->alloc(&tmp, tb));
        PYG_CUDA(cub::DeviceSelect::Flagged(tmp, tb, it, flag, eid, nsel, (int)E, s));
        PYG_LAUNCHED();
        int64_t n_loc = 0;
        PYG_CUDA(cudaMemcpyAsync(&n_loc, nsel, 8, cudaMemcpyDeviceToHost, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        P->n_loc = n_loc;
        PYG_TRY(P->alloc(&P->eid_loc, (size_t)n_loc));  // exact size; the E-sized temporaries go
        if (n_loc > 0)
            PYG_CUDA(cudaMemcpyAsync(P->eid_loc, eid, 8 * (size_t)n_loc, cudaMemcpyDeviceToDevice, s));
        PYG_CUDA(cudaStreamSynchronize(s));
        for (void* t : {(void*)flag, (void*)eid, (void*)nsel, (void*)tmp}) P->release(t);
        eid = P->eid_loc;
        PYG_TRY(P->alloc(&P->ledges, 2 * (size_t)n_loc));
        if (n_loc > 0) {
            local_edges_kernel<<<grid_for(n_loc), 256, 0, s>>>(edge_index, E, eid, n_loc, P->lo, P->hi, per,
                                                               halo ? P->halo_ids : nullptr, P->n_halo, P->ledges,
                                                               P->ledges + n_loc);
            PYG_LAUNCHED();
        }
        PYG_TRY(build_plan(P.get(), P->ledges, P->ledges + n_loc, n_loc, P->n_src_space, P->n_own, 0, &P->planT, s));
        PYG_TRY(P->alloc(&P->perm_g, (size_t)n_loc));
        pyg_plan_view_t v;
        PYG_TRY(pyg_plan_view(P->planT, &v));
        if (n_loc > 0) {
            compose_perm_kernel<<<grid_for(n_loc), 256, 0, s>>>(v.perm, eid, n_loc, P->perm_g);
            PYG_LAUNCHED();
        }
        P->planT_g = new pyg_plan(*P->planT);
        P->planT_g->perm = P->perm_g;
        P->planT_g->perm_identity = 0;
        PYG_TRY(P->alloc(&P->deg_loc, (size_t)P->n_own));
        PYG_TRY(pyg_degree(P->ledges + n_loc, n_loc, P->n_own, 0, P->deg_loc, stream));
        PYG_TRY(P->alloc(&P->part, (size_t)P->n_src_space * ld));
        PYG_CUDA(cudaMemsetAsync(P->part, 0, (size_t)P->n_src_space * ld * 4, s));
    }
    // scratch for every call of this plan: the max over forward / backward / reverse-halo needs
    size_t wb = 0;
    for (int r = PYG_SUM; r <= PYG_MAX; ++r) {
        size_t b = 0;
        PYG_TRY(pyg_workspace_size(halo ? P->halo_plan : P->slice, E, P->n_own, F, (pyg_reduce_t)r, 0, &b));
        wb = std::max(wb, b);
        PYG_TRY(pyg_workspace_size(P->planT, P->n_loc, P->n_src_space, F, PYG_SUM, 0, &b));
        wb = std::max(wb, b);
        if (P->rev_plan) {
            PYG_TRY(pyg_workspace_size(P->rev_plan, P->n_send, P->n_own, F, PYG_SUM, 0, &b));
            wb = std::max(wb, b);
        }
    }
    P->ws_bytes = wb;
    char* wsp = nullptr;
    PYG_TRY(P->alloc(&wsp, wb));
    P->ws = wsp;
    PYG_CUDA(cudaStreamSynchronize(s));
    *out = P.release();
    return PYG_OK;
}

pyg_status_t pyg_dist_plan_info(const pyg_dist_plan_t* P, pyg_dist_plan_info_t* info) {
    REQUIRE(P && info, PYG_ERR_INVALID_ARGUMENT, "dist_plan_info: null");
    info->lo = P->lo;
    info->hi = P->hi;
    info->per = P->per;
    info->exchange = P->exchange;
    info->n_halo = P->n_halo;
    info->n_send = P->n_send;
    info->n_local_edges = P->n_loc;
    info->col_block = P->col_block;
    info->x_shard = P->exchange == PYG_EXCHANGE_HALO ? P->xbuf : P->xbuf + (size_t)P->d->rank * P->per * P->ld;
    info->ldx = P->ld;
    info->plan = P->slice;
    return PYG_OK;
}

void pyg_dist_plan_destroy(pyg_dist_plan_t* P) { delete P; }

pyg_status_t pyg_dist_propagate(pyg_dist_plan_t* P, const float* x_shard, int64_t ldx, const float* edge_weight,
                                pyg_reduce_t reduce, uint32_t flags, float* out, int64_t ldo, int64_t* arg_out,
                                void* stream) {
    REQUIRE(P, PYG_ERR_INVALID_ARGUMENT, "dist_propagate: null plan");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "dist_propagate: bad reduce");
    REQUIRE(!(flags & PYG_PHI_CONCAT_XI), PYG_ERR_UNSUPPORTED, "dist_propagate: CONCAT_XI is not supported");
    REQUIRE(P->n_own * P->F == 0 || (x_shard && out), PYG_ERR_INVALID_ARGUMENT, "dist_propagate: null x / out");
    REQUIRE(ldx >= P->F && ldo >= P->F, PYG_ERR_DIMENSION, "dist_propagate: leading dimension < F");
    REQUIRE(reduce != PYG_MAX || P->n_own * P->F == 0 || arg_out, PYG_ERR_INVALID_ARGUMENT,
            "dist_propagate: max needs arg_out");
    pyg_dist* d = P->d;
    cudaStream_t s = as_stream(stream);
    const int64_t F = P->F, ld = P->ld;
    const int W = d->world, R = d->rank;
    const bool halo = P->exchange == PYG_EXCHANGE_HALO;
    float* own = halo ? P->xbuf : P->xbuf + (size_t)R * P->per * ld;
    if (x_shard != own && P->n_own > 0)
        PYG_CUDA(cudaMemcpy2DAsync(own, ld * 4, x_shard, ldx * 4, F * 4, P->n_own, cudaMemcpyDeviceToDevice, s));
    if (halo) {
        if (P->n_send > 0) PYG_TRY(pyg_gather_rows(own, P->per, F, ld, P->send_rows, P->n_send, 0, P->sendbuf, ld, stream));
        PYG_NCCL(nccl().GroupStart());
        for (int q = 0; q < W; ++q) {
            if (P->send_counts[q] > 0)
                PYG_NCCL(nccl().Send(P->sendbuf + P->soff[q] * ld, (size_t)(P->send_counts[q] * ld), ncclFloat32, q,
                                     d->comm, s));
            if (P->recv_counts[q] > 0)
                PYG_NCCL(nccl().Recv(P->xbuf + (P->per + P->roff[q]) * ld, (size_t)(P->recv_counts[q] * ld),
                                     ncclFloat32, q, d->comm, s));
        }
        PYG_NCCL(nccl().GroupEnd());
        return pyg_propagate(P->xbuf, P->per + P->n_halo, F, ld, nullptr, 0, P->n_own, nullptr, P->E, nullptr, 0, 0,
                             edge_weight, reduce, flags, out, ldo, arg_out, P->halo_plan, P->ws, P->ws_bytes, stream);
    }
    const size_t shard = (size_t)P->per * ld;
    if (!P->views.empty()) {
        // overlapped all-gather: owner q's broadcast on the side stream, its source blocks as soon as
        // its event fires; blocks stay in ascending order (bitwise the one-GPU result)
        cudaEvent_t ready = P->events[W];
        PYG_CUDA(cudaEventRecord(ready, s));
        PYG_CUDA(cudaStreamWaitEvent(d->side, ready, 0));
        for (int q = 0; q < W; ++q) {
            PYG_NCCL(nccl().Broadcast(P->xbuf + q * shard, P->xbuf + q * shard, shard, ncclFloat32, q, d->comm, d->side));
            PYG_CUDA(cudaEventRecord(P->events[q], d->side));
        }
        for (int q = 0; q < W; ++q) {
            PYG_CUDA(cudaStreamWaitEvent(s, P->events[q], 0));
            if (P->views[q])
                PYG_TRY(pyg_propagate(P->xbuf, P->n, F, ld, nullptr, 0, P->n_own, nullptr, P->E, nullptr, 0, 0,
                                      edge_weight, reduce, flags, out, ldo, arg_out, P->views[q], P->ws, P->ws_bytes,
                                      stream));
        }
        return PYG_OK;
    }
    PYG_NCCL(nccl().AllGather(own, P->xbuf, shard, ncclFloat32, d->comm, s));
    return pyg_propagate(P->xbuf, P->n, F, ld, nullptr, 0, P->n_own, nullptr, P->E, nullptr, 0, 0, edge_weight, reduce,
                         flags, out, ldo, arg_out, P->slice, P->ws, P->ws_bytes, stream);
}

pyg_status_t pyg_dist_propagate_backward(pyg_dist_plan_t* P, const float* grad_out, int64_t ldg,
                                         const float* edge_weight, pyg_reduce_t reduce, const int64_t* arg_out,
                                         int64_t lda, float* grad_x_shard, int64_t ldgx, void* stream) {
    REQUIRE(P, PYG_ERR_INVALID_ARGUMENT, "dist_propagate_backward: null plan");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "dist_propagate_backward: bad reduce");
    REQUIRE(P->n_own * P->F == 0 || (grad_out && grad_x_shard), PYG_ERR_INVALID_ARGUMENT,
            "dist_propagate_backward: null pointer");
    REQUIRE(ldg >= P->F && ldgx >= P->F, PYG_ERR_DIMENSION, "dist_propagate_backward: leading dimension < F");
    REQUIRE(reduce != PYG_MAX || P->n_own * P->F == 0 || (arg_out && lda >= P->F), PYG_ERR_INVALID_ARGUMENT,
            "dist_propagate_backward: max needs arg_out (stride lda)");
    pyg_dist* d = P->d;
    cudaStream_t s = as_stream(stream);
    const int64_t F = P->F, ld = P->ld;
    const int W = d->world, R = d->rank;
    const bool halo = P->exchange == PYG_EXCHANGE_HALO;
    // 1. partial dL/dX over the rank's source space from its local edges
    if (reduce == PYG_MAX) {
        PYG_CUDA(cudaMemset2DAsync(P->part, ld * 4, 0, F * 4, P->n_src_space, s));
        if (P->n_own * F > 0) {
            dist_max_route_kernel<<<grid_for(P->n_own * F), 256, 0, s>>>(grad_out, ldg, arg_out, lda, (int)F, P->n_own,
                                                                         P->eid_loc, P->ledges, P->n_loc, edge_weight,
                                                                         P->E, P->part, ld);
            PYG_LAUNCHED();
            PYG_CUDA(cudaGetLastError());
        }
    } else if (F > 0) {
        SegArgs a;
        a.X = grad_out; a.ldx = ldg; a.ncols = (int)F;
        a.rowptr = P->planT_g->rowptr; a.gidx = P->planT_g->col; a.eid = P->planT_g->perm;
        a.w = edge_weight; a.gdeg = reduce == PYG_MEAN ? P->deg_loc : nullptr;
        a.out = P->part; a.ldo = ld; a.n_rows = P->n_src_space; a.E_sentinel = P->E;
        a.heavy_threshold = P->planT_g->heavy_threshold;
        PYG_TRY(segment_reduce(a, PYG_SUM, P->planT_g, P->ws, P->ws_bytes, s));
    }
    // 2. send every partial to the owner of its source row
    if (!halo) {
        PYG_NCCL(nccl().ReduceScatter(P->part, P->rs_out, (size_t)P->per * ld, ncclFloat32, ncclSum, d->comm, s));
        if (P->n_own > 0)
            PYG_CUDA(cudaMemcpy2DAsync(grad_x_shard, ldgx * 4, P->rs_out, ld * 4, F * 4, P->n_own,
                                       cudaMemcpyDeviceToDevice, s));
        (void)R;
        return PYG_OK;
    }
    // reverse halo: my halo rows' partials go back to their owners; I receive, per peer, the partials
    // of the own rows that peer referenced (send_rows order) and add them in rank order
    PYG_NCCL(nccl().GroupStart());
    for (int q = 0; q < W; ++q) {
        if (P->recv_counts[q] > 0)
            PYG_NCCL(nccl().Send(P->part + (P->per + P->roff[q]) * ld, (size_t)(P->recv_counts[q] * ld), ncclFloat32,
                                 q, d->comm, s));
        if (P->send_counts[q] > 0)
            PYG_NCCL(nccl().Recv(P->rbuf + P->soff[q] * ld, (size_t)(P->send_counts[q] * ld), ncclFloat32, q, d->comm,
                                 s));
    }
    PYG_NCCL(nccl().GroupEnd());
    if (P->n_own == 0 || F == 0) return PYG_OK;
    // grad = (sum of the received partials of each own row, in peer order) + own partial
    pyg_plan_view_t v;
    PYG_TRY(pyg_plan_view(P->rev_plan, &v));
    SegArgs a;
    a.X = P->rbuf; a.ldx = ld; a.ncols = (int)F;
    a.rowptr = v.rowptr; a.gidx = nullptr; a.eid = v.perm_is_identity ? nullptr : v.perm;
    a.out = grad_x_shard; a.ldo = ldgx; a.n_rows = P->n_own; a.E_sentinel = P->n_send;
    a.heavy_threshold = v.heavy_threshold;
    a.blend = P->part; a.ldb = ld; a.blend_a = 1.0f; a.blend_b = 1.0f;
    return segment_reduce(a, PYG_SUM, P->rev_plan, P->ws, P->ws_bytes, s);
}

}  // extern "C"
