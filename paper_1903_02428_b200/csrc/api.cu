// api.cu -- the extern "C" boundary of libpygs.so (include/pyg_gs.h): host-side
// validation, strategy selection (plan => CSR segment-reduce, no plan => atomic
// COO) and the launch sequence of each call.  No compute happens here.
#include <stdarg.h>
#include <stdio.h>

#include <cmath>
#include <string>

#include "kernels.cuh"

namespace pyg {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_err;

void set_error(const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
}

pyg_status_t fail(pyg_status_t st, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    t_err = buf;
    return st;
}

pyg_status_t cuda_check(cudaError_t e, const char* what) {
    return fail(PYG_ERR_CUDA, "CUDA error %s (%s) in %s", cudaGetErrorName(e), cudaGetErrorString(e), what);
}

static Knobs read_knobs() {
    Knobs k;
    auto get = [](const char* name, int dflt) {
        const char* e = getenv(name);
        return (e && *e) ? atoi(e) : dflt;
    };
    k.seg_tma = get("PYG_SEG_TMA", -1);
    k.tma_hubs = get("PYG_TMA_HUBS", 1);
    k.tma_warp_kb = get("PYG_TMA_WARP_KB", 4);
    k.tma_warps = get("PYG_TMA_WARPS", 8);
    k.seg_bulk = get("PYG_SEG_BULK", -1);
    k.bulk_warp_kb = get("PYG_BULK_WARP_KB", 8);
    k.gat_warp_kb = get("PYG_GAT_WARP_KB", 10);
    k.gat_sm_kb = get("PYG_GAT_SM_KB", 160);
    k.gat_fused = get("PYG_GAT_FUSED", 1);
    k.gat_warps = get("PYG_GAT_WARPS", 8);
    k.coo_l2_mb = get("PYG_COO_L2_MB", 72);
    k.coo_tile = get("PYG_COO_TILE", 1);
    k.coo_compact = get("PYG_COO_COMPACT", 1);
    k.coo_chunk = get("PYG_COO_CHUNK", 128);
    k.coo_l2_mb_max = get("PYG_COO_L2_MB_MAX", 96);
    k.gat_fwd_warp_kb = get("PYG_GAT_FWD_WARP_KB", 5);
    k.gat_fwd_sm_kb = get("PYG_GAT_FWD_SM_KB", 160);
    return k;
}
static Knobs g_knobs = read_knobs();
const Knobs& knobs() { return g_knobs; }


// PYG_VALIDATE flag: one pinned, mapped int per host thread (so concurrent calls on other threads
// never consume each other's errors).  validate_begin() clears it before a validating call launches
// its checking kernels (every earlier use on this thread ended with the synchronising check).
namespace {
struct MappedFlag {
    int* p = nullptr;
    ~MappedFlag() {
        if (p) cudaFreeHost(p);
    }
};
thread_local MappedFlag t_flag;
}  // namespace

int* validate_flag_dev() {
    if (!t_flag.p) {
        if (cudaHostAlloc(reinterpret_cast<void**>(&t_flag.p), sizeof(int),
                          cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
            t_flag.p = nullptr;
            return nullptr;
        }
        *t_flag.p = 0;
    }
    return t_flag.p;  // UVA: the host pointer is valid on the device
}

void validate_begin() {
    int* f = validate_flag_dev();
    if (f) *reinterpret_cast<volatile int*>(f) = 0;
}

pyg_status_t validate_flag_check(cudaStream_t s, const char* what) {
    PYG_CUDA(cudaStreamSynchronize(s));
    int* f = validate_flag_dev();
    const int v = f ? *reinterpret_cast<volatile int*>(f) : 0;
    if (f) *f = 0;
    if (v == 1) return fail(PYG_ERR_INDEX_OUT_OF_BOUNDS, "%s", what);
    if (v == 2) return fail(PYG_ERR_DIMENSION, "%s", what);
    return PYG_OK;
}

// defined in plan.cu / misc.cu
pyg_status_t plan_workspace(int64_t E, int64_t n_rows, int64_t n_cols, int64_t col_block, size_t* bytes);
pyg_status_t plan_build_impl(const int64_t* row, const int64_t* col, int64_t E, int64_t n_rows, int64_t n_cols,
                             int64_t col_block, void* ws, size_t bytes, pyg_plan** out, cudaStream_t s);
pyg_status_t plan_slice_impl(const pyg_plan* p, int64_t lo, int64_t hi, pyg_plan** out);
pyg_status_t plan_passes_impl(const pyg_plan* p, int64_t lo, int64_t hi, pyg_plan** out);
pyg_status_t plan_export_impl(const pyg_plan* p, int64_t* rowptr, int64_t* col, int64_t* perm, cudaStream_t s);
pyg_status_t gcn_norm_impl(const int64_t* ei, int64_t E, int64_t N, const float* w, int64_t* eo, float* wo,
                           int64_t* E_out, void* ws, size_t bytes, cudaStream_t s, size_t* need);
pyg_status_t collate_impl(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr, const int64_t* local,
                          int64_t Et, int64_t Nt, uint32_t flags, int64_t* ei, int64_t* batch, int64_t* node_ptr,
                          cudaStream_t s);
pyg_status_t halo_workspace_impl(const pyg_plan* p, int64_t n_src, size_t* bytes);
pyg_status_t halo_build_impl(const pyg_plan* p, int64_t n_src, int64_t own_lo, int64_t own_hi, int64_t own_rows,
                             void* ws, size_t bytes, pyg_plan** out, int64_t* halo_ids, int64_t* n_halo,
                             cudaStream_t s);
pyg_status_t dense_transform_impl(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W, int64_t N,
                                  int64_t ldw, const float* bias, const float* row_scale, float* Y, int64_t ldy,
                                  cudaStream_t s, const float* att_src = nullptr, const float* att_dst = nullptr,
                                  float* s_src = nullptr, float* s_dst = nullptr, int heads = 0);
pyg_status_t gcn_dinv(const int64_t* rowptr, const int32_t* deg, int64_t n, float* dinv, cudaStream_t s);
pyg_status_t halo_push_impl(const float* x, int64_t ldx, int64_t F, const int64_t* rows, const int64_t* ptr,
                            void* const* dst, const int64_t* dst_row, int64_t ldd, int n_peers, cudaStream_t s);
pyg_status_t ipc_handle_impl(const void* ptr, void* handle, int64_t* offset);
pyg_status_t ipc_open_impl(const void* handle, int64_t offset, void** ptr);
pyg_status_t ipc_close_impl(void* ptr, int64_t offset);
pyg_status_t global_pool_impl(const float* x, int64_t ldx, int F, const int64_t* node_ptr, int64_t G, int reduce,
                              float* out, int64_t ldo, int64_t* arg, int64_t N, cudaStream_t s);
pyg_status_t gather_rows_impl(const float* x, int64_t ldx, int64_t F, const int64_t* rows, int64_t n, float* out,
                              int64_t ldo, cudaStream_t s);

constexpr int64_t kMaxI32 = 0x7fffffffLL - 1;
constexpr int kAttnMaxHeads = 8;
constexpr double kL2BlockFraction = 0.4;  // X block per pass as a fraction of L2
// share of L2 that keeps serving a random row gather from a matrix close to L2's size: an unblocked GCN
// aggregation over Reddit's 119 MB transformed H (0.9 x L2) ran at 0.50 of the L2 roof (6.07 ms), in
// 2 blocks at 0.83 (3.63 ms; gpurun_out/r3o), so only half of L2 is counted as reuse capacity
constexpr double kL2Reuse = 0.5;

// deg + first edge per target (atomic propagate with CONCAT_XI / MEAN), carved before coo_reduce's own
static size_t coo_deg_bytes(int64_t n_out) { return 2 * align_up((size_t)std::max<int64_t>(n_out, 1) * 4, 256); }

static bool use_plan(const pyg_plan* plan, uint32_t flags) { return plan && !(flags & PYG_FORCE_ATOMIC); }

}  // namespace pyg

using namespace pyg;

#define REQUIRE(cond, st, ...)                   \
    do {                                         \
        if (!(cond)) return fail(st, __VA_ARGS__); \
    } while (0)

extern "C" {

const char* pyg_version(void) { return "pygs 0.1.0 (sm_100a)"; }
const char* pyg_last_error(void) { return t_err.c_str(); }
void pyg_refresh_env(void) { g_knobs = read_knobs(); }
uint64_t pyg_launch_count(void) { return g_launches.load(); }

pyg_status_t pyg_degree(const int64_t* index, int64_t E, int64_t n, uint32_t flags, int32_t* deg, void* stream) {
    REQUIRE(E >= 0 && n >= 0, PYG_ERR_INVALID_ARGUMENT, "degree: negative size");
    REQUIRE((E == 0 || index) && (n == 0 || deg), PYG_ERR_INVALID_ARGUMENT, "degree: null pointer");
    REQUIRE(E <= kMaxI32 && n <= kMaxI32, PYG_ERR_UNSUPPORTED, "degree: sizes must be < 2^31");
    cudaStream_t s = as_stream(stream);
    if (flags & PYG_VALIDATE) {
        validate_begin();
        PYG_TRY(validate_index(index, E, 0, n, s));
        PYG_TRY(validate_flag_check(s, "degree: index out of range"));
    }
    return coo_degree(index, E, n, deg, nullptr, s);
}

pyg_status_t pyg_plan_workspace_size(int64_t E, int64_t n_rows, int64_t n_cols, int64_t col_block, size_t* bytes) {
    REQUIRE(bytes && E >= 0 && n_rows >= 0 && n_cols >= 0 && col_block >= 0, PYG_ERR_INVALID_ARGUMENT,
            "plan_workspace_size: bad args");
    REQUIRE(E <= kMaxI32 && n_rows <= kMaxI32 && n_cols <= kMaxI32, PYG_ERR_UNSUPPORTED, "plan: sizes must be < 2^31");
    return plan_workspace(E, n_rows, n_cols, col_block, bytes);
}

pyg_status_t pyg_atomic_tile_cols(int64_t n_out, int64_t n_src, int64_t ncols, pyg_reduce_t reduce, int64_t* cols) {
    REQUIRE(cols && n_out >= 0 && n_src >= 0 && ncols >= 0 && ncols <= kMaxI32, PYG_ERR_INVALID_ARGUMENT,
            "atomic_tile_cols: bad args");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "atomic_tile_cols: bad reduce");
    *cols = coo_tile_cols(n_out, n_src, ncols, reduce);
    return PYG_OK;
}

pyg_status_t pyg_plan_suggest_col_block(int64_t E, int64_t n_rows, int64_t n_cols, int64_t row_bytes,
                                        int64_t* col_block) {
    REQUIRE(col_block && E >= 0 && n_rows >= 0 && n_cols >= 0 && row_bytes > 0, PYG_ERR_INVALID_ARGUMENT,
            "plan_suggest_col_block: bad args");
    *col_block = 0;
    int dev = 0, l2 = 0;
    PYG_CUDA(cudaGetDevice(&dev));
    PYG_CUDA(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    const double x_bytes = (double)n_cols * (double)row_bytes;
    const double budget = kL2BlockFraction * (double)l2;
    if (x_bytes <= budget || n_rows == 0) return PYG_OK;  // X fits one block: one pass
    const int64_t nb = (int64_t)std::ceil(x_bytes / budget);
    // DRAM saved on the gather vs the extra read+write of `out` per additional pass
    const double saved = (double)E * (double)row_bytes * std::max(0.0, 1.0 - kL2Reuse * (double)l2 / x_bytes);
    const double cost = 2.0 * (double)(nb - 1) * (double)n_rows * (double)row_bytes;
    if (saved < 4.0 * cost || nb * n_rows > kMaxI32) return PYG_OK;
    *col_block = cdiv(n_cols, nb);
    return PYG_OK;
}

pyg_status_t pyg_plan_build(const int64_t* row_index, const int64_t* col_index, int64_t E, int64_t n_rows,
                            int64_t n_cols, int64_t col_block, uint32_t flags, void* workspace, size_t bytes,
                            pyg_plan_t** plan, void* stream) {
    (void)flags;
    REQUIRE(plan && E >= 0 && n_rows >= 0 && n_cols >= 0 && col_block >= 0, PYG_ERR_INVALID_ARGUMENT,
            "plan_build: bad args");
    REQUIRE(E == 0 || row_index, PYG_ERR_INVALID_ARGUMENT, "plan_build: null row_index");
    REQUIRE(E <= kMaxI32 && n_rows <= kMaxI32 && n_cols <= kMaxI32, PYG_ERR_UNSUPPORTED, "plan: sizes must be < 2^31");
    *plan = nullptr;
    return plan_build_impl(row_index, col_index, E, n_rows, n_cols, col_block, workspace, bytes, plan,
                           as_stream(stream));
}

pyg_status_t pyg_plan_slice(const pyg_plan_t* plan, int64_t lo, int64_t hi, pyg_plan_t** slice) {
    REQUIRE(plan && slice, PYG_ERR_INVALID_ARGUMENT, "plan_slice: null");
    REQUIRE(0 <= lo && lo <= hi && hi <= plan->n_rows, PYG_ERR_DIMENSION, "plan_slice: rows [%lld, %lld) outside [0, %lld)",
            (long long)lo, (long long)hi, (long long)plan->n_rows);
    return plan_slice_impl(plan, lo, hi, slice);
}

pyg_status_t pyg_plan_passes(const pyg_plan_t* plan, int64_t pass_lo, int64_t pass_hi, pyg_plan_t** view) {
    REQUIRE(plan && view, PYG_ERR_INVALID_ARGUMENT, "plan_passes: null");
    REQUIRE(!plan->parts.empty(), PYG_ERR_UNSUPPORTED, "plan_passes: needs a source-blocked plan (col_block > 0)");
    REQUIRE(0 <= pass_lo && pass_lo < pass_hi && pass_hi <= (int64_t)plan->parts.size(), PYG_ERR_DIMENSION,
            "plan_passes: passes [%lld, %lld) outside [0, %lld)", (long long)pass_lo, (long long)pass_hi,
            (long long)plan->parts.size());
    return plan_passes_impl(plan, pass_lo, pass_hi, view);
}

pyg_status_t pyg_plan_view(const pyg_plan_t* p, pyg_plan_view_t* v) {
    REQUIRE(p && v, PYG_ERR_INVALID_ARGUMENT, "plan_view: null");
    v->n_rows = p->n_rows;
    v->n_cols = p->n_cols;
    v->E = p->E;
    v->row_offset = p->row_offset;
    v->rowptr = p->rowptr;
    v->col = p->col;
    v->perm = p->perm;
    v->perm_is_identity = p->perm_identity;
    v->n_heavy_rows = p->h_hi - p->h_lo;
    v->n_heavy_chunks = p->item_hi - p->item_lo;
    v->heavy_threshold = p->heavy_threshold;
    v->chunk_size = p->chunk;
    v->col_block = p->col_block;
    v->n_col_blocks = p->parts.empty() ? 1 : (int64_t)p->parts.size();
    return PYG_OK;
}

void pyg_plan_destroy(pyg_plan_t* p) { delete p; }

pyg_status_t pyg_halo_workspace_size(const pyg_plan_t* slice, int64_t n_src, size_t* bytes) {
    REQUIRE(slice && bytes && n_src >= 0, PYG_ERR_INVALID_ARGUMENT, "halo_workspace_size: bad args");
    REQUIRE(slice->col && slice->parts.empty(), PYG_ERR_UNSUPPORTED,
            "halo: needs an unblocked forward plan (col_index given, col_block = 0)");
    REQUIRE(slice->n_cols <= n_src, PYG_ERR_DIMENSION, "halo: plan n_cols > n_src");
    return halo_workspace_impl(slice, n_src, bytes);
}

pyg_status_t pyg_halo_build(const pyg_plan_t* slice, int64_t n_src, int64_t own_lo, int64_t own_hi, int64_t own_rows,
                            void* workspace, size_t bytes, pyg_plan_t** halo_plan, int64_t* halo_ids, int64_t* n_halo,
                            void* stream) {
    REQUIRE(slice && halo_plan && n_halo && n_src >= 0, PYG_ERR_INVALID_ARGUMENT, "halo_build: bad args");
    REQUIRE(n_src == 0 || halo_ids, PYG_ERR_INVALID_ARGUMENT, "halo_build: null halo_ids");
    REQUIRE(slice->col && slice->parts.empty(), PYG_ERR_UNSUPPORTED,
            "halo: needs an unblocked forward plan (col_index given, col_block = 0)");
    REQUIRE(0 <= own_lo && own_lo <= own_hi && own_hi <= n_src && own_rows >= own_hi - own_lo, PYG_ERR_DIMENSION,
            "halo_build: own range [%lld, %lld) / own_rows %lld inconsistent with n_src %lld", (long long)own_lo,
            (long long)own_hi, (long long)own_rows, (long long)n_src);
    REQUIRE(slice->n_cols <= n_src, PYG_ERR_DIMENSION, "halo: plan n_cols > n_src");
    *halo_plan = nullptr;
    return halo_build_impl(slice, n_src, own_lo, own_hi, own_rows, workspace, bytes, halo_plan, halo_ids, n_halo,
                           as_stream(stream));
}

pyg_status_t pyg_ipc_handle(const void* dev_ptr, void* handle, int64_t* offset) {
    REQUIRE(dev_ptr && handle && offset, PYG_ERR_INVALID_ARGUMENT, "ipc_handle: null pointer");
    return ipc_handle_impl(dev_ptr, handle, offset);
}

pyg_status_t pyg_ipc_open(const void* handle, int64_t offset, void** dev_ptr) {
    REQUIRE(handle && dev_ptr && offset >= 0, PYG_ERR_INVALID_ARGUMENT, "ipc_open: bad args");
    return ipc_open_impl(handle, offset, dev_ptr);
}

pyg_status_t pyg_ipc_close(void* dev_ptr, int64_t offset) {
    REQUIRE(dev_ptr && offset >= 0, PYG_ERR_INVALID_ARGUMENT, "ipc_close: bad args");
    return ipc_close_impl(dev_ptr, offset);
}

pyg_status_t pyg_halo_push(const float* x, int64_t n_x, int64_t F, int64_t ldx, const int64_t* send_rows,
                           const int64_t* send_ptr, void* const* dst, const int64_t* dst_row, int64_t ldd, int n_peers,
                           void* stream) {
    REQUIRE(n_x >= 0 && F >= 0 && n_peers >= 0, PYG_ERR_INVALID_ARGUMENT, "halo_push: negative size");
    REQUIRE(ldx >= F && ldd >= F, PYG_ERR_DIMENSION, "halo_push: leading dimension < F");
    REQUIRE(n_peers == 0 || (send_ptr && dst && dst_row), PYG_ERR_INVALID_ARGUMENT, "halo_push: null host array");
    for (int q = 0; q < n_peers; ++q)
        REQUIRE(send_ptr[q] <= send_ptr[q + 1] && (send_ptr[q] == send_ptr[q + 1] || dst[q]) && dst_row[q] >= 0,
                PYG_ERR_INVALID_ARGUMENT, "halo_push: bad peer %d", q);
    REQUIRE(n_peers == 0 || send_ptr[n_peers] == 0 || (x && send_rows), PYG_ERR_INVALID_ARGUMENT,
            "halo_push: null x / send_rows");
    return halo_push_impl(x, ldx, F, send_rows, send_ptr, dst, dst_row, ldd, n_peers, as_stream(stream));
}

pyg_status_t pyg_peer_signal(uint32_t* const* flags, int n, uint32_t value, void* stream) {
    REQUIRE(n >= 0 && (n == 0 || flags), PYG_ERR_INVALID_ARGUMENT, "peer_signal: bad flags");
    for (int i = 0; i < n; ++i) REQUIRE(flags[i], PYG_ERR_INVALID_ARGUMENT, "peer_signal: null flag %d", i);
    return peer_flags_impl(flags, n, value, 0, as_stream(stream));
}

pyg_status_t pyg_peer_wait(uint32_t* const* flags, int n, uint32_t value, void* stream) {
    REQUIRE(n >= 0 && (n == 0 || flags), PYG_ERR_INVALID_ARGUMENT, "peer_wait: bad flags");
    for (int i = 0; i < n; ++i) REQUIRE(flags[i], PYG_ERR_INVALID_ARGUMENT, "peer_wait: null flag %d", i);
    return peer_flags_impl(flags, n, value, 1, as_stream(stream));
}

pyg_status_t pyg_gather_rows(const float* x, int64_t n_x, int64_t F, int64_t ldx, const int64_t* rows, int64_t n,
                             uint32_t flags, float* out, int64_t ldo, void* stream) {
    REQUIRE(n_x >= 0 && F >= 0 && n >= 0, PYG_ERR_INVALID_ARGUMENT, "gather_rows: negative size");
    REQUIRE(ldx >= F && ldo >= F, PYG_ERR_DIMENSION, "gather_rows: leading dimension < F");
    REQUIRE(n * F == 0 || (x && rows && out), PYG_ERR_INVALID_ARGUMENT, "gather_rows: null pointer");
    cudaStream_t s = as_stream(stream);
    if (flags & PYG_VALIDATE) {
        validate_begin();
        PYG_TRY(validate_index(rows, n, 0, n_x, s));
        PYG_TRY(validate_flag_check(s, "gather_rows: row index out of range"));
    }
    return gather_rows_impl(x, ldx, F, rows, n, out, ldo, s);
}

pyg_status_t pyg_plan_export(const pyg_plan_t* p, int64_t* rowptr, int64_t* col, int64_t* perm, void* stream) {
    REQUIRE(p, PYG_ERR_INVALID_ARGUMENT, "plan_export: null plan");
    REQUIRE(!col || p->col, PYG_ERR_INVALID_ARGUMENT, "plan_export: plan has no col array");
    REQUIRE(p->parts.empty(), PYG_ERR_UNSUPPORTED, "plan_export: source-blocked plans have one CSR per block");
    return plan_export_impl(p, rowptr, col, perm, as_stream(stream));
}

pyg_status_t pyg_workspace_size(const pyg_plan_t* plan, int64_t E, int64_t n_out, int64_t F_out,
                                pyg_reduce_t reduce, uint32_t flags, size_t* bytes) {
    REQUIRE(bytes && E >= 0 && n_out >= 0 && F_out >= 0, PYG_ERR_INVALID_ARGUMENT, "workspace_size: bad args");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "workspace_size: bad reduce");
    size_t b;
    if (use_plan(plan, flags)) b = std::max(coo_deg_bytes(n_out), segment_ws_bytes(plan, F_out, (int)reduce));
    else b = coo_deg_bytes(n_out) + coo_ws_bytes(E, n_out, F_out, (int)reduce, n_out);  // n_src = n_out
    *bytes = b + 256;
    return PYG_OK;
}

pyg_status_t pyg_scatter(const float* src, int64_t E, int64_t F, int64_t lds, const int64_t* index, int64_t dim_size,
                         pyg_reduce_t reduce, uint32_t flags, float* out, int64_t ldo, int64_t* arg_out,
                         const pyg_plan_t* plan, void* ws, size_t ws_bytes, void* stream) {
    REQUIRE(E >= 0 && F >= 0 && dim_size >= 0, PYG_ERR_INVALID_ARGUMENT, "scatter: negative size");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "scatter: bad reduce");
    REQUIRE(lds >= F && ldo >= F, PYG_ERR_DIMENSION, "scatter: leading dimension < F");
    REQUIRE(E <= kMaxI32 && dim_size <= kMaxI32 && F <= kMaxI32, PYG_ERR_UNSUPPORTED, "scatter: sizes must be < 2^31");
    REQUIRE((E == 0 || F == 0 || src) && (E == 0 || index) && (dim_size * F == 0 || out), PYG_ERR_INVALID_ARGUMENT,
            "scatter: null pointer");
    REQUIRE(reduce != PYG_MAX || dim_size * F == 0 || arg_out, PYG_ERR_INVALID_ARGUMENT, "scatter: max needs arg_out");
    REQUIRE(!(flags & PYG_FORCE_SEGMENT) || plan, PYG_ERR_INVALID_ARGUMENT, "scatter: FORCE_SEGMENT without plan");
    cudaStream_t s = as_stream(stream);
    if (flags & PYG_VALIDATE) {
        validate_begin();
        PYG_TRY(validate_index(index, E, 0, dim_size, s));
        PYG_TRY(validate_flag_check(s, "scatter: index out of range"));
    }
    if (dim_size == 0 || F == 0) return PYG_OK;
    if (use_plan(plan, flags)) {
        REQUIRE(plan->n_rows == dim_size && (plan->col == nullptr || plan->E == 0), PYG_ERR_DIMENSION,
                "scatter: plan is not a scatter plan over dim_size rows");
        SegArgs a;
        a.X = src; a.ldx = lds; a.ncols = (int)F;
        a.rowptr = plan->rowptr;
        a.eid = plan->perm_identity ? nullptr : plan->perm;
        a.out = out; a.ldo = ldo; a.arg = arg_out; a.lda = ldo;
        a.n_rows = dim_size; a.E_sentinel = E;
        a.heavy_threshold = plan->heavy_threshold;
        return segment_reduce(a, reduce, plan, ws, ws_bytes, s);
    }
    CooArgs c;
    c.X = src; c.ldx = lds; c.ncols = (int)F;
    c.sidx = index;
    c.out = out; c.ldo = ldo;
    c.keys = reinterpret_cast<unsigned long long*>(arg_out); c.ldk = ldo;
    c.E = E; c.n_out = dim_size;
    return coo_reduce(c, reduce, ws, ws_bytes, s);
}

pyg_status_t pyg_scatter_backward(const float* grad_out, int64_t ldg, const int64_t* index, int64_t E, int64_t F,
                                  int64_t dim_size, pyg_reduce_t reduce, const int64_t* arg_out, const int32_t* deg,
                                  float* grad_src, int64_t lds, void* stream) {
    REQUIRE(E >= 0 && F >= 0 && dim_size >= 0, PYG_ERR_INVALID_ARGUMENT, "scatter_backward: negative size");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "scatter_backward: bad reduce");
    REQUIRE(ldg >= F && lds >= F, PYG_ERR_DIMENSION, "scatter_backward: leading dimension < F");
    REQUIRE(E <= kMaxI32 && F <= kMaxI32, PYG_ERR_UNSUPPORTED, "scatter_backward: sizes must be < 2^31");
    REQUIRE(E * F == 0 || (grad_out && index && grad_src), PYG_ERR_INVALID_ARGUMENT, "scatter_backward: null pointer");
    REQUIRE(reduce != PYG_MEAN || deg, PYG_ERR_INVALID_ARGUMENT, "scatter_backward: mean needs deg");
    REQUIRE(reduce != PYG_MAX || arg_out, PYG_ERR_INVALID_ARGUMENT, "scatter_backward: max needs arg_out");
    return edge_gather_grad(grad_out, ldg, index, E, (int)F, reduce, arg_out, ldg, deg, grad_src, lds,
                            as_stream(stream));
}

pyg_status_t pyg_propagate(const float* x_src, int64_t n_src, int64_t F, int64_t ldx, const float* x_dst, int64_t ldxd,
                           int64_t n_dst, const int64_t* edge_index, int64_t E, const float* edge_attr, int64_t D,
                           int64_t lde, const float* edge_weight, pyg_reduce_t reduce, uint32_t flags, float* out,
                           int64_t ldo, int64_t* arg_out, const pyg_plan_t* plan, void* ws, size_t ws_bytes,
                           void* stream) {
    const bool cat = flags & PYG_PHI_CONCAT_XI;
    REQUIRE(n_src >= 0 && F >= 0 && n_dst >= 0 && E >= 0 && D >= 0, PYG_ERR_INVALID_ARGUMENT, "propagate: negative size");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "propagate: bad reduce");
    const int64_t F_out = (cat ? F : 0) + F + D;
    REQUIRE(ldx >= F && ldo >= F_out && (D == 0 || lde >= D), PYG_ERR_DIMENSION, "propagate: leading dimension too small");
    REQUIRE(!cat || x_dst || n_dst <= n_src, PYG_ERR_DIMENSION, "propagate: concat x_i with x_dst=NULL needs n_dst <= n_src");
    if (cat && x_dst) REQUIRE(ldxd >= F, PYG_ERR_DIMENSION, "propagate: ldxd < F");
    REQUIRE(E <= kMaxI32 && n_src <= kMaxI32 && n_dst <= kMaxI32 && F_out <= kMaxI32, PYG_ERR_UNSUPPORTED,
            "propagate: sizes must be < 2^31");
    REQUIRE(n_dst * F_out == 0 || out, PYG_ERR_INVALID_ARGUMENT, "propagate: null out");
    REQUIRE(reduce != PYG_MAX || n_dst * F_out == 0 || arg_out, PYG_ERR_INVALID_ARGUMENT, "propagate: max needs arg_out");
    REQUIRE(E == 0 || F == 0 || x_src, PYG_ERR_INVALID_ARGUMENT, "propagate: null x_src");
    REQUIRE(E == 0 || D == 0 || edge_attr, PYG_ERR_INVALID_ARGUMENT, "propagate: null edge_attr");
    REQUIRE(!(flags & PYG_FORCE_SEGMENT) || plan, PYG_ERR_INVALID_ARGUMENT, "propagate: FORCE_SEGMENT without plan");
    const bool seg = use_plan(plan, flags);
    REQUIRE(seg || E == 0 || edge_index, PYG_ERR_INVALID_ARGUMENT, "propagate: null edge_index without plan");
    cudaStream_t s = as_stream(stream);
    if ((flags & PYG_VALIDATE) && edge_index) {
        PYG_TRY(validate_index(edge_index, E, 0, n_src, s));
        PYG_TRY(validate_index(edge_index + E, E, 0, n_dst, s));
        PYG_TRY(validate_flag_check(s, "propagate: edge_index out of range"));
    }
    if (n_dst == 0 || F_out == 0) return PYG_OK;
    const float* xd = x_dst ? x_dst : x_src;  // (offset below for slices)
    const int64_t ldd = x_dst ? ldxd : ldx;
    const int64_t off1 = cat ? F : 0, off2 = off1 + F;

    if (seg) {
        REQUIRE(plan->n_rows == n_dst && (plan->col != nullptr || plan->E == 0) && plan->n_cols <= n_src, PYG_ERR_DIMENSION,
                "propagate: plan does not match (n_rows %lld vs n_dst %lld)", (long long)plan->n_rows, (long long)n_dst);
        const int32_t* eid = plan->perm_identity ? nullptr : plan->perm;
        if (cat && !x_dst && plan->row_offset > 0) {
            // a slice's output row r is global row row_offset + r: its x_i is x_src[row_offset + r]
            REQUIRE(plan->row_offset + n_dst <= n_src, PYG_ERR_DIMENSION,
                    "propagate: CONCAT_XI on a slice with x_dst = NULL needs row_offset + n_dst <= n_src");
            xd = x_src + plan->row_offset * ldx;
        }
        if (cat && !plan->parts.empty()) {
            REQUIRE(reduce != PYG_MAX, PYG_ERR_UNSUPPORTED, "propagate: CONCAT_XI + MAX needs an unblocked plan");
            REQUIRE(plan->n_passes == 0, PYG_ERR_UNSUPPORTED, "propagate: CONCAT_XI needs the whole plan, not a pass view");
            PYG_TRY(xi_block(xd, ldd, (int)F, n_dst, nullptr, nullptr, plan->deg, nullptr, reduce, out, ldo, arg_out,
                             ldo, E, s));
        } else if (cat) {
            PYG_TRY(xi_block(xd, ldd, (int)F, n_dst, plan->rowptr, eid, nullptr, nullptr, reduce, out, ldo, arg_out,
                             ldo, E, s));
        }
        if (F > 0) {
            SegArgs a;
            a.X = x_src; a.ldx = ldx; a.ncols = (int)F;
            a.rowptr = plan->rowptr; a.gidx = plan->col; a.eid = eid; a.w = edge_weight;
            a.out = out + off1; a.ldo = ldo; a.arg = arg_out ? arg_out + off1 : nullptr; a.lda = ldo;
            a.n_rows = n_dst; a.E_sentinel = E; a.heavy_threshold = plan->heavy_threshold;
            a.allow_pad_read = 1;
            a.flags = flags;
            PYG_TRY(segment_reduce(a, reduce, plan, ws, ws_bytes, s));
        }
        if (D > 0) {
            SegArgs a;
            a.X = edge_attr; a.ldx = lde; a.ncols = (int)D;
            a.rowptr = plan->rowptr; a.gidx = nullptr; a.eid = eid;
            a.out = out + off2; a.ldo = ldo; a.arg = arg_out ? arg_out + off2 : nullptr; a.lda = ldo;
            a.n_rows = n_dst; a.E_sentinel = E; a.heavy_threshold = plan->heavy_threshold;
            PYG_TRY(segment_reduce(a, reduce, plan, ws, ws_bytes, s));
        }
        return PYG_OK;
    }

    // atomic COO
    Carver cv(ws, ws_bytes);
    int32_t* deg = cv.take<int32_t>((size_t)n_dst);
    int32_t* first = cv.take<int32_t>((size_t)n_dst);
    const bool need_deg = cat || reduce == PYG_MEAN;
    if (need_deg) {
        REQUIRE(ws && cv.ok(), PYG_ERR_NO_MEMORY, "propagate: workspace too small (see pyg_workspace_size)");
        PYG_TRY(coo_degree(edge_index + E, E, n_dst, deg, (cat && reduce == PYG_MAX) ? first : nullptr, s));
    }
    if (cat) PYG_TRY(xi_block(xd, ldd, (int)F, n_dst, nullptr, nullptr, deg, first, reduce, out, ldo, arg_out, ldo, E, s));
    auto block = [&](const float* X, int64_t ld, int64_t nc, const int64_t* gidx, const float* w, int64_t off) -> pyg_status_t {
        CooArgs c;
        c.X = X; c.ldx = ld; c.ncols = (int)nc;
        c.gidx = gidx; c.sidx = edge_index + E; c.w = w;
        c.out = out + off; c.ldo = ldo;
        c.keys = arg_out ? reinterpret_cast<unsigned long long*>(arg_out + off) : nullptr; c.ldk = ldo;
        c.E = E; c.n_out = n_dst; c.n_src = gidx ? n_src : E;
        c.allow_pad_read = (X == x_src);
        c.deg = need_deg ? deg : nullptr;
        return coo_reduce(c, reduce, cv.rest(), cv.rest_bytes(), s);
    };
    if (F > 0) PYG_TRY(block(x_src, ldx, F, edge_index, edge_weight, off1));
    if (D > 0) PYG_TRY(block(edge_attr, lde, D, nullptr, nullptr, off2));
    return PYG_OK;
}

pyg_status_t pyg_propagate_backward(const float* x_src, int64_t n_src, int64_t F, int64_t ldx, int64_t n_dst,
                                    const int64_t* edge_index, int64_t E, int64_t D, const float* edge_weight,
                                    pyg_reduce_t reduce, uint32_t flags, const float* grad_out, int64_t ldg,
                                    const int64_t* arg_out, const int32_t* deg_dst, float* grad_x_src, int64_t ldgx,
                                    float* grad_x_dst, int64_t ldgxd, float* grad_edge_attr, int64_t ldge,
                                    float* grad_edge_weight, const pyg_plan_t* plan_T, void* ws, size_t ws_bytes,
                                    void* stream) {
    const bool cat = flags & PYG_PHI_CONCAT_XI;
    REQUIRE(n_src >= 0 && F >= 0 && n_dst >= 0 && E >= 0 && D >= 0, PYG_ERR_INVALID_ARGUMENT,
            "propagate_backward: negative size");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "propagate_backward: bad reduce");
    const int64_t F_out = (cat ? F : 0) + F + D;
    REQUIRE(ldg >= F_out, PYG_ERR_DIMENSION, "propagate_backward: ldg < F_out");
    REQUIRE(E <= kMaxI32 && n_src <= kMaxI32 && n_dst <= kMaxI32 && F_out <= kMaxI32, PYG_ERR_UNSUPPORTED,
            "propagate_backward: sizes must be < 2^31");
    REQUIRE(n_dst * F_out == 0 || grad_out, PYG_ERR_INVALID_ARGUMENT, "propagate_backward: null grad_out");
    REQUIRE(E == 0 || edge_index, PYG_ERR_INVALID_ARGUMENT, "propagate_backward: null edge_index");
    REQUIRE(reduce != PYG_MAX || n_dst * F_out == 0 || arg_out, PYG_ERR_INVALID_ARGUMENT,
            "propagate_backward: max needs arg_out");
    REQUIRE(!(reduce == PYG_MEAN || (cat && reduce == PYG_SUM && grad_x_dst)) || deg_dst || n_dst == 0,
            PYG_ERR_INVALID_ARGUMENT, "propagate_backward: deg_dst required");
    cudaStream_t s = as_stream(stream);
    if (flags & PYG_VALIDATE) {
        validate_begin();
        PYG_TRY(validate_index(edge_index, E, 0, n_src, s));
        PYG_TRY(validate_index(edge_index + E, E, 0, n_dst, s));
        PYG_TRY(validate_flag_check(s, "propagate_backward: edge_index out of range"));
    }
    const int64_t off1 = cat ? F : 0, off2 = off1 + F;
    const int64_t* src = edge_index;
    const int64_t* dst = edge_index ? edge_index + E : nullptr;
    const int64_t* argx = arg_out ? arg_out + off1 : nullptr;

    if (cat && grad_x_dst) {
        REQUIRE(ldgxd >= F, PYG_ERR_DIMENSION, "propagate_backward: ldgxd < F");
        PYG_TRY(xdst_grad(grad_out, ldg, (int)F, n_dst, deg_dst, arg_out, ldg, E, reduce, grad_x_dst, ldgxd, s));
    }
    if (grad_x_src && F > 0 && n_src > 0) {
        REQUIRE(ldgx >= F, PYG_ERR_DIMENSION, "propagate_backward: ldgx < F");
        if (reduce == PYG_MAX) {
            PYG_TRY(fill_rows(grad_x_src, ldgx, (int)F, n_src, s));
            PYG_TRY(max_route_grad(grad_out + off1, ldg, argx, ldg, (int)F, n_dst, src, edge_weight, E, grad_x_src,
                                   ldgx, s));
        } else if (use_plan(plan_T, flags)) {
            REQUIRE(plan_T->n_rows == n_src && (plan_T->col != nullptr || plan_T->E == 0) && plan_T->n_cols <= n_dst, PYG_ERR_DIMENSION,
                    "propagate_backward: plan_T must be built with row_index = sources, col_index = targets");
            SegArgs a;
            a.X = grad_out + off1; a.ldx = ldg; a.ncols = (int)F;
            a.rowptr = plan_T->rowptr; a.gidx = plan_T->col;
            a.eid = plan_T->perm_identity ? nullptr : plan_T->perm;
            a.w = edge_weight; a.gdeg = reduce == PYG_MEAN ? deg_dst : nullptr;
            a.out = grad_x_src; a.ldo = ldgx; a.n_rows = n_src; a.E_sentinel = E;
            a.heavy_threshold = plan_T->heavy_threshold;
            PYG_TRY(segment_reduce(a, PYG_SUM, plan_T, ws, ws_bytes, s));
        } else {
            CooArgs c;
            c.X = grad_out + off1; c.ldx = ldg; c.ncols = (int)F;
            c.gidx = dst; c.sidx = src; c.w = edge_weight; c.gdeg = reduce == PYG_MEAN ? deg_dst : nullptr;
            c.out = grad_x_src; c.ldo = ldgx; c.E = E; c.n_out = n_src; c.n_src = n_dst;
            PYG_TRY(coo_reduce(c, PYG_SUM, ws, ws_bytes, s));
        }
    }
    if (grad_edge_attr && D > 0) {
        REQUIRE(ldge >= D, PYG_ERR_DIMENSION, "propagate_backward: ldge < D");
        PYG_TRY(edge_gather_grad(grad_out + off2, ldg, dst, E, (int)D, reduce, arg_out ? arg_out + off2 : nullptr, ldg,
                                 deg_dst, grad_edge_attr, ldge, s));
    }
    if (grad_edge_weight) {
        REQUIRE(x_src && ldx >= F, PYG_ERR_INVALID_ARGUMENT, "propagate_backward: grad_edge_weight needs x_src");
        PYG_TRY(edge_weight_grad(x_src, ldx, grad_out + off1, ldg, argx, ldg, edge_index, E, (int)F, reduce, deg_dst,
                                 grad_edge_weight, s));
    }
    return PYG_OK;
}

pyg_status_t pyg_gcn_norm_workspace_size(int64_t E, int64_t N, size_t* bytes) {
    REQUIRE(bytes && E >= 0 && N >= 0, PYG_ERR_INVALID_ARGUMENT, "gcn_norm_workspace_size: bad args");
    return gcn_norm_impl(nullptr, E, N, nullptr, nullptr, nullptr, nullptr, nullptr, 0, nullptr, bytes);
}

pyg_status_t pyg_gcn_norm(const int64_t* edge_index, int64_t E, int64_t N, const float* edge_weight, uint32_t flags,
                          int64_t* edge_index_out, float* weight_out, int64_t* E_out, void* ws, size_t bytes,
                          void* stream) {
    REQUIRE(E >= 0 && N >= 0 && E_out, PYG_ERR_INVALID_ARGUMENT, "gcn_norm: bad args");
    REQUIRE(E + N == 0 || (edge_index_out && weight_out), PYG_ERR_INVALID_ARGUMENT, "gcn_norm: null output");
    REQUIRE(E == 0 || edge_index, PYG_ERR_INVALID_ARGUMENT, "gcn_norm: null edge_index");
    REQUIRE(E + N <= kMaxI32, PYG_ERR_UNSUPPORTED, "gcn_norm: sizes must be < 2^31");
    cudaStream_t s = as_stream(stream);
    if (flags & PYG_VALIDATE) {
        validate_begin();
        PYG_TRY(validate_index(edge_index, 2 * E, 0, N, s));
        PYG_TRY(validate_flag_check(s, "gcn_norm: edge_index out of range"));
    }
    return gcn_norm_impl(edge_index, E, N, edge_weight, edge_index_out, weight_out, E_out, ws, bytes, s, nullptr);
}

pyg_status_t pyg_collate(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr, const int64_t* local_edge_index,
                         int64_t E_total, int64_t N_total, uint32_t flags, int64_t* edge_index, int64_t* batch,
                         int64_t* node_ptr, void* stream) {
    REQUIRE(G > 0, PYG_ERR_INVALID_ARGUMENT, "collate: empty list of graphs (G <= 0)");
    REQUIRE(E_total >= 0 && N_total >= 0, PYG_ERR_INVALID_ARGUMENT, "collate: negative size");
    REQUIRE(num_nodes && edge_ptr && node_ptr, PYG_ERR_INVALID_ARGUMENT, "collate: null pointer");
    REQUIRE(E_total == 0 || (local_edge_index && edge_index), PYG_ERR_INVALID_ARGUMENT, "collate: null edge arrays");
    REQUIRE(N_total == 0 || batch, PYG_ERR_INVALID_ARGUMENT, "collate: null batch");
    return collate_impl(G, num_nodes, edge_ptr, local_edge_index, E_total, N_total, flags, edge_index, batch, node_ptr,
                        as_stream(stream));
}

pyg_status_t pyg_global_pool(const float* x, int64_t N, int64_t F, int64_t ldx, const int64_t* node_ptr, int64_t G,
                             pyg_reduce_t reduce, float* out, int64_t ldo, int64_t* arg_out, void* stream) {
    REQUIRE(N >= 0 && F >= 0 && G >= 0, PYG_ERR_INVALID_ARGUMENT, "global_pool: negative size");
    REQUIRE(reduce >= PYG_SUM && reduce <= PYG_MAX, PYG_ERR_INVALID_ARGUMENT, "global_pool: bad reduce");
    REQUIRE(ldx >= F && ldo >= F, PYG_ERR_DIMENSION, "global_pool: leading dimension < F");
    REQUIRE(N <= kMaxI32 && F <= kMaxI32, PYG_ERR_UNSUPPORTED, "global_pool: sizes must be < 2^31");
    REQUIRE(G * F == 0 || (out && node_ptr), PYG_ERR_INVALID_ARGUMENT, "global_pool: null pointer");
    REQUIRE(reduce != PYG_MAX || G * F == 0 || arg_out, PYG_ERR_INVALID_ARGUMENT, "global_pool: max needs arg_out");
    if (G == 0 || F == 0) return PYG_OK;
    return global_pool_impl(x, ldx, (int)F, node_ptr, G, reduce, out, ldo, arg_out, N, as_stream(stream));
}

// ---- NEXT-1: segment softmax + GAT attention aggregation (attention.cu) ----------

static bool scatter_plan_ok(const pyg_plan* p, int64_t n, int64_t E) {
    return p && p->n_rows == n && p->col == nullptr && p->parts.empty() && p->E == E;
}

pyg_status_t pyg_segment_softmax(const float* src, int64_t E, int64_t H, int64_t lds, const int64_t* index,
                                 int64_t dim_size, const pyg_plan_t* plan, float* out, int64_t ldo, void* stream) {
    (void)index;
    REQUIRE(E >= 0 && H >= 0 && dim_size >= 0, PYG_ERR_INVALID_ARGUMENT, "segment_softmax: negative size");
    REQUIRE(lds >= H && ldo >= H, PYG_ERR_DIMENSION, "segment_softmax: leading dimension < H");
    REQUIRE(H <= kAttnMaxHeads, PYG_ERR_UNSUPPORTED, "segment_softmax: at most %d columns", kAttnMaxHeads);
    REQUIRE(scatter_plan_ok(plan, dim_size, E), PYG_ERR_DIMENSION,
            "segment_softmax: needs an unblocked scatter plan over dim_size rows and E edges");
    REQUIRE(E * H == 0 || (src && out), PYG_ERR_INVALID_ARGUMENT, "segment_softmax: null pointer");
    if (E == 0 || H == 0) return PYG_OK;
    return attention_softmax(plan, nullptr, plan->perm_identity ? nullptr : plan->perm, src, lds, nullptr, nullptr,
                             (int)H, 0.0f, out, ldo, as_stream(stream));
}

pyg_status_t pyg_segment_softmax_backward(const float* out, int64_t ldo, const float* grad_out, int64_t ldg, int64_t E,
                                          int64_t H, int64_t dim_size, const pyg_plan_t* plan, float* grad_src,
                                          int64_t lds, void* stream) {
    REQUIRE(E >= 0 && H >= 0 && dim_size >= 0, PYG_ERR_INVALID_ARGUMENT, "segment_softmax_backward: negative size");
    REQUIRE(ldo >= H && ldg >= H && lds >= H, PYG_ERR_DIMENSION, "segment_softmax_backward: leading dimension < H");
    REQUIRE(H <= kAttnMaxHeads, PYG_ERR_UNSUPPORTED, "segment_softmax_backward: at most %d columns", kAttnMaxHeads);
    REQUIRE(scatter_plan_ok(plan, dim_size, E), PYG_ERR_DIMENSION,
            "segment_softmax_backward: needs the scatter plan of the forward");
    REQUIRE(E * H == 0 || (out && grad_out && grad_src), PYG_ERR_INVALID_ARGUMENT,
            "segment_softmax_backward: null pointer");
    if (E == 0 || H == 0) return PYG_OK;
    return attention_softmax_bwd(plan, nullptr, plan->perm_identity ? nullptr : plan->perm, (int)H, 1, (int)H, out, ldo,
                                 grad_out, ldg, nullptr, 0, nullptr, nullptr, 0.0f, grad_src, lds, nullptr,
                                 as_stream(stream));
}

// alpha-weighted sum over a plan (forward: X = z over the forward plan; grad_z: X = grad_out
// over the transposed plan): the segment-reduce in mode kRedHeadW
static pyg_status_t headw_sum(const pyg_plan* p, const float* X, int64_t ldx, int64_t F, int64_t C, int64_t H,
                              const float* alpha, float* out, int64_t ldo, int64_t n_rows, void* ws, size_t ws_bytes,
                              cudaStream_t s) {
    SegArgs a;
    a.X = X; a.ldx = ldx; a.ncols = (int)F;
    a.rowptr = p->rowptr; a.gidx = p->col; a.eid = p->perm_identity ? nullptr : p->perm;
    a.out = out; a.ldo = ldo; a.n_rows = n_rows; a.E_sentinel = p->E;
    a.heavy_threshold = p->heavy_threshold;
    a.hw = alpha; a.hH = (int)H; a.hC = (int)C;
    return segment_reduce(a, kRedHeadW, p, ws, ws_bytes, s);
}

pyg_status_t pyg_gat_propagate_workspace_size(const pyg_plan_t* plan, int64_t H, int64_t C, size_t* bytes) {
    REQUIRE(bytes && plan && H > 0 && C >= 0, PYG_ERR_INVALID_ARGUMENT, "gat_propagate_workspace_size: bad args");
    *bytes = plan->parts.empty() ? std::max(gat_fwd_tma_ws_bytes(plan, H, H * C), segment_ws_bytes(plan, H * C, PYG_SUM))
                                 : gat_fwd_blocked_ws_bytes(plan, H);
    return PYG_OK;
}

pyg_status_t pyg_gat_propagate(const float* z, int64_t n_src, int64_t H, int64_t C, int64_t ldz, const float* s_src,
                               const float* s_dst, int64_t n_dst, int64_t E, float negative_slope,
                               const pyg_plan_t* plan, float* out, int64_t ldo, float* alpha, float* row_sums,
                               void* ws, size_t ws_bytes, void* stream) {
    REQUIRE(n_src >= 0 && H > 0 && C >= 0 && n_dst >= 0 && E >= 0, PYG_ERR_INVALID_ARGUMENT,
            "gat_propagate: bad sizes");
    const int64_t F = H * C;
    REQUIRE(ldz >= F && ldo >= F, PYG_ERR_DIMENSION, "gat_propagate: leading dimension < H*C");
    REQUIRE(F <= 16384 && H <= kAttnMaxHeads, PYG_ERR_UNSUPPORTED, "gat_propagate: H <= %d", kAttnMaxHeads);
    REQUIRE(plan && plan->n_rows == n_dst && (plan->col || plan->E == 0) && plan->n_cols <= n_src && plan->E == E,
            PYG_ERR_DIMENSION, "gat_propagate: needs a forward plan over n_dst rows and E edges");
    REQUIRE(n_dst * F == 0 || out, PYG_ERR_INVALID_ARGUMENT, "gat_propagate: null out");
    REQUIRE(E == 0 || (z && s_src && s_dst && alpha), PYG_ERR_INVALID_ARGUMENT, "gat_propagate: null input");
    cudaStream_t s = as_stream(stream);
    if (!plan->parts.empty()) {  // source-blocked plan: one L2-resident pass per block of z rows
        REQUIRE(plan->n_passes == 0 || plan->n_passes == (int64_t)plan->parts.size(), PYG_ERR_UNSUPPORTED,
                "gat_propagate: needs the whole source-blocked plan, not a pass view");
        if (n_dst == 0 || F == 0) return PYG_OK;
        return gat_fwd_blocked(plan, (int)H, (int)C, (int)F, z, n_src, ldz, s_src, s_dst, negative_slope, out, ldo,
                               alpha, row_sums, ws, ws_bytes, s);
    }
    if (E > 0 && n_dst > 0 && gat_fwd_tma_eligible(plan, (int)H, (int)C, (int)F, z, ldz, out, ldo, alpha, s_src, s_dst))
        // softmax with a per-row shift bounded from the global max of s_src + the weighted sum, one pass
        return gat_fwd_tma(plan, (int)H, (int)C, (int)F, z, n_src, ldz, s_src, s_dst, negative_slope, out, ldo, alpha,
                           row_sums, ws, ws_bytes, s);
    if (E > 0)
        PYG_TRY(attention_softmax(plan, plan->col, plan->perm_identity ? nullptr : plan->perm, nullptr, 0, s_src, s_dst,
                                  (int)H, negative_slope, alpha, H, s));
    if (row_sums && n_dst > 0) PYG_TRY(fill_const(row_sums, n_dst * H, 1.0f, s));  // alpha is normalised here
    if (n_dst == 0 || F == 0) return PYG_OK;
    return headw_sum(plan, z, ldz, F, C, H, alpha, out, ldo, n_dst, ws, ws_bytes, s);
}

static size_t gat_bwd_ws_main(const pyg_plan* plan, const pyg_plan* plan_T, int64_t H, int64_t C) {
    return align_up(std::max(gat_bwd_tma_ws_bytes(plan, H), segment_ws_bytes(plan_T, H * C, PYG_SUM)), 256);
}

pyg_status_t pyg_gat_backward_workspace_size(const pyg_plan_t* plan, const pyg_plan_t* plan_T, int64_t H, int64_t C,
                                             int with_row_sums, size_t* bytes) {
    REQUIRE(bytes && plan && plan_T && H > 0 && C >= 0, PYG_ERR_INVALID_ARGUMENT, "gat_backward_workspace_size: bad args");
    // + grad_out scaled by 1 / row_sums per head (the alpha-weighted grad_z with unnormalised alpha)
    *bytes = gat_bwd_ws_main(plan, plan_T, H, C) + (with_row_sums ? (size_t)plan->n_rows * H * C * 4 : 0);
    return PYG_OK;
}

pyg_status_t pyg_gat_backward(const float* z, int64_t n_src, int64_t H, int64_t C, int64_t ldz, const float* s_src,
                              const float* s_dst, int64_t n_dst, int64_t E, float negative_slope, const float* alpha,
                              const float* row_sums, const float* grad_out, int64_t ldg, const float* out, int64_t ldo,
                              const pyg_plan_t* plan,
                              const pyg_plan_t* plan_T, float* grad_z, int64_t ldgz, float* grad_s_src,
                              float* grad_s_dst, float* grad_logit, void* ws, size_t ws_bytes, void* stream) {
    REQUIRE(n_src >= 0 && H > 0 && C >= 0 && n_dst >= 0 && E >= 0, PYG_ERR_INVALID_ARGUMENT,
            "gat_backward: bad sizes");
    const int64_t F = H * C;
    REQUIRE(ldz >= F && ldg >= F && (!grad_z || ldgz >= F), PYG_ERR_DIMENSION, "gat_backward: leading dimension < H*C");
    REQUIRE(F <= 4096 && H <= kAttnMaxHeads, PYG_ERR_UNSUPPORTED, "gat_backward: H*C <= 4096 and H <= %d",
            kAttnMaxHeads);
    REQUIRE(plan && plan->n_rows == n_dst && (plan->col || plan->E == 0) && plan->parts.empty() && plan->E == E,
            PYG_ERR_DIMENSION, "gat_backward: `plan` must be the forward plan");
    // plan_T may be source-blocked (blocks of grad_out rows): grad_z and grad_s_src are segment sums over it,
    // one L2-resident pass per block when grad_out exceeds L2
    REQUIRE(plan_T && plan_T->n_rows == n_src && (plan_T->col || plan_T->E == 0) && plan_T->n_cols <= n_dst &&
                plan_T->E == E && (plan_T->parts.empty() || plan_T->n_passes == 0 ||
                                   plan_T->n_passes == (int64_t)plan_T->parts.size()),
            PYG_ERR_DIMENSION, "gat_backward: plan_T must be built with row_index = sources, col_index = targets "
                               "(whole plan, not a pass view)");
    REQUIRE(E == 0 || (z && s_src && s_dst && alpha && grad_out && grad_logit), PYG_ERR_INVALID_ARGUMENT,
            "gat_backward: null input (grad_logit [E x H] is required)");
    REQUIRE(n_dst * H == 0 || grad_s_dst, PYG_ERR_INVALID_ARGUMENT, "gat_backward: null grad_s_dst");
    REQUIRE(!out || ldo >= F, PYG_ERR_DIMENSION, "gat_backward: ldo < H*C");
    cudaStream_t s = as_stream(stream);
    // row_sums (the forward's factored alpha): grad_z = sum_i p_ij g_i / row_sums_i takes grad_out
    // scaled per row and head, kept behind the main workspace
    float* gsc = nullptr;
    const size_t main_ws = gat_bwd_ws_main(plan, plan_T, H, C);
    if (row_sums && n_dst > 0 && F > 0) {
        REQUIRE(ws && ws_bytes >= main_ws + (size_t)n_dst * F * 4, PYG_ERR_NO_MEMORY,
                "gat_backward: workspace too small (pyg_gat_backward_workspace_size with row_sums)");
        gsc = reinterpret_cast<float*>(static_cast<char*>(ws) + main_ws);
    }
    if (E > 0 && gat_bwd_tma_eligible(plan, (int)H, (int)C, (int)F, z, ldz, grad_out, ldg, out, ldo, alpha, s_src, s_dst,
                                      grad_s_dst)) {
        // one pass: SDDMM + softmax backward with t_i = g_i . out_i (gat_tma.cu)
        PYG_TRY(gat_bwd_tma(plan, (int)H, (int)C, (int)F, z, n_src, ldz, grad_out, ldg, out, ldo, alpha, row_sums, s_src,
                            s_dst, negative_slope, grad_logit, grad_s_dst, gsc, ws, main_ws, s));
    } else {
        if (n_dst > 0) PYG_TRY(fill_rows(grad_s_dst, H, (int)H, n_dst, s));  // rows without in-edges
        if (E > 0)
            PYG_TRY(attention_softmax_bwd(plan, plan->col, plan->perm_identity ? nullptr : plan->perm, (int)H, (int)C,
                                          (int)F, alpha, H, grad_out, ldg, z, ldz, s_src, s_dst, negative_slope,
                                          grad_logit, H, grad_s_dst, s, row_sums));
        if (gsc) PYG_TRY(gat_scale_rows(grad_out, ldg, n_dst, (int)H, (int)C, row_sums, gsc, s));
    }
    if (grad_z && n_src > 0 && F > 0) {
        if (gsc) PYG_TRY(headw_sum(plan_T, gsc, F, F, C, H, alpha, grad_z, ldgz, n_src, ws, main_ws, s));
        else PYG_TRY(headw_sum(plan_T, grad_out, ldg, F, C, H, alpha, grad_z, ldgz, n_src, ws, ws_bytes, s));
    }
    if (grad_s_src && n_src > 0) {
        SegArgs a;
        a.X = grad_logit; a.ldx = H; a.ncols = (int)H;
        a.rowptr = plan_T->rowptr; a.gidx = plan_T->perm; a.eid = nullptr;
        a.out = grad_s_src; a.ldo = H; a.n_rows = n_src; a.E_sentinel = E;
        a.heavy_threshold = plan_T->heavy_threshold;
        a.flags = PYG_NO_TMA;
        PYG_TRY(segment_reduce(a, PYG_SUM, plan_T, ws, ws_bytes, s));
    }
    return PYG_OK;
}

// ---- NEXT-2: K-step propagation (APPNP / SGC) reusing one plan -------------------

pyg_status_t pyg_appnp(const float* h, int64_t n, int64_t F, int64_t ldh, const float* edge_weight, int64_t K,
                       float alpha, const pyg_plan_t* plan, float* out, int64_t ldo, float* scratch, void* ws,
                       size_t ws_bytes, void* stream) {
    REQUIRE(n >= 0 && F >= 0 && K >= 0, PYG_ERR_INVALID_ARGUMENT, "appnp: negative size");
    REQUIRE(alpha >= 0.0f && alpha <= 1.0f, PYG_ERR_INVALID_ARGUMENT, "appnp: alpha outside [0, 1]");
    REQUIRE(ldh >= F && ldo >= F, PYG_ERR_DIMENSION, "appnp: leading dimension < F");
    REQUIRE(n <= kMaxI32 && F <= kMaxI32, PYG_ERR_UNSUPPORTED, "appnp: sizes must be < 2^31");
    REQUIRE(n * F == 0 || (h && out), PYG_ERR_INVALID_ARGUMENT, "appnp: null pointer");
    REQUIRE(K <= 1 || scratch, PYG_ERR_INVALID_ARGUMENT, "appnp: K > 1 needs scratch [n x F] (stride ldo)");
    REQUIRE(plan && plan->n_rows == n && plan->n_cols <= n && (plan->col || plan->E == 0), PYG_ERR_DIMENSION,
            "appnp: needs a forward plan over n targets and n sources");
    cudaStream_t s = as_stream(stream);
    if (n == 0 || F == 0) return PYG_OK;
    if (K == 0) {
        PYG_CUDA(cudaMemcpy2DAsync(out, (size_t)ldo * 4, h, (size_t)ldh * 4, (size_t)F * 4, (size_t)n,
                                   cudaMemcpyDeviceToDevice, s));
        return PYG_OK;
    }
    const int32_t* eid = plan->perm_identity ? nullptr : plan->perm;
    const float* wk = edge_weight;
    // the K steps read the same weights in the same plan order: with room in the workspace they are
    // gathered into position order once (w_pos[p] = w[perm[p]]), so every step streams 4 bytes per
    // position instead of an edge id plus a random 32-byte sector of w
    const size_t seg_need = segment_ws_bytes(plan, F, PYG_SUM) + 256;
    if (edge_weight && eid && plan->E > 0 && ws && ws_bytes >= seg_need + (size_t)plan->E * 4 + 256) {
        float* w_pos = reinterpret_cast<float*>(static_cast<char*>(ws) + align_up(seg_need, 256));
        PYG_TRY(gather_by_index(edge_weight, eid, plan->E, w_pos, s));
        wk = w_pos;
        eid = nullptr;  // SUM reads edge ids only for the weights
    }
    const float* z = h;
    int64_t ldz = ldh;
    for (int64_t k = 0; k < K; ++k) {
        // the last iteration writes `out`; earlier ones alternate so that they never read what they write
        float* dst = ((K - 1 - k) % 2 == 0) ? out : scratch;
        SegArgs a;
        a.X = z; a.ldx = ldz; a.ncols = (int)F;
        a.rowptr = plan->rowptr; a.gidx = plan->col; a.eid = eid; a.w = wk;
        a.out = dst; a.ldo = ldo; a.n_rows = n; a.E_sentinel = plan->E;
        a.heavy_threshold = plan->heavy_threshold; a.allow_pad_read = 1;
        a.blend = alpha != 0.0f ? h : nullptr; a.ldb = ldh;
        a.blend_a = 1.0f - alpha; a.blend_b = alpha;
        PYG_TRY(segment_reduce(a, PYG_SUM, plan, ws, ws_bytes, s));
        z = dst;
        ldz = ldo;
    }
    return PYG_OK;
}

// ---- NEXT-2: dense feature transform on tcgen05 (transform.cu) -------------------------

pyg_status_t pyg_dense_transform(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W, int64_t N,
                                 int64_t ldw, const float* bias, const float* row_scale, float* Y, int64_t ldy,
                                 void* stream) {
    REQUIRE(M >= 0 && K >= 1 && N >= 0, PYG_ERR_INVALID_ARGUMENT, "dense_transform: bad sizes (K >= 1)");
    REQUIRE(ldx >= K && ldw >= K && ldy >= N, PYG_ERR_DIMENSION, "dense_transform: leading dimension too small");
    REQUIRE(N <= 65535LL * 256, PYG_ERR_UNSUPPORTED, "dense_transform: F_out too large");
    REQUIRE(M <= kMaxI32 && K <= kMaxI32, PYG_ERR_UNSUPPORTED, "dense_transform: sizes must be < 2^31");
    REQUIRE(M * N == 0 || (X && W && Y), PYG_ERR_INVALID_ARGUMENT, "dense_transform: null pointer");
    REQUIRE((reinterpret_cast<uintptr_t>(X) % 16 == 0) && (reinterpret_cast<uintptr_t>(W) % 16 == 0) &&
                (ldx % 4 == 0) && (ldw % 4 == 0),
            PYG_ERR_ALIGNMENT, "dense_transform: X and W must be 16-byte aligned with ld %% 4 == 0 (TMA)");
    return dense_transform_impl(X, M, K, ldx, W, N, ldw, bias, row_scale, Y, ldy, as_stream(stream));
}

// GCN layer: out = D^-1/2 (A+I) D^-1/2 X W^T + b, with the normalisation fused into the
// epilogues: the transform scales its rows by D^-1/2 and the unweighted aggregation over A+I scales
// its output rows by D^-1/2 and adds b -- no per-edge weights are read.
static void gcn_layer_layout(const pyg_plan* plan, int64_t n, int64_t F_out, Carver& cv, float** dinv, float** H,
                             int64_t* ldh, void** seg_ws, size_t* seg_bytes) {
    *dinv = cv.take<float>((size_t)std::max<int64_t>(n, 1));
    *ldh = (int64_t)align_up((size_t)std::max<int64_t>(F_out, 1), 8);
    *H = cv.take<float>((size_t)std::max<int64_t>(n, 1) * (size_t)*ldh);
    const size_t sb = segment_ws_bytes(plan, F_out, PYG_SUM) + 256;
    *seg_ws = cv.take<char>(sb);
    *seg_bytes = sb;
}

pyg_status_t pyg_gcn_layer_workspace_size(const pyg_plan_t* plan, int64_t n, int64_t F_out, size_t* bytes) {
    REQUIRE(plan && bytes && n >= 0 && F_out >= 0, PYG_ERR_INVALID_ARGUMENT, "gcn_layer_workspace_size: bad args");
    Carver cv(nullptr, 0);
    float *dinv, *H;
    int64_t ldh;
    void* sw;
    size_t sb;
    gcn_layer_layout(plan, n, F_out, cv, &dinv, &H, &ldh, &sw, &sb);
    *bytes = cv.off + 256;
    return PYG_OK;
}

pyg_status_t pyg_gcn_layer(const float* X, int64_t n, int64_t K, int64_t ldx, const float* W, int64_t F_out,
                           int64_t ldw, const float* bias, const pyg_plan_t* plan, float* out, int64_t ldo, void* ws,
                           size_t ws_bytes, void* stream) {
    REQUIRE(n >= 0 && K >= 1 && F_out >= 0, PYG_ERR_INVALID_ARGUMENT, "gcn_layer: bad sizes");
    REQUIRE(ldo >= F_out, PYG_ERR_DIMENSION, "gcn_layer: ldo < F_out");
    REQUIRE(plan && plan->n_rows == n && plan->n_cols <= n && (plan->col || plan->E == 0), PYG_ERR_DIMENSION,
            "gcn_layer: needs a forward plan over n nodes (edges incl. self-loops, e.g. from pyg_gcn_norm)");
    REQUIRE(n * F_out == 0 || out, PYG_ERR_INVALID_ARGUMENT, "gcn_layer: null out");
    Carver cv(ws, ws_bytes);
    float *dinv, *H;
    int64_t ldh;
    void* sw;
    size_t sb;
    gcn_layer_layout(plan, n, F_out, cv, &dinv, &H, &ldh, &sw, &sb);
    REQUIRE(ws && cv.ok(), PYG_ERR_NO_MEMORY, "gcn_layer: workspace too small (pyg_gcn_layer_workspace_size)");
    if (n == 0 || F_out == 0) return PYG_OK;
    cudaStream_t s = as_stream(stream);
    // degrees of A+I: the plan's row lengths (source-blocked plans: the total in-degree they keep per row;
    // the aggregation then runs one L2-resident pass per source block and applies D^-1/2 and the bias in
    // the last pass)
    REQUIRE(plan->parts.empty() || plan->n_passes == 0, PYG_ERR_UNSUPPORTED, "gcn_layer: needs the whole plan, not a pass view");
    PYG_TRY(gcn_dinv(plan->rowptr, plan->parts.empty() ? nullptr : plan->deg, n, dinv, s));
    PYG_TRY(pyg_dense_transform(X, n, K, ldx, W, F_out, ldw, nullptr, dinv, H, ldh, stream));
    SegArgs a;
    a.X = H; a.ldx = ldh; a.ncols = (int)F_out;
    a.rowptr = plan->rowptr; a.gidx = plan->col; a.eid = nullptr;
    a.out = out; a.ldo = ldo; a.n_rows = n; a.E_sentinel = plan->E;
    a.heavy_threshold = plan->heavy_threshold; a.allow_pad_read = 1;
    a.row_scale = dinv; a.col_bias = bias;
    return segment_reduce(a, PYG_SUM, plan, sw, sb, s);
}

// GAT transform: z = X W^T on the tensor cores with the attention projections of every head fused
// into the epilogue ("z = xW; logit = leaky_relu([z_i || z_j] . a)")
pyg_status_t pyg_gat_transform(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W, int64_t H,
                               int64_t C, int64_t ldw, const float* att_src, const float* att_dst, float* Z, int64_t ldz,
                               float* s_src, float* s_dst, void* stream) {
    REQUIRE(M >= 0 && K >= 1 && H >= 1 && C >= 1, PYG_ERR_INVALID_ARGUMENT, "gat_transform: bad sizes");
    const int64_t N = H * C;
    REQUIRE(H <= kAttnMaxHeads && N <= 256, PYG_ERR_UNSUPPORTED, "gat_transform: H <= %d and H*C <= 256",
            kAttnMaxHeads);
    REQUIRE(ldx >= K && ldw >= K && ldz >= N, PYG_ERR_DIMENSION, "gat_transform: leading dimension too small");
    REQUIRE(M == 0 || (X && W && Z && att_src && att_dst && s_src && s_dst), PYG_ERR_INVALID_ARGUMENT,
            "gat_transform: null pointer");
    REQUIRE((reinterpret_cast<uintptr_t>(X) % 16 == 0) && (reinterpret_cast<uintptr_t>(W) % 16 == 0) &&
                (ldx % 4 == 0) && (ldw % 4 == 0),
            PYG_ERR_ALIGNMENT, "gat_transform: X and W must be 16-byte aligned with ld %% 4 == 0 (TMA)");
    if (M == 0) return PYG_OK;
    return dense_transform_impl(X, M, K, ldx, W, N, ldw, nullptr, nullptr, Z, ldz, as_stream(stream), att_src,
                                att_dst, s_src, s_dst, (int)H);
}

}  // extern "C"
