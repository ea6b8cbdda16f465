// kernels.cuh -- internal launch interfaces of libpygs (not part of the ABI).
#pragma once

#include <vector>

#include "common.cuh"

// Host-side plan object (opaque in the ABI).
struct pyg_plan {
    int64_t n_rows = 0, n_cols = 0, E = 0, row_offset = 0;
    const int64_t* rowptr = nullptr;  // offset by row_offset for slices
    const int32_t* col = nullptr;     // [E] or null
    const int32_t* perm = nullptr;    // [E]
    int perm_identity = 0;
    // split hub rows ("heavy"): global arrays of the root plan
    const int32_t* heavy_rows = nullptr;      // [n_heavy_total] global row ids, ascending
    const int64_t* heavy_item_ptr = nullptr;  // [n_heavy_total + 1]
    std::vector<int32_t> h_heavy_rows;
    std::vector<int64_t> h_heavy_item_ptr;
    int64_t h_lo = 0, h_hi = 0;        // heavy rows of this plan: [h_lo, h_hi)
    int64_t item_lo = 0, item_hi = 0;  // chunks of this plan
    int32_t heavy_threshold = 0, chunk = 0;
    // Source-blocked plans: edges sorted by (source block, target, id); `parts[b]` is the
    // slice of virtual rows of source block b restricted to this plan's target rows.
    // Light rows are visited in descending degree bucket (floor log2) order, stable by row id:
    // a CTA's rows then have similar lengths and the longest go first (power-law graphs).
    const int32_t* row_order = nullptr;  // [order_len] root row ids, or null
    int64_t order_len = 0;
    // TMA-pipelined light rows: tasks are runs of consecutive light rows holding <= kTaskPositions
    // positions (cut at row boundaries and at every split hub row), so task t is the contiguous
    // position range [task_pos[2t], task_pos[2t+1]); pos_row maps a position to its root row.
    // Empty rows are the tail of row_order (from empty_begin) and are zero-filled separately.
    const int64_t* task_pos = nullptr;  // [2 * n_tasks]
    const int32_t* task_item = nullptr; // [n_tasks] split-row item id of a hub chunk task, -1 light
    const int32_t* pos_row = nullptr;   // [E]
    int64_t n_tasks = 0;
    int64_t n_light_tasks = 0;          // tasks [0, n_light_tasks) are light rows, the rest hub chunks
    int64_t empty_begin = 0, n_empty = 0;
    int64_t col_block = 0;            // source rows per block (0 = not blocked)
    int64_t pass_base = 0;            // pass views: global index of parts[0] among the source blocks
    int64_t n_passes = 0;             // total source blocks of the root plan (0: parts.size())
    const int32_t* deg = nullptr;     // [n_rows] total in-degree (blocked plans), offset like rowptr
    std::vector<pyg_plan> parts;
};

namespace pyg {

constexpr int kHeavyThreshold = 2048;  // rows longer than this are split (reading Q12)
constexpr int kChunk = 512;            // positions per chunk of a split row
constexpr int kTaskPositions = 4096;   // light positions per TMA-pipeline task
constexpr int kRedHeadW = 3;           // internal reduce mode: SUM with per-(edge, head) weights
                                       // hw[eid * hH + c / hC] (GAT alpha-weighted aggregation)
constexpr int kRedMaxW = 5;            // internal TMA-kernel mode: MAX of weighted messages (the plain
                                       // PYG_MAX instantiation assumes w == null: no multiply)
constexpr int kRedSumEpi = 4;          // internal TMA-kernel mode: SUM with the row-scale / blend /
                                       // bias epilogue (a separate instantiation keeps the plain SUM
                                       // kernel at its register count)

// ---- CSR segment-reduce ---------------------------------------------------------
struct SegArgs {
    const float* X = nullptr;  // gathered matrix, column offset applied
    int64_t ldx = 0;
    int ncols = 0;             // valid columns of this block
    const int64_t* rowptr = nullptr;
    const int32_t* gidx = nullptr;  // gathered row per position (null -> edge id)
    const int32_t* eid = nullptr;   // edge id per position (null -> position)
    const float* w = nullptr;       // per edge id
    const int32_t* gdeg = nullptr;  // divisor per gathered row (mean backward)
    float* out = nullptr;           // column offset applied
    int64_t ldo = 0;
    int64_t* arg = nullptr;         // MAX, stride lda, column offset applied
    int64_t lda = 0;
    int64_t n_rows = 0;
    int64_t E_sentinel = 0;
    int64_t heavy_threshold = 0;    // light pass skips rows longer than this
    int allow_pad_read = 0;         // X rows may be read up to round_up(ncols, 4)
    const int32_t* row_order = nullptr;  // light-row visiting order (root row ids), or null
    int64_t order_len = 0;          // entries of row_order (root rows)
    int64_t order_offset = 0;       // root row id of this plan's row 0 (slices skip others)
    uint32_t flags = 0;             // PYG_NO_TMA, ...
    int accum = 0;                  // add into out/arg (source-blocked passes after the first)
    int finalize = 1;               // apply the mean division in this pass
    const int32_t* deg_total = nullptr;  // mean divisor per row when segments are partial
    // APPNP blend epilogue (SUM/MEAN, finalize pass): out = blend_a * reduced + blend_b * blend[row]
    const float* blend = nullptr;
    int64_t ldb = 0;
    float blend_a = 1.0f, blend_b = 0.0f;
    // GCN-layer epilogue (SUM/MEAN, finalize pass): out = row_scale[row] * reduced (+ col_bias[c]);
    // order: mean divide, row scale, blend, column bias
    const float* row_scale = nullptr;
    const float* col_bias = nullptr;
    // kRedHeadW: weights [E x hH] by edge id; column c belongs to head c / hC (hC % V == 0)
    const float* hw = nullptr;
    int hH = 0, hC = 0;
};
// Full segment reduce of a block of columns: light rows, split hub rows (plan
// may be null for plan-free segment inputs such as pooling), fp64 combine.
pyg_status_t segment_reduce(const SegArgs& a, int reduce, const pyg_plan* plan, void* ws,
                            size_t ws_bytes, cudaStream_t s);
size_t segment_ws_bytes(const pyg_plan* plan, int64_t ncols, int reduce);
// out[p] = v[idx[p]] (per-edge values into plan position order)
pyg_status_t gather_by_index(const float* v, const int32_t* idx, int64_t n, float* out, cudaStream_t s);

// ---- atomic COO --------------------------------------------------------------------
struct CooArgs {
    const float* X = nullptr;
    int64_t ldx = 0;
    int ncols = 0;
    const int64_t* gidx = nullptr;  // gathered row per edge (null -> edge id)
    const int64_t* sidx = nullptr;  // scatter target per edge
    const float* w = nullptr;
    const int32_t* gdeg = nullptr;
    float* out = nullptr;  // SUM / MEAN accumulation target (zeroed by the launcher)
    int64_t ldo = 0;
    unsigned long long* keys = nullptr;  // MAX keys (zeroed by the launcher)
    int64_t ldk = 0;
    int64_t E = 0;
    int64_t n_out = 0;
    int64_t n_src = 0;  // rows gidx gathers from (L2 column-tile sizing; 0 -> E rows streamed once)
    int allow_pad_read = 0;
    const int32_t* deg = nullptr;   // in-degree of the targets if the caller has it (else computed)
    // hub routing (SUM / MEAN; set up by coo_reduce): rows with more than kHeavyThreshold entries
    // spread their edges over slots of <= kCooSlot entries, combined in fp64 (reading Q12)
    const int32_t* hub_base = nullptr;  // [n_out] first slot of a hub row (read for hubs only)
    const uint32_t* hub_bits = nullptr; // [n_out / 32] 1 bit per row: is a hub
    int32_t* hub_cursor = nullptr;      // [slots x column tiles] entry counters (by first slot)
    const int32_t* hub_count = nullptr; // device: number of hub rows (hub_assign_kernel)
    int tile_y = 0, n_tiles = 0;        // compact column tiles launched one by one (0: grid.y tiles)
    float* part = nullptr;              // [slots x ldp] slot partials = virtual rows n_out + slot
    int64_t ldp = 0;
};
// Whole atomic reduce of one column block: zero the target, degrees and hub slots (SUM / MEAN),
// the COO kernel, then the epilogue (mean divide + fp64 hub combine, or the MAX key decode).
pyg_status_t coo_reduce(const CooArgs& a, int reduce, void* ws, size_t ws_bytes, cudaStream_t s);
// n_src: rows the call gathers from (0: edge-space rows), sizes the compact-tile scratch
size_t coo_ws_bytes(int64_t E, int64_t n_out, int64_t ncols, int reduce, int64_t n_src);
// L2 column-tile width of the atomic path (0: one tile)
int64_t coo_tile_cols(int64_t n_out, int64_t n_src, int64_t ncols, int reduce);
// counts (and first edge id) per target for the COO path
pyg_status_t coo_degree(const int64_t* sidx, int64_t E, int64_t n, int32_t* deg, int32_t* first,
                        cudaStream_t s);
pyg_status_t mean_divide(float* out, int64_t ldo, int ncols, int64_t n, const int32_t* deg,
                         cudaStream_t s);
pyg_status_t max_decode(unsigned long long* keys, int64_t ldk, float* out, int64_t ldo, int ncols,
                        int64_t n, int64_t E, cudaStream_t s);

// ---- elementwise helpers -----------------------------------------------------------
// concat x_i block: out[i][c] = f(deg_i) * x[i][c]; arg = first edge of the segment
// deg from rowptr (plan) or deg array; first from plan perm/rowptr or array.
pyg_status_t xi_block(const float* x, int64_t ldx, int F, int64_t n, const int64_t* rowptr,
                      const int32_t* perm, const int32_t* deg, const int32_t* first, int reduce,
                      float* out, int64_t ldo, int64_t* arg, int64_t lda, int64_t E,
                      cudaStream_t s);
// per-edge gather of grad (scatter backward / edge_attr grad)
pyg_status_t edge_gather_grad(const float* g, int64_t ldg, const int64_t* index, int64_t E, int F,
                              int reduce, const int64_t* arg, int64_t lda, const int32_t* deg,
                              float* out, int64_t ldo, cudaStream_t s);
pyg_status_t xdst_grad(const float* g, int64_t ldg, int F, int64_t n, const int32_t* deg,
                       const int64_t* arg, int64_t lda, int64_t E, int reduce, float* out,
                       int64_t ldo, cudaStream_t s);
pyg_status_t max_route_grad(const float* g, int64_t ldg, const int64_t* arg, int64_t lda, int F,
                            int64_t n_dst, const int64_t* src, const float* w, int64_t E,
                            float* gx, int64_t ldgx, cudaStream_t s);
pyg_status_t edge_weight_grad(const float* x, int64_t ldx, const float* g, int64_t ldg,
                              const int64_t* arg, int64_t lda, const int64_t* ei, int64_t E, int F,
                              int reduce, const int32_t* deg, float* gw, cudaStream_t s);
pyg_status_t fill_rows(float* out, int64_t ldo, int ncols, int64_t n, cudaStream_t s);

// ---- attention (NEXT-1; attention.cu) ----------------------------------------------
// alpha[eid][h] = softmax over each row's positions of the logits: values src[eid][h] (s_src
// null) or GAT leaky_relu(s_src[col][h] + s_dst[row][h], slope).  Warp per light row, CTA per
// split hub row of `plan`.
pyg_status_t attention_softmax(const pyg_plan* plan, const int32_t* col, const int32_t* eid, const float* src,
                               int64_t lds, const float* s_src, const float* s_dst, int H, float slope, float* alpha,
                               int64_t lda, cudaStream_t s);
// dlogit = alpha (d_alpha - sum alpha d_alpha) per row (* leaky' for GAT, z != null: d_alpha is the
// SDDMM grad[row] . z[col] per head, and grad_s_dst gets the row sums)
pyg_status_t attention_softmax_bwd(const pyg_plan* plan, const int32_t* col, const int32_t* eid, int H, int C, int F,
                                   const float* alpha, int64_t lda, const float* grad, int64_t ldg, const float* z,
                                   int64_t ldz, const float* s_src, const float* s_dst, float slope, float* dlogit,
                                   int64_t ldd, float* grad_s_dst, cudaStream_t s, const float* row_sums = nullptr);

// GAT backward in one TMA gather4 pass (gat_tma.cu): dlogit and grad_s_dst from z, alpha, s_src,
// s_dst, grad_out and the forward output (t_i = g_i . out_i)
bool gat_bwd_tma_eligible(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t ldz, const float* g,
                          int64_t ldg, const float* out, int64_t ldo, const float* alpha, const float* s_src,
                          const float* s_dst, const float* gsd);
size_t gat_bwd_tma_ws_bytes(const pyg_plan* plan, int64_t H);
// GAT forward in one TMA gather4 pass (softmax shift bounded by max s_src; gat_tma.cu)
bool gat_fwd_tma_eligible(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t ldz, float* out,
                          int64_t ldo, const float* alpha, const float* s_src, const float* s_dst);
size_t gat_fwd_tma_ws_bytes(const pyg_plan* plan, int64_t H, int64_t F);
// GAT forward on a source-blocked plan: one pass per block, additive thanks to the fixed shift
size_t gat_fwd_blocked_ws_bytes(const pyg_plan* plan, int64_t H);
pyg_status_t gat_fwd_blocked(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                             const float* s_src, const float* s_dst, float slope, float* out, int64_t ldo, float* alpha,
                             float* row_sums, void* ws, size_t ws_bytes, cudaStream_t s);
pyg_status_t gat_fwd_tma(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                         const float* s_src, const float* s_dst, float slope, float* out, int64_t ldo, float* alpha,
                         float* row_sums, void* ws, size_t ws_bytes, cudaStream_t s);
pyg_status_t gat_bwd_tma(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                         const float* g, int64_t ldg, const float* out, int64_t ldo, const float* alpha,
                         const float* row_sums, const float* s_src, const float* s_dst, float slope, float* dlogit,
                         float* gsd, float* gsc, void* ws, size_t ws_bytes, cudaStream_t s);
// gsc[r][c] = g[r][c] / row_sums[r][c / C] (grad_out for the factored alpha, packed ld H*C)
pyg_status_t gat_scale_rows(const float* g, int64_t ldg, int64_t n, int H, int C, const float* row_sums, float* gsc,
                            cudaStream_t s);
pyg_status_t fill_const(float* p, int64_t n, float v, cudaStream_t s);

// device-side peer flags (halo.cu): release-store `value` into each flag, or spin until each >= value
pyg_status_t peer_flags_impl(uint32_t* const* flags, int n, uint32_t value, int wait, cudaStream_t s);

}  // namespace pyg
