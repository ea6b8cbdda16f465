/*
 * pyg_gs.h -- C ABI of libpygs.so: B200 (sm_100a) gather / phi / scatter-reduce
 * neighbourhood aggregation, the data-parallel hot path of Fey & Lenssen,
 * "Fast Graph Representation Learning with PyTorch Geometric" (arXiv 1903.02428).
 *
 * Citations: P:n = PAPER.md line n (section / equation named beside it),
 *            S:n = SPEC.md line n (interface shapes and edge-case conventions only).
 * Readings of ambiguous passages (Q1..Q20) are listed in DESIGN.md.
 *
 * The method (Eq. 1, without gamma):
 *     x'_i = BOX_{j in N(i)} phi(x_i, x_j, e_{j,i}),   BOX in {sum, mean, max}
 * computed as gather (node -> edge space) + phi + scatter (edge -> node space)
 * (Fig. 1), with the E x F edge space never materialised.
 *
 * ---------------------------------------------------------------------------
 * Conventions shared by every entry point
 *  - Memory: every tensor argument is a DEVICE pointer owned by the caller
 *    (allocated e.g. by torch).  The library never allocates, frees or retains
 *    caller memory.  Exceptions are marked (host) explicitly.  Plans
 *    (pyg_plan_t) are small host objects created by pyg_plan_build and released
 *    by pyg_plan_destroy; their device arrays live in caller-provided workspace.
 *  - Layout: row-major.  A matrix argument M[n x F] has a leading dimension
 *    ldM >= F in elements (floats); row r starts at M + r * ldM.  When
 *    ldM >= round_up(F, 4), ldM % 4 == 0 and M is 16-byte aligned, the kernels
 *    may READ (never use, never write) the padding columns [F, round_up(F,4))
 *    of each row, so such buffers must span n * ldM elements.
 *  - Indices: int64 (PyG's torch.long; P:25 I in N^{2 x E}).  edge_index is
 *    [2 x E] row-major: row 0 = source j, row 1 = target i; messages flow
 *    j -> i (reading Q1).  Arg outputs are int64 original edge ids.
 *    Internally E < 2^31 and node counts < 2^31 are required
 *    (PYG_ERR_UNSUPPORTED otherwise).
 *  - Precision: fp32 values, fp32 accumulation (hub rows are split into chunks
 *    and combined in fp64; reading Q12), IEEE division (no fast-math).
 *  - Outputs are OVERWRITTEN, never accumulated into (reading Q14).
 *  - Streams: `stream` is a cudaStream_t passed as void* (NULL = legacy default
 *    stream).  Every call is asynchronous on `stream` unless documented as
 *    synchronous.  Return codes cover host-side validation; with the
 *    PYG_VALIDATE flag a device pre-pass checks index ranges and the call
 *    synchronises `stream` to report PYG_ERR_INDEX_OUT_OF_BOUNDS.
 *  - Aliasing: outputs must not alias inputs.
 *  - Errors: a non-OK status leaves outputs unspecified; pyg_last_error()
 *    returns a thread-local message for the last failing call.
 */
#ifndef PYG_GS_H
#define PYG_GS_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Aggregation BOX of Eq. (1) ("sum, mean or max"). */
typedef enum { PYG_SUM = 0, PYG_MEAN = 1, PYG_MAX = 2 } pyg_reduce_t;

typedef enum {
    PYG_OK = 0,
    PYG_ERR_INVALID_ARGUMENT = 1,   /* null pointer, negative size, bad flag */
    PYG_ERR_DIMENSION = 2,          /* inconsistent shapes / leading dims */
    PYG_ERR_INDEX_OUT_OF_BOUNDS = 3,/* an index outside its range */
    PYG_ERR_ALIGNMENT = 4,          /* a forced vector path on unaligned data */
    PYG_ERR_UNSUPPORTED = 5,        /* sizes beyond the int32-internal limits */
    PYG_ERR_CUDA = 6,               /* a CUDA runtime error (message in pyg_last_error) */
    PYG_ERR_NCCL = 7,               /* NCCL missing or an NCCL call failed (pyg_dist_*) */
    PYG_ERR_NO_MEMORY = 8           /* workspace smaller than the size query returned */
} pyg_status_t;

/* flags */
#define PYG_PHI_CONCAT_XI  (1u << 0)  /* message = [x_i || w x_j || e_ji] */
#define PYG_VALIDATE       (1u << 8)  /* device index-range pre-pass; synchronous */
#define PYG_FORCE_ATOMIC   (1u << 9)  /* ignore `plan`, use the atomic COO strategy */
#define PYG_FORCE_SEGMENT  (1u << 10) /* require a plan (error if NULL) */
#define PYG_NO_TMA         (1u << 11) /* segment path: use the LDG kernel, not the TMA gather4
                                         pipeline (A/B testing; results are bitwise identical) */

typedef struct pyg_plan pyg_plan_t;   /* opaque host handle */

/* Read-only view of a plan's device arrays (for tests and the Python layer). */
typedef struct {
    int64_t n_rows;          /* segments (targets for a forward plan) */
    int64_t n_cols;          /* range of the gathered index (sources), 0 if none */
    int64_t E;               /* edges in the plan (all rows, before slicing) */
    int64_t row_offset;      /* first global row of this (possibly sliced) plan */
    const int64_t* rowptr;   /* [n_rows + 1] absolute positions; row r = [rowptr[r], rowptr[r+1]) */
    const int32_t* col;      /* [E] gathered index at each sorted position, or NULL */
    const int32_t* perm;     /* [E] original edge id at each sorted position */
    int32_t perm_is_identity;/* 1 if the input was already target-sorted */
    int64_t n_heavy_rows;    /* rows longer than heavy_threshold (split into chunks) */
    int64_t n_heavy_chunks;  /* chunks of at most chunk_size positions */
    int32_t heavy_threshold;
    int32_t chunk_size;
    int64_t col_block;       /* source rows per block (0: not source-blocked) */
    int64_t n_col_blocks;    /* passes per call (1 unless source-blocked) */
} pyg_plan_view_t;

/* ---- library ------------------------------------------------------------ */
const char* pyg_version(void);
const char* pyg_last_error(void);           /* thread-local, never NULL */
/* Number of kernels this library has launched since it was loaded (monotonic,
 * process-wide).  Used by bench.py to report gpu_launches. */
uint64_t pyg_launch_count(void);
/* Re-read the tuning / test knobs (PYG_SEG_TMA, PYG_TMA_HUBS, PYG_TMA_WARP_KB, PYG_TMA_WARPS; DESIGN.md
 * "knobs") from the environment.  They are read once when the library loads; tests that change them
 * call this.  Not thread-safe against concurrent calls. */
void pyg_refresh_env(void);

/* ---- degree ------------------------------------------------- */
/* deg[i] = #{k : index[k] == i}, i in [0, n); multi-edges and self-loops count
 * (reading Q6).  deg: int32 [n], overwritten.  Asynchronous. */
pyg_status_t pyg_degree(const int64_t* index, int64_t E, int64_t n, uint32_t flags, int32_t* deg,
                        void* stream);

/* ---- plan: CSR / target-sorted segments (App. A) --------------- */
/* A plan is the stable sort of edges by `row_index` (the target for a forward
 * plan; the source for the transposed plan the backward uses), i.e. CSR with
 * row = target.  P:276: coalescing is "expensive to compute on
 * GPUs and should be hence performed as part of the pre-processing" -- a plan
 * is built once per graph and reused by every call.
 *   row_index [E] int64 in [0, n_rows);  col_index [E] int64 in [0, n_cols)
 *   or NULL (scatter plans: the gathered row is the edge id itself).
 * col_block > 0 (forward plans only) builds a SOURCE-BLOCKED plan: edges are
 * sorted by (col_index / col_block, row, id), and calls make one pass per
 * block of col_block source rows, accumulating into `out` in block order, so
 * the block of X a pass gathers stays resident in the 126 MB L2 (B200-specific;
 * see DESIGN.md "source-blocked passes").  Results are deterministic; the sum
 * order differs from the unblocked plan's.  col_block = 0: one CSR.
 * Workspace: `bytes` from pyg_plan_workspace_size; it holds the plan's device
 * arrays and must outlive the plan.  SYNCHRONOUS (reads back counts); returns
 * PYG_ERR_INDEX_OUT_OF_BOUNDS if an index is out of range. */
pyg_status_t pyg_plan_workspace_size(int64_t E, int64_t n_rows, int64_t n_cols, int64_t col_block,
                                     size_t* bytes);
pyg_status_t pyg_plan_build(const int64_t* row_index, const int64_t* col_index, int64_t E,
                            int64_t n_rows, int64_t n_cols, int64_t col_block, uint32_t flags,
                            void* workspace, size_t bytes, pyg_plan_t** plan, void* stream);
/* Suggest col_block for gathering rows of `row_bytes` bytes (ldx * 4) on the
 * current device: blocks of ~0.4 x L2; 0 when X fits one block or when the
 * reuse (E / n_cols) does not repay the extra read+write of `out` per pass, with
 * half of L2 counted as the reuse capacity of an unblocked random gather
 * (host-only; queries the L2 size). */
pyg_status_t pyg_plan_suggest_col_block(int64_t E, int64_t n_rows, int64_t n_cols,
                                        int64_t row_bytes, int64_t* col_block);
/* Column-tile width of the atomic strategy (plan NULL) for a reduce into n_out rows
 * of `ncols` floats gathering from n_src rows (n_src = 0: edge-space src, as
 * pyg_scatter): the tile keeps the accumulation target (fp32 out, or the 64-bit
 * MAX keys) and the gathered slice inside the L2 budget (PYG_COO_L2_MB /
 * PYG_COO_L2_MB_MAX), so every red.global hits L2 (P:270-271's atomics, sized
 * for B200's L2).  *cols = 0: one tile (everything fits,
 * or even 8 columns do not).  Host-only; never fails for valid sizes. */
pyg_status_t pyg_atomic_tile_cols(int64_t n_out, int64_t n_src, int64_t ncols, pyg_reduce_t reduce,
                                  int64_t* cols);
/* Sub-plan of rows [row_lo, row_hi) sharing the parent's arrays (dst-range
 * partitioning for the multi-GPU layer).  Output row r of a call using the
 * slice is global row row_lo + r; arg outputs stay GLOBAL edge ids. */
pyg_status_t pyg_plan_slice(const pyg_plan_t* plan, int64_t row_lo, int64_t row_hi,
                            pyg_plan_t** slice);
/* Pass view of a SOURCE-BLOCKED plan (or a slice of one): the source blocks [pass_lo, pass_hi)
 * only.  Calls made with the views of consecutive block ranges, in order and on one stream, give
 * exactly the result of one call with the whole plan (the root's first block writes `out`, later
 * blocks accumulate, its last block finalizes) -- so a multi-GPU step can run block b as soon as
 * the X rows of block b have arrived (compute / communication overlap).  Zero-copy; the parent
 * must outlive the view.  CONCAT_XI is not supported with views. */
pyg_status_t pyg_plan_passes(const pyg_plan_t* plan, int64_t pass_lo, int64_t pass_hi,
                             pyg_plan_t** view);
pyg_status_t pyg_plan_view(const pyg_plan_t* plan, pyg_plan_view_t* view);
/* Copy a plan's CSR arrays into caller device buffers (any may be NULL):
 * rowptr [n_rows + 1] int64 (positions relative to the plan's first row),
 * col [E_p] int64 and perm [E_p] int64 for the E_p positions of the plan's
 * rows.  Asynchronous. */
pyg_status_t pyg_plan_export(const pyg_plan_t* plan, int64_t* rowptr, int64_t* col, int64_t* perm,
                             void* stream);
void pyg_plan_destroy(pyg_plan_t* plan);

/* ---- halo exchange of the dst-range partition (north_star (3)) ---- */
/* For a rank owning targets [own_lo, own_hi) (and the X rows of the same range,
 * stored as the first own_rows >= own_hi - own_lo rows of a rank-local buffer),
 * pyg_halo_build derives from `slice` (pyg_plan_slice of an UNBLOCKED forward
 * plan over n_src sources) the halo: the sources referenced by the slice's
 * edges that lie outside [own_lo, own_hi), in ascending global id (so grouped
 * by owner rank when ranks own contiguous ascending ranges).
 *   halo_ids: (device) int64 capacity n_src; receives the n_halo halo ids.
 *   n_halo:   (host) receives the halo size.
 *   halo_plan: a plan equal to `slice` except that every gathered index is
 *     rank-local: own source j -> j - own_lo, halo source halo_ids[h] ->
 *     own_rows + h.  A pyg_propagate with this plan reads
 *     x_src = X_loc [(own_rows + n_halo) x F], the own shard followed by the
 *     halo rows in halo_ids order; outputs (and max arg edge ids, which stay
 *     GLOBAL) are bitwise equal to the slice's on the full X.
 * Workspace (pyg_halo_workspace_size) holds the halo plan's index array and
 * must outlive it; `slice` (and its root plan) must outlive it too.
 * SYNCHRONOUS (n_halo is read back).  PYG_ERR_UNSUPPORTED for source-blocked
 * or scatter plans. */
pyg_status_t pyg_halo_workspace_size(const pyg_plan_t* slice, int64_t n_src, size_t* bytes);
pyg_status_t pyg_halo_build(const pyg_plan_t* slice, int64_t n_src, int64_t own_lo, int64_t own_hi,
                            int64_t own_rows, void* workspace, size_t bytes, pyg_plan_t** halo_plan,
                            int64_t* halo_ids, int64_t* n_halo, void* stream);
/* Row gather (the halo "pack": the rows a peer requested, contiguous for the
 * all-to-all): out[r] = x[rows[r]], r in [0, n).  x [n_x x F] stride ldx;
 * rows int64 in [0, n_x) (checked synchronously with PYG_VALIDATE);
 * out [n x F] stride ldo, overwritten.  Asynchronous. */
pyg_status_t pyg_gather_rows(const float* x, int64_t n_x, int64_t F, int64_t ldx, const int64_t* rows,
                             int64_t n, uint32_t flags, float* out, int64_t ldo, void* stream);
/* Peer-store halo (the alternative to pack + NCCL all-to-all): the owner stores the rows each
 * peer requested straight into the peer's X_loc over NVLink (one kernel: gather + transfer).
 * Peers' buffers are mapped with CUDA IPC (same node):
 *   pyg_ipc_handle: (host) 64-byte handle of the allocation containing dev_ptr + the byte offset
 *     of dev_ptr inside it;  pyg_ipc_open: map a peer's (handle, offset) -> dev_ptr (peer access
 *     enabled lazily);  pyg_ipc_close: unmap (dev_ptr, offset as opened).
 *   pyg_halo_push: for peer q < n_peers (<= 16): local rows send_rows[send_ptr[q] ..
 *     send_ptr[q+1]) of x [n_x x F] (stride ldx) are stored to rows dst_row[q] + i of dst[q]
 *     (stride ldd).  send_ptr [n_peers + 1], dst [n_peers] (device pointers, e.g. from
 *     pyg_ipc_open) and dst_row [n_peers] are HOST arrays; send_rows is a device array.
 *     Asynchronous; the caller orders the peers' reads after the pushes (pyg_peer_signal /
 *     pyg_peer_wait below, or a stream sync + a process-group barrier). */
pyg_status_t pyg_ipc_handle(const void* dev_ptr, void* handle, int64_t* offset);
pyg_status_t pyg_ipc_open(const void* handle, int64_t offset, void** dev_ptr);
pyg_status_t pyg_ipc_close(void* dev_ptr, int64_t offset);
pyg_status_t pyg_halo_push(const float* x, int64_t n_x, int64_t F, int64_t ldx, const int64_t* send_rows,
                           const int64_t* send_ptr, void* const* dst, const int64_t* dst_row,
                           int64_t ldd, int n_peers, void* stream);
/* Device-side step flags between the ranks of a node (replace the host stream-sync + process-group
 * barrier around a peer-store exchange; P:26 multi-GPU, north_star (3)).  flags: HOST array of n
 * (<= 16) device addresses of uint32 flags (a peer's, mapped with pyg_ipc_open, or local).
 *   pyg_peer_signal: enqueue on `stream`: make every earlier write of the stream visible system-wide
 *     (the peer stores of pyg_halo_push), then release-store `value` into each flag.
 *   pyg_peer_wait: enqueue on `stream`: spin until each flag reaches `value` (acquire; wrap-safe
 *     uint32 comparison), so later work on the stream sees the writes made before the matching
 *     signal.  Deadlock-free use: every rank signals what it owes before it waits (dist.HaloPush).
 * Asynchronous. */
pyg_status_t pyg_peer_signal(uint32_t* const* flags, int n, uint32_t value, void* stream);
pyg_status_t pyg_peer_wait(uint32_t* const* flags, int n, uint32_t value, void* stream);

/* Scratch needed by pyg_scatter / pyg_propagate / pyg_propagate_backward for
 * an output of n_out rows x F_out columns over E edges.
 *   plan path: the fp32 partials of split hub rows, combined in fp64 (reading Q12).
 *   atomic path (plan NULL or PYG_FORCE_ATOMIC): the in-degree array and, for
 *   SUM / MEAN, the hub slots -- rows with more than 2048 entries spread their
 *   edges over slots of <= 2048 entries (one atomic counter per hub hands out
 *   positions) whose fp32 partials are combined in fp64, so no fp32 atomic chain
 *   exceeds 2048 terms (Q12).  The size is the worst case for E edges
 *   (E/2048 + E/2049 slots x F_out floats).  When the output is split into L2
 *   column tiles (pyg_atomic_tile_cols > 0) it also holds the compact-tile
 *   scratch -- the tile's accumulation target (n_out x W floats, or 64-bit keys
 *   for MAX) and its gathered slice (n_src x W floats, sized with n_src = n_out);
 *   with less workspace (e.g. bipartite n_src > n_out) the tiles run in place,
 *   slower but with the same results.
 * For pyg_propagate_backward pass (plan_T, E, n_src, F).  Host-only. */
pyg_status_t pyg_workspace_size(const pyg_plan_t* plan, int64_t E, int64_t n_out, int64_t F_out,
                                pyg_reduce_t reduce, uint32_t flags, size_t* bytes);

/* ---- scatter: edge space -> node space -------------- */
/* out[i] = BOX_{k : index[k] = i} src[k]; empty segment -> 0 (Q2).
 *   src [E x F] stride lds; index [E] int64 in [0, dim_size)
 *   out [dim_size x F] stride ldo, overwritten
 *   arg_out [dim_size x F] int64 stride ldo, REQUIRED iff reduce == PYG_MAX:
 *     the lowest edge id attaining the max (north_star tie rule, Q4); E for
 *     empty segments (Q3).  (On the atomic path it doubles as the 64-bit key
 *     buffer before being decoded in place.)
 *   plan: built with row_index = index, col_index = NULL -> deterministic
 *     CSR segment-reduce; NULL -> atomic COO (warp-aggregated
 *     red.global.add.v4.f32, hub rows through fp64-combined slots / 64-bit
 *     atomicMax keys), non-deterministic for sum/mean.
 *   workspace: pyg_workspace_size(plan, E, dim_size, F, reduce, flags). */
pyg_status_t pyg_scatter(const float* src, int64_t E, int64_t F, int64_t lds, const int64_t* index,
                         int64_t dim_size, pyg_reduce_t reduce, uint32_t flags, float* out,
                         int64_t ldo, int64_t* arg_out, const pyg_plan_t* plan, void* workspace,
                         size_t workspace_bytes, void* stream);

/* scatter backward w.r.t. src: grad_src[k] = g[index[k]] (sum),
 * g[index[k]] / deg[index[k]] (mean, IEEE float divide), g[i] where
 * arg_out[i] == k else 0 (max).  deg (int32 [dim_size], from pyg_degree)
 * required for MEAN; arg_out (stride ldg) required for MAX.  Pure gather,
 * deterministic. */
pyg_status_t pyg_scatter_backward(const float* grad_out, int64_t ldg, const int64_t* index, int64_t E,
                                  int64_t F, int64_t dim_size, pyg_reduce_t reduce,
                                  const int64_t* arg_out, const int32_t* deg, float* grad_src,
                                  int64_t lds, void* stream);

/* ---- propagate: fused gather + phi + reduce (Eq. 1; Fig. 1) ----------------- */
/* For every edge k = (j -> i) the message is
 *     m_k = [ x_dst[i] (only if PYG_PHI_CONCAT_XI) || w_k * x_src[j] || edge_attr[k] (if D > 0) ]
 * (phi in {identity, edge-weight scale, concatenation})
 * and out[i] = BOX_k m_k, F_out = (CONCAT_XI ? F : 0) + F + D, computed
 * without materialising the messages.
 *   x_src [n_src x F] stride ldx; x_dst [n_dst x F] stride ldxd (NULL -> x_src,
 *     requires n_dst <= n_src); edge_index [2 x E] int64 (row-major, see top);
 *   edge_attr [E x D] stride lde or NULL (D = 0); edge_weight [E] or NULL (w=1);
 *   out [n_dst x F_out] stride ldo; arg_out [n_dst x F_out] int64 stride ldo
 *   (MAX only).  mean divides by the integer in-degree (Q6).
 *   plan: forward plan (row_index = edge_index[1], col_index = edge_index[0]),
 *   possibly a slice; NULL -> atomic COO.  workspace: pyg_workspace_size. */
pyg_status_t pyg_propagate(const float* x_src, int64_t n_src, int64_t F, int64_t ldx,
                           const float* x_dst, int64_t ldxd, int64_t n_dst,
                           const int64_t* edge_index, int64_t E, const float* edge_attr,
                           int64_t D, int64_t lde, const float* edge_weight,
                           pyg_reduce_t reduce, uint32_t flags, float* out, int64_t ldo,
                           int64_t* arg_out, const pyg_plan_t* plan, void* workspace,
                           size_t workspace_bytes, void* stream);

/* propagate backward ("both for forward and backward passes", P:277;
 * S:142).  grad_out [n_dst x F_out] stride ldg.  Outputs, each
 * optional (NULL to skip), overwritten:
 *   grad_x_src [n_src x F] stride ldgx:  sum_k w_k * dL/dm_k  over k with src_k = j
 *       (mean: dL/dm_k = g[dst_k] / deg[dst_k]; max: g routed to arg_out).
 *       SUM / MEAN with plan_T (row_index = edge_index[0], col_index =
 *       edge_index[1]): a deterministic segment-reduce over sources; else atomic
 *       COO.  MAX always routes g[i][c] to source src[arg[i][c]] with fp32
 *       atomicAdd (plan_T unused): each (i, c) contributes to exactly one
 *       source, so only sources that are the argmax of several (target, column)
 *       pairs sum more than one term, in an unspecified (non-deterministic)
 *       order -- within the summation bound, not bitwise reproducible.
 *   grad_x_dst [n_dst x F] stride ldgxd (CONCAT_XI block): deg*g (sum),
 *       g if deg > 0 (mean, max).
 *   grad_edge_attr [E x D] stride ldge: the e block of dL/dm_k.
 *   grad_edge_weight [E]: sum_c x_src[j][c] * dL/dm_k[c] over the x_j block.
 * deg_dst (int32 [n_dst], pyg_degree of edge_index[1]) is required for MEAN
 * and for the CONCAT_XI block with SUM; arg_out (stride ldg) for MAX. */
pyg_status_t pyg_propagate_backward(const float* x_src, int64_t n_src, int64_t F, int64_t ldx,
                                    int64_t n_dst, const int64_t* edge_index, int64_t E, int64_t D,
                                    const float* edge_weight, pyg_reduce_t reduce, uint32_t flags,
                                    const float* grad_out, int64_t ldg, const int64_t* arg_out,
                                    const int32_t* deg_dst, float* grad_x_src, int64_t ldgx,
                                    float* grad_x_dst, int64_t ldgxd, float* grad_edge_attr,
                                    int64_t ldge, float* grad_edge_weight,
                                    const pyg_plan_t* plan_T, void* workspace,
                                    size_t workspace_bytes, void* stream);

/* ---- GCN normalisation ------------------------- */
/* Appends (i,i) with weight 1 after the E original edges, in ascending i, for
 * every node lacking a self-loop (existing loops kept; Q8); d[i] = sum of
 * weights into i (Q7); w'_k = d[src]^-1/2 * w_k * d[dst]^-1/2.
 *   edge_index_out: capacity 2 x (E + N) int64; written as a packed row-major
 *   [2 x E_out] array (targets start at edge_index_out + E_out).
 *   weight_out: capacity E + N floats.  E_out: (host) receives E'.
 * SYNCHRONOUS (E_out is read back).  Workspace: pyg_gcn_norm_workspace_size. */
pyg_status_t pyg_gcn_norm_workspace_size(int64_t E, int64_t N, size_t* bytes);
pyg_status_t pyg_gcn_norm(const int64_t* edge_index, int64_t E, int64_t N,
                          const float* edge_weight, uint32_t flags, int64_t* edge_index_out,
                          float* weight_out, int64_t* E_out, void* workspace, size_t bytes,
                          void* stream);

/* ---- mini-batch collate ------------------------------- */
/* Block-diagonal batching: node_ptr = exclusive prefix sum of num_nodes
 * (G+1 entries); edge_index[:, e] = local_edge_index[:, e] + node_ptr[g(e)]
 * where g(e) is the graph owning column e (edge_ptr[g] <= e < edge_ptr[g+1]);
 * batch[v] = g for node_ptr[g] <= v < node_ptr[g+1].
 *   num_nodes [G], edge_ptr [G+1] (device, int64); local_edge_index and
 *   edge_index [2 x E_total]; batch [N_total]; node_ptr [G+1].
 *   E_total = edge_ptr[G] and N_total = sum num_nodes are passed by the host
 *   (it sized the outputs).  G <= 0 -> PYG_ERR_INVALID_ARGUMENT.
 *   With PYG_VALIDATE the call synchronises and returns
 *   PYG_ERR_INDEX_OUT_OF_BOUNDS if a local id is outside [0, N_g) or
 *   PYG_ERR_DIMENSION if E_total / N_total disagree with the arrays. */
pyg_status_t pyg_collate(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr,
                         const int64_t* local_edge_index, int64_t E_total, int64_t N_total,
                         uint32_t flags, int64_t* edge_index, int64_t* batch, int64_t* node_ptr,
                         void* stream);

/* ---- global pooling readout ------------------------ */
/* out[g] = BOX over nodes v in [node_ptr[g], node_ptr[g+1]) of x[v]
 * (contiguous segments of the collated batch).  arg_out = node id (MAX). */
pyg_status_t pyg_global_pool(const float* x, int64_t N, int64_t F, int64_t ldx,
                             const int64_t* node_ptr, int64_t G, pyg_reduce_t reduce, float* out,
                             int64_t ldo, int64_t* arg_out, void* stream);

/* ---- NEXT-1: segment softmax and GAT attention aggregation ------------------ */
/* The paper's only other custom kernels: "our own optimized sparse softmax
 * kernels" for GAT (GAT P:52).  Semantics from S:161-169 / S:421-429.
 * All deterministic; they run on the CSR plans (no atomic variant).
 *
 * pyg_segment_softmax: out[k][h] = exp(src[k][h] - m_i) / sum_{k' : index[k'] = i}
 *   exp(src[k'][h] - m_i), m_i the segment max, for i = index[k].
 *   src [E x H] stride lds; out [E x H] stride ldo (overwritten; edges keep their
 *   ids); plan: the SCATTER plan of index (pyg_plan_build(index, NULL, ...)),
 *   unblocked; `index` itself is not read (may be NULL).  Empty segments have no
 *   entries.  Asynchronous. */
pyg_status_t pyg_segment_softmax(const float* src, int64_t E, int64_t H, int64_t lds,
                                 const int64_t* index, int64_t dim_size, const pyg_plan_t* plan,
                                 float* out, int64_t ldo, void* stream);
/* grad_src[k][h] = out[k][h] * (g[k][h] - sum_{k' in seg(k)} out[k'][h] g[k'][h]);
 * H <= 8.  Same plan as the forward.  Asynchronous. */
pyg_status_t pyg_segment_softmax_backward(const float* out, int64_t ldo, const float* grad_out,
                                          int64_t ldg, int64_t E, int64_t H, int64_t dim_size,
                                          const pyg_plan_t* plan, float* grad_src, int64_t lds,
                                          void* stream);
/* Scratch of pyg_gat_propagate.  Host-only. */
pyg_status_t pyg_gat_propagate_workspace_size(const pyg_plan_t* plan, int64_t H, int64_t C, size_t* bytes);
/* GAT aggregation with H heads of C channels: for edge k = (j -> i),
 *   alpha[k][h] = softmax over the in-edges of i of
 *                 leaky_relu(s_src[j][h] + s_dst[i][h], negative_slope),
 *   out[i][h*C + c] = sum_k alpha[k][h] * z[j][h*C + c]   (empty segment -> 0).
 * z [n_src x H*C] stride ldz (the transformed features x W, computed by the
 * caller); s_src [n_src x H], s_dst [n_dst x H] packed (the attention
 * projections a_src . z_j and a_dst . z_i per head, computed by the caller);
 * out [n_dst x H*C] stride ldo; alpha [E x H] packed, OUTPUT (by original edge
 * id; needed by the backward).  plan: unblocked forward plan (row = target,
 * col = source).  H <= 8.  workspace: pyg_gat_propagate_workspace_size(plan, H, C).
 * Large graphs (H in {4, 8}, 16-byte aligned rows) take ONE streaming pass: softmax is
 * shift-invariant, and c_i[h] = leaky_relu(max_j s_src[j][h] + s_dst[i][h]) bounds every
 * logit of row i (leaky_relu is monotone), so the weights exp(l - c_i) <= 1 are accumulated
 * with z_j as they are gathered and divided by their row sum at the row's end; rows whose sum
 * underflows (< 1e-30) are recomputed with their own max.
 * row_sums [n_dst x H] packed, OPTIONAL OUTPUT: the attention in factored form -- alpha then holds
 * weights p with alpha_true[k][h] = alpha[k][h] / row_sums[dst_k][h] (on the one-pass path the
 * division over all E x H entries, a random read-modify-write, is skipped; pyg_gat_backward takes
 * the pair).  NULL -> alpha is normalised.  Asynchronous. */
pyg_status_t pyg_gat_propagate(const float* z, int64_t n_src, int64_t H, int64_t C, int64_t ldz,
                               const float* s_src, const float* s_dst, int64_t n_dst, int64_t E,
                               float negative_slope, const pyg_plan_t* plan, float* out,
                               int64_t ldo, float* alpha, float* row_sums, void* workspace,
                               size_t workspace_bytes, void* stream);
/* Scratch of pyg_gat_backward (both its paths; with_row_sums: alpha passed in factored form,
 * + n_dst x H*C floats).  Host-only. */
pyg_status_t pyg_gat_backward_workspace_size(const pyg_plan_t* plan, const pyg_plan_t* plan_T,
                                             int64_t H, int64_t C, int with_row_sums, size_t* bytes);
/* Backward of pyg_gat_propagate, g = grad_out [n_dst x H*C] stride ldg:
 *   grad_z[j][h*C+c] = sum_{k: src_k = j} alpha[k][h] g[dst_k][h*C+c]     (grad_z optional)
 *   grad_logit[k][h] = alpha[k][h] (g_i . z_j|_h - sum_{k' in seg(i)} alpha[k'][h] g_i . z_j'|_h)
 *                      * leaky_relu'(s_src[j][h] + s_dst[i][h])   (dL/d pre-activation; REQUIRED,
 *                      [E x H] packed, by edge id)
 *   grad_s_dst[i][h] = sum over i's in-edges of grad_logit     ([n_dst x H] packed, required)
 *   grad_s_src[j][h] = sum over j's out-edges of grad_logit    ([n_src x H] packed, optional)
 * out [n_dst x H*C] stride ldo: the forward output of pyg_gat_propagate, or NULL.  With it,
 *   sum_{k' in seg(i)} alpha[k'][h] g_i . z_j'|_h = g_i . out_i|_h (the aggregation is linear in
 *   z), so the SDDMM and the softmax backward run as ONE streaming pass over the plan (TMA
 *   gather4 pipeline; H in {4, 8}, C a power of two <= 128 or a multiple of 128, 16-byte
 *   aligned rows); without it (or outside those shapes) two passes per row recompute the sum.
 * row_sums: NULL (alpha normalised) or the forward's row_sums (alpha in factored form).
 * plan: the forward plan (unblocked); plan_T: row_index = sources, col_index = targets -- it may be
 *   source-blocked (blocks of grad_out rows, pyg_plan_suggest_col_block with row_bytes = 4*H*C):
 *   grad_z and grad_s_src then run as one L2-resident pass per block.  The forward may have run
 *   on a blocked plan of the same edges: alpha (by edge id) and row_sums mean the same.
 * H*C <= 4096.  workspace: pyg_gat_backward_workspace_size(plan, plan_T, H, C, row_sums != NULL).
 * Asynchronous. */
pyg_status_t pyg_gat_backward(const float* z, int64_t n_src, int64_t H, int64_t C, int64_t ldz,
                              const float* s_src, const float* s_dst, int64_t n_dst, int64_t E,
                              float negative_slope, const float* alpha, const float* row_sums,
                              const float* grad_out,
                              int64_t ldg, const float* out, int64_t ldo,
                              const pyg_plan_t* plan, const pyg_plan_t* plan_T,
                              float* grad_z, int64_t ldgz, float* grad_s_src, float* grad_s_dst,
                              float* grad_logit, void* workspace, size_t workspace_bytes,
                              void* stream);

/* ---- NEXT-2: K-step propagation (APPNP; SGC) on one plan ------------------- */
/* APPNP's propagation: z_0 = h, z_{k+1} = (1 - alpha) S z_k + alpha h,
 * out = z_K, with S the weighted adjacency of the plan (edge_weight [E] by edge id,
 * e.g. GCN's D^-1/2 (A+I) D^-1/2 from pyg_gcn_norm; NULL = 1).  alpha = 0 gives
 * SGC's S^K h.  The teleport term is fused into the segment-reduce
 * epilogue (no extra pass over z).  The backward w.r.t. h is the same recurrence on
 * the transposed plan with h := dL/dout (w_K = T^K g + alpha sum_{j<K} T^j g,
 * T = (1 - alpha) S^T), i.e. pyg_appnp(g, ..., plan_T).
 *   h [n x F] stride ldh; out [n x F] stride ldo (overwritten); scratch [n x F]
 *   stride ldo, required for K > 1 (ping-pong buffer); K >= 0 (K = 0 copies h);
 *   0 <= alpha <= 1.  plan: forward plan over n targets / n sources.  Per-call
 *   fp32 rounding of every z_k.  workspace: pyg_workspace_size(plan, n, F, SUM);
 *   with E * 4 + 256 more bytes the weights are gathered into plan order once and
 *   every step streams them (same results).  Asynchronous. */
pyg_status_t pyg_appnp(const float* h, int64_t n, int64_t F, int64_t ldh, const float* edge_weight,
                       int64_t K, float alpha, const pyg_plan_t* plan, float* out, int64_t ldo,
                       float* scratch, void* workspace, size_t workspace_bytes, void* stream);

/* ---- NEXT-2: dense feature transform on the tensor cores ------------------------ */
/* Y[m][n] = row_scale[m] * sum_k X[m][k] W[n][k] + bias[n]: the x W of GCN / SGC /
 * APPNP layers, on tcgen05 tensor cores in TF32 with fp32 accumulation (both
 * operands keep 10 mantissa bits: |error| <= ~2^-9 sum_k |X[m][k] W[n][k]|, A7).
 *   X [M x K] stride ldx (row-major; 16-byte aligned, ldx % 4 == 0);
 *   W [N x K] stride ldw (the torch.nn.Linear weight layout [out x in]; same alignment);
 *   bias [N] or NULL; row_scale [M] or NULL (e.g. GCN's D^-1/2, applied before the bias);
 *   Y [M x N] stride ldy, overwritten.  K >= 1; N > 256 runs as several 256-column tiles (X is
 *   then read once per tile).  Asynchronous. */
pyg_status_t pyg_dense_transform(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W,
                                 int64_t N, int64_t ldw, const float* bias, const float* row_scale,
                                 float* Y, int64_t ldy, void* stream);

/* GCN layer (Kipf & Welling's operator): out = D^-1/2 (A+I) D^-1/2 X W^T + bias,
 * with d_i = the in-degree in `plan` (which must already contain the self-loops, e.g. a
 * plan of pyg_gcn_norm's edge_index; reading Q7/Q8).  Transform first on the tensor cores
 * (pyg_dense_transform, rows scaled by D^-1/2 in its epilogue, so the aggregation runs at
 * width F_out), then an UNWEIGHTED segment sum over the plan whose epilogue scales rows by
 * D^-1/2 and adds the bias: no per-edge weights or edge ids are read.
 *   X [n x K] stride ldx, W [F_out x K] stride ldw (alignment as pyg_dense_transform),
 *   bias [F_out] or NULL, out [n x F_out] stride ldo.  plan: forward plan, n x n -- unblocked, or
 *   source-blocked (pyg_plan_suggest_col_block with row_bytes = 4 * F_out: the transformed rows are
 *   then aggregated one L2-resident block at a time, D^-1/2 and the bias applied in the last pass).
 *   workspace: pyg_gcn_layer_workspace_size (D^-1/2, the transformed rows, split rows).
 *   Asynchronous. */
pyg_status_t pyg_gcn_layer_workspace_size(const pyg_plan_t* plan, int64_t n, int64_t F_out,
                                          size_t* bytes);
pyg_status_t pyg_gcn_layer(const float* X, int64_t n, int64_t K, int64_t ldx, const float* W,
                           int64_t F_out, int64_t ldw, const float* bias, const pyg_plan_t* plan,
                           float* out, int64_t ldo, void* workspace, size_t workspace_bytes,
                           void* stream);

/* GAT transform: z = X W^T on the tensor cores (as pyg_dense_transform, TF32) with
 * the attention projections fused into the epilogue:
 *   s_src[m][h] = sum_{c < C} z[m][h*C + c] att_src[h*C + c],  s_dst likewise with att_dst
 * (the split form of S:424's [z_i || z_j] . a; the inputs of pyg_gat_propagate).
 *   X [M x K] stride ldx; W [H*C x K] stride ldw (alignment as pyg_dense_transform); att_src /
 *   att_dst [H*C]; Z [M x H*C] stride ldz; s_src / s_dst [M x H] packed.  H <= 8, H*C <= 256.
 *   The projections use the fp32 z values before they are stored.  Asynchronous. */
pyg_status_t pyg_gat_transform(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W,
                               int64_t H, int64_t C, int64_t ldw, const float* att_src,
                               const float* att_dst, float* Z, int64_t ldz, float* s_src, float* s_dst,
                               void* stream);

/* ---- multi-GPU: dst-range partitioned propagate over NCCL ------------------------------------
 * north_star (3), SURVEY 8(b) pyg_dist_init / pyg_dist_propagate and 8(e); the paper's own system
 * is single-GPU (P:26 names multi-GPU support as PyG's, without a scheme).  One process per GPU.
 * Rank p owns the targets -- and the X rows -- [lo_p, hi_p) = [p*per, min((p+1)*per, n)) with
 * per = ceil(n / world) (rounded up to a multiple of the source block for source-blocked plans), and
 * every in-edge of them, so the reduction is local and results equal the single-GPU call's (max /
 * argmax bitwise; arg ids stay GLOBAL edge ids).  The exchange moves only source rows:
 *   PYG_EXCHANGE_ALLGATHER  ncclAllGather of the X shards (dense graphs); with a source-blocked plan
 *                           one ncclBroadcast per owner on a side stream, each owner's source blocks
 *                           computed as soon as its rows land (compute / transfer overlap);
 *   PYG_EXCHANGE_HALO       only the referenced remote rows (the halo, ascending global id), packed
 *                           by the owner and delivered with grouped ncclSend / ncclRecv;
 *   PYG_EXCHANGE_AUTO       halo if the largest halo is < half the all-gather rows, else all-gather
 *                           (always all-gather for source-blocked plans).
 * Backward: the local edges transposed give partial dL/dX for every referenced source, then
 * ncclReduceScatter to the owners (all-gather) or the reverse halo (partials of the halo rows sent
 * back, added per own row in rank order: deterministic for SUM / MEAN).
 * NCCL is loaded at run time (dlopen libnccl.so.2, or $PYG_NCCL_LIB); if it is missing or an NCCL
 * call fails the call returns PYG_ERR_NCCL.  All calls taking a comm or a dist plan are
 * COLLECTIVE: every rank makes the same sequence of them.  Dist plans OWN their device buffers
 * (cudaMalloc at build, freed by pyg_dist_plan_destroy) -- the exception to "the library never
 * allocates" above; the communicator is released by pyg_dist_finalize. */
typedef struct pyg_dist pyg_dist_t;
typedef struct pyg_dist_plan pyg_dist_plan_t;
#define PYG_EXCHANGE_AUTO 0
#define PYG_EXCHANGE_ALLGATHER 1
#define PYG_EXCHANGE_HALO 2
typedef struct {
    int64_t lo, hi, per;      /* own target / X rows [lo, hi); shard capacity per rank */
    int exchange;             /* PYG_EXCHANGE_ALLGATHER or PYG_EXCHANGE_HALO (resolved) */
    int64_t n_halo;           /* halo rows received per call (halo) */
    int64_t n_send;           /* rows sent per call (halo) */
    int64_t n_local_edges;    /* in-edges of the own targets */
    int64_t col_block;        /* source rows per block (0: unblocked plan) */
    float* x_shard;           /* (device) where this rank's X rows live inside the exchange buffer:
                                 writing them here saves pyg_dist_propagate's copy */
    int64_t ldx;              /* its row stride */
    const pyg_plan_t* plan;   /* the rank's slice of the global forward plan */
} pyg_dist_plan_info_t;

/* 128-byte ncclUniqueId (host) for rank 0 to broadcast over its process group.  Synchronous. */
pyg_status_t pyg_dist_unique_id(void* nccl_unique_id);
/* Communicator over `world` ranks (call with the rank's GPU current).  Synchronous, collective. */
pyg_status_t pyg_dist_init(const void* nccl_unique_id, int rank, int world, pyg_dist_t** comm);
void pyg_dist_finalize(pyg_dist_t* comm);
/* One rank's share of a graph: edge_index [2 x E] (device; the FULL graph, identical on every rank,
 * read during the build only), n nodes, feature width F whose exchange buffers have row stride ld
 * (ld >= F, ld % 4 == 0), col_block as pyg_plan_build (0: unblocked; see
 * pyg_plan_suggest_col_block), exchange PYG_EXCHANGE_*.  Builds the global plan and its slice, the
 * halo and its request lists (exchanged over NCCL), and the transposed plan of the local edges.
 * SYNCHRONOUS, collective.  PYG_ERR_UNSUPPORTED for the halo with col_block > 0. */
pyg_status_t pyg_dist_plan_build(pyg_dist_t* comm, const int64_t* edge_index, int64_t E, int64_t n, int64_t F,
                                 int64_t ld, int64_t col_block, int exchange, pyg_dist_plan_t** plan,
                                 void* stream);
pyg_status_t pyg_dist_plan_info(const pyg_dist_plan_t* plan, pyg_dist_plan_info_t* info);
void pyg_dist_plan_destroy(pyg_dist_plan_t* plan);
/* out [hi - lo x F] stride ldo (+ arg_out int64, same stride, GLOBAL edge ids, for MAX) = the rows
 * [lo, hi) of pyg_propagate over the whole graph (Eq. 1).  x_shard [hi - lo x F] stride ldx: this
 * rank's X rows (may be info.x_shard itself); edge_weight [E] by GLOBAL edge id or NULL.  flags:
 * PYG_NO_TMA (PYG_PHI_CONCAT_XI unsupported).  Asynchronous on `stream` (NCCL enqueues there too),
 * collective. */
pyg_status_t pyg_dist_propagate(pyg_dist_plan_t* plan, const float* x_shard, int64_t ldx, const float* edge_weight,
                                pyg_reduce_t reduce, uint32_t flags, float* out, int64_t ldo, int64_t* arg_out,
                                void* stream);
/* grad_x_shard [hi - lo x F] stride ldgx (overwritten) = the rows [lo, hi) of pyg_propagate_backward's
 * grad_x_src over the whole graph, from this rank's grad_out [hi - lo x F] (stride ldg) and, for MAX,
 * its arg_out (stride lda) from pyg_dist_propagate.  MEAN divides by the in-degree; MAX routes
 * through argmax with fp32 atomics (see pyg_propagate_backward).  Asynchronous, collective. */
pyg_status_t pyg_dist_propagate_backward(pyg_dist_plan_t* plan, const float* grad_out, int64_t ldg,
                                         const float* edge_weight, pyg_reduce_t reduce, const int64_t* arg_out,
                                         int64_t lda, float* grad_x_shard, int64_t ldgx, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* PYG_GS_H */
