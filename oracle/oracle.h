/*
 * oracle.h -- plain, slow, single-threaded CPU oracle for the gather / phi /
 * scatter-reduce aggregation of Fey & Lenssen, "Fast Graph Representation
 * Learning with PyTorch Geometric" (arXiv 1903.02428).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and the
 * cpu_baseline / --impl reference legs of bench.py may load this library.
 * The product path (paper_1903_02428_b200/, libpygs.so) never includes,
 * links or calls anything in oracle/, and this file shares no code, enum or
 * constant with include/pyg_gs.h.
 *
 * Citations: P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n.
 * Readings of ambiguous passages (Q1..Q20) are listed in DESIGN.md.
 *
 * Conventions (all functions):
 *   - every array is host memory, row-major, packed unless a leading
 *     dimension is given;
 *   - edge_index is int64 [2 x E] row-major: row 0 = source j, row 1 =
 *     target i; messages flow j -> i (reading Q1);
 *   - floating point accumulation is in double and rounded to float once;
 *   - return value: ORC_OK or an ORC_ERR_* code; outputs are unspecified on
 *     error.
 */
#ifndef PYG_ORACLE_H
#define PYG_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { ORC_OK = 0, ORC_ERR_INVALID = 1, ORC_ERR_DIMENSION = 2, ORC_ERR_OOB = 3 };
enum { ORC_SUM = 0, ORC_MEAN = 1, ORC_MAX = 2 };

/* deg[i] = #{k : index[k] == i}; multi-edges and self-loops count (reading Q6). */
int orc_degree(const int64_t* index, int64_t E, int64_t n, int64_t* deg);

/* Stable counting sort of edge ids by target (CSR, row = target).
 * rowptr[n+1], perm[E]: perm lists the original edge ids of row i in
 * ascending order at perm[rowptr[i] .. rowptr[i+1]). */
int orc_csr(const int64_t* dst, int64_t E, int64_t n, int64_t* rowptr, int64_t* perm);

/* scatter(src, index, reduce).  src[E x F] with row
 * stride lds; out[dim_size x F] packed; arg[dim_size x F] (MAX only, else may
 * be NULL).  abs_sum[dim_size x F] (optional) = sum of |src| over each
 * segment, for the conditioned summation bound (reading Q11). */
int orc_scatter(const float* src, int64_t E, int64_t F, int64_t lds, const int64_t* index,
                int64_t dim_size, int reduce, float* out, int64_t* arg, double* abs_sum);

/* Eq. (1) without gamma: out[i] = BOX_{k : dst_k = i} phi(x_i, x_j, e_k)
 * (Fig. 1).  The message of edge k = (j -> i) is
 *   [ x_dst[i] (if concat_xi) || w_k * x_src[j] || edge_attr[k] (if D > 0) ]
 * with w_k = 1 when edge_weight is NULL.  F_out = (concat_xi ? F : 0) + F + D.
 * x_src[n_src x F] stride ldx; x_dst[n_dst x F] stride ldxd (NULL => x_src,
 * which then requires n_dst <= n_src); edge_attr[E x D] packed.
 * out[n_dst x F_out] packed; arg[n_dst x F_out] (MAX only).
 * abs_sum as in orc_scatter (optional). */
int orc_propagate(const float* x_src, int64_t n_src, int64_t F, int64_t ldx, const float* x_dst,
                  int64_t ldxd, int64_t n_dst, const int64_t* edge_index, int64_t E,
                  const float* edge_attr, int64_t D, const float* edge_weight, int reduce,
                  int concat_xi, float* out, int64_t* arg, double* abs_sum);

/* Backward of orc_scatter w.r.t. src: grad_src[E x F] packed from
 * grad_out[dim_size x F] packed.  arg required for MAX. */
int orc_scatter_backward(const float* grad_out, int64_t F, const int64_t* index, int64_t E,
                         int64_t dim_size, int reduce, const int64_t* arg, float* grad_src);

/* Backward of orc_propagate.  grad_out[n_dst x
 * F_out] packed; arg from the forward (MAX only).  Outputs (each optional,
 * NULL to skip), all overwritten:
 *   grad_x_src[n_src x F], grad_x_dst[n_dst x F] (concat_xi block),
 *   grad_edge_attr[E x D], grad_edge_weight[E].
 * abs_sum_x_src[n_src x F] (optional) = sum of |terms| for grad_x_src. */
int orc_propagate_backward(const float* x_src, int64_t n_src, int64_t F, int64_t ldx,
                           int64_t n_dst, const int64_t* edge_index, int64_t E, int64_t D,
                           const float* edge_weight, int reduce, int concat_xi,
                           const float* grad_out, const int64_t* arg, float* grad_x_src,
                           float* grad_x_dst, float* grad_edge_attr, float* grad_edge_weight,
                           double* abs_sum_x_src);

/* GCN normalisation D^-1/2 (A+I) D^-1/2.
 * Appends (i,i) with weight 1 for every node i in ascending order that has no
 * self-loop (existing loops kept; reading Q8), after the E original edges.
 * deg_hat[i] = sum of weights of edges with target i (reading Q7);
 * w'_k = deg_hat[src]^-1/2 * w_k * deg_hat[dst]^-1/2.
 * ei_src_out/ei_dst_out/w_out have capacity E + N; *E_out receives E'. */
int orc_gcn_norm(const int64_t* edge_index, int64_t E, int64_t N, const float* edge_weight,
                 int64_t* ei_src_out, int64_t* ei_dst_out, float* w_out, int64_t* E_out);

/* Block-diagonal mini-batch collate.  G graphs;
 * num_nodes[G]; edge_ptr[G+1] (graph g's edges are columns
 * edge_ptr[g] .. edge_ptr[g+1]) of local_ei[2 x Etot], Etot = edge_ptr[G],
 * ids local to their graph.  Writes ei[2 x Etot], batch[sum N_g],
 * node_ptr[G+1].  Errors: G <= 0 -> INVALID; local id outside [0, N_g) -> OOB. */
int orc_collate(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr,
                const int64_t* local_ei, int64_t* ei, int64_t* batch, int64_t* node_ptr);

/* Global add/mean/max pooling over the assignment vector (
 * S:478-486): out[G x F] = scatter(x, batch, reduce) with dim_size = G. */
int orc_global_pool(const float* x, int64_t N, int64_t F, const int64_t* batch, int64_t G,
                    int reduce, float* out, int64_t* arg);

/* NEXT-1: segment softmax ("optimized sparse
 * softmax kernels") over [E x H] values grouped by index, and its backward. */
int orc_segment_softmax(const float* src, int64_t E, int64_t H, const int64_t* index, int64_t n,
                        float* out);
int orc_segment_softmax_backward(const float* out, const float* grad, int64_t E, int64_t H,
                                 const int64_t* index, int64_t n, float* grad_src, double* abs_out);
/* GAT attention aggregation with H heads of C channels:
 * alpha = segment softmax over targets of leaky_relu(s_src[j] + s_dst[i]);
 * out[i] = sum alpha * z[j] per head; and its backward w.r.t. z, s_src, s_dst. */
int orc_gat(const float* z, int64_t n_src, int64_t H, int64_t C, const float* s_src,
            const float* s_dst, int64_t n_dst, const int64_t* ei, int64_t E, double slope,
            float* out, float* alpha_out, double* abs_out);
int orc_gat_backward(const float* z, int64_t n_src, int64_t H, int64_t C, const float* s_src,
                     const float* s_dst, int64_t n_dst, const int64_t* ei, int64_t E, double slope,
                     const float* g, float* grad_z, float* grad_s_src, float* grad_s_dst,
                     double* abs_z, double* abs_ssrc, double* abs_sdst);

/* NEXT-2: APPNP / SGC K-step propagation:
 * z_{k+1} = (1 - alpha) S z_k + alpha h, z_0 = h; out = z_K (double state). */
int orc_appnp(const float* h, int64_t n, int64_t F, const int64_t* ei, int64_t E,
              const float* edge_weight, int64_t K, double alpha, float* out);

/* NEXT-2: dense transform Y = diag(row_scale) X W^T + bias, double. */
int orc_dense_transform(const float* X, int64_t M, int64_t K, const float* W, int64_t N,
                        const float* bias, const float* row_scale, float* Y, double* abs_out);

#ifdef __cplusplus
}
#endif
#endif
