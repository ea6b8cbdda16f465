// misc.cu -- the elementwise / per-edge kernels around the reduction:
//   the x_i block of the concatenated message, the backward
//   gathers and routings, GCN normalisation (
//   S:233-259), the block-diagonal collate and index
//   validation.  All are HBM-streaming kernels: grid-stride loops sized to a
//   multiple of the 148 SMs, coalesced along the feature dimension.
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

__global__ void xi_kernel(const float* __restrict__ x, int64_t ldx, int F, int64_t n,
                          const int64_t* __restrict__ rowptr, const int32_t* __restrict__ perm,
                          const int32_t* __restrict__ deg, const int32_t* __restrict__ first, int reduce,
                          float* out, int64_t ldo, int64_t* arg, int64_t lda, int64_t E) {
    GRID_STRIDE(t, n * F) {
        const int64_t i = t / F;
        const int c = (int)(t - i * F);
        int64_t d, f = E;
        if (rowptr) {
            const int64_t b = rowptr[i];
            d = rowptr[i + 1] - b;
            if (d > 0) f = perm ? (int64_t)perm[b] : b;
        } else {
            d = deg[i];
            if (d > 0 && first) f = first[i];
        }
        const float xv = x[i * ldx + c];
        float r;
        if (reduce == PYG_SUM) r = (float)d * xv;  // sum of d copies of x_i (exact product, one rounding)
        else r = d > 0 ? xv : 0.0f;                // mean of d copies / max of d copies
        out[i * ldo + c] = r;
        if (reduce == PYG_MAX) arg[i * lda + c] = d > 0 ? f : E;  // first (lowest) edge id: Q4
    }
}

__global__ void edge_gather_grad_kernel(const float* __restrict__ g, int64_t ldg, const int64_t* __restrict__ index,
                                        int64_t E, int F, int reduce, const int64_t* __restrict__ arg, int64_t lda,
                                        const int32_t* __restrict__ deg, float* out, int64_t ldo) {
    GRID_STRIDE(t, E * F) {
        const int64_t k = t / F;
        const int c = (int)(t - k * F);
        const int64_t i = index[k];
        const float gv = g[i * ldg + c];
        float r;
        if (reduce == PYG_SUM) r = gv;
        else if (reduce == PYG_MEAN) r = gv / (float)deg[i];  // IEEE divide
        else r = arg[i * lda + c] == k ? gv : 0.0f;
        out[k * ldo + c] = r;
    }
}

__global__ void xdst_grad_kernel(const float* __restrict__ g, int64_t ldg, int F, int64_t n,
                                 const int32_t* __restrict__ deg, const int64_t* __restrict__ arg, int64_t lda,
                                 int64_t E, int reduce, float* out, int64_t ldo) {
    GRID_STRIDE(t, n * F) {
        const int64_t i = t / F;
        const int c = (int)(t - i * F);
        const float gv = g[i * ldg + c];
        float r;
        if (reduce == PYG_SUM) r = (float)deg[i] * gv;
        else if (reduce == PYG_MEAN) r = deg[i] > 0 ? gv : 0.0f;
        else r = arg[i * lda + c] != E ? gv : 0.0f;
        out[i * ldo + c] = r;
    }
}

__global__ void max_route_kernel(const float* __restrict__ g, int64_t ldg, const int64_t* __restrict__ arg,
                                 int64_t lda, int F, int64_t n, const int64_t* __restrict__ src,
                                 const float* __restrict__ w, int64_t E, float* gx, int64_t ldgx) {
    GRID_STRIDE(t, n * F) {
        const int64_t i = t / F;
        const int c = (int)(t - i * F);
        const int64_t k = arg[i * lda + c];
        if (k < 0 || k >= E) continue;
        const float gv = g[i * ldg + c];
        const float v = w ? w[k] * gv : gv;
        atomicAdd(gx + src[k] * ldgx + c, v);
    }
}

// one warp per edge: dot(x_src[j], dL/dm_k) over the x_j block
__global__ void edge_weight_grad_kernel(const float* __restrict__ x, int64_t ldx, const float* __restrict__ g,
                                        int64_t ldg, const int64_t* __restrict__ arg, int64_t lda,
                                        const int64_t* __restrict__ ei, int64_t E, int F, int reduce,
                                        const int32_t* __restrict__ deg, float* gw) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < E; k += warps) {
        const int64_t j = ei[k], i = ei[E + k];
        float s = 0.0f;
        for (int c = lane; c < F; c += 32) {
            const float gv = g[i * ldg + c];
            const float xv = x[j * ldx + c];
            if (reduce == PYG_MAX) { if (arg[i * lda + c] == k) s = fmaf(xv, gv, s); }
            else s = fmaf(xv, gv, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) gw[k] = (reduce == PYG_MEAN) ? (deg[i] > 0 ? s / (float)deg[i] : 0.0f) : s;
    }
}

__global__ void validate_kernel(const int64_t* __restrict__ idx, int64_t n, int64_t lo, int64_t hi, int* flag) {
    GRID_STRIDE(t, n) {
        const int64_t v = idx[t];
        if (v < lo || v >= hi) *flag = 1;
    }
}

// ---- GCN normalisation ------------------------------------------------------------
__global__ void gcn_mark_loops(const int64_t* __restrict__ ei, int64_t E, int64_t N, int32_t* missing) {
    // missing[i] = 1 initially (set by memset-like fill), cleared for nodes with a loop
    GRID_STRIDE(k, E) {
        const int64_t s = ei[k], d = ei[E + k];
        if (s == d) missing[s] = 0;
    }
}
__global__ void fill_i32(int32_t* p, int64_t n, int32_t v) { GRID_STRIDE(t, n) p[t] = v; }
__global__ void gcn_total(const int32_t* missing, const int32_t* scan, int64_t N, int64_t E, int64_t* total) {
    *total = E + (N > 0 ? (int64_t)scan[N - 1] + missing[N - 1] : 0);
}
__global__ void gcn_write_edges(const int64_t* __restrict__ ei, int64_t E, int64_t N, const float* __restrict__ w,
                                const int32_t* __restrict__ missing, const int32_t* __restrict__ scan,
                                const int64_t* __restrict__ total, int64_t* eo, float* wo, double* deg) {
    const int64_t Eo = *total;
    GRID_STRIDE(t, E + N) {
        if (t < E) {
            const int64_t s = ei[t], d = ei[E + t];
            const float wk = w ? w[t] : 1.0f;
            eo[t] = s;
            eo[Eo + t] = d;
            wo[t] = wk;
            atomicAdd(deg + d, (double)wk);
        } else {
            const int64_t i = t - E;
            if (missing[i]) {
                const int64_t p = E + scan[i];  // appended in ascending node order (Q8)
                eo[p] = i;
                eo[Eo + p] = i;
                wo[p] = 1.0f;
                atomicAdd(deg + i, 1.0);
            }
        }
    }
}
__global__ void gcn_weights(const int64_t* __restrict__ eo, const int64_t* __restrict__ total,
                            const double* __restrict__ deg, float* wo) {
    const int64_t Eo = *total;
    GRID_STRIDE(k, Eo) {
        const double ds = deg[eo[k]], dd = deg[eo[Eo + k]];
        const double is = ds > 0 ? 1.0 / sqrt(ds) : 0.0;
        const double id = dd > 0 ? 1.0 / sqrt(dd) : 0.0;
        wo[k] = (float)(is * (double)wo[k] * id);  // fp64, one rounding
    }
}

// ---- collate ----------------------------------------------------------------------------
__global__ void scan_ptr_kernel(const int64_t* __restrict__ cnt, int64_t G, int64_t* ptr, int* flag) {
    // single block exclusive scan with carry; G is small (graphs per batch)
    __shared__ int64_t carry;
    __shared__ int64_t warp_sums[32];
    if (threadIdx.x == 0) { carry = 0; ptr[0] = 0; }
    __syncthreads();
    for (int64_t base = 0; base < G; base += blockDim.x) {
        const int64_t t = base + threadIdx.x;
        int64_t v = t < G ? cnt[t] : 0;
        if (v < 0) { if (flag) *flag = 2; v = 0; }
        // inclusive warp scan
        const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
        int64_t x = v;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int64_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) warp_sums[wid] = x;
        __syncthreads();
        if (wid == 0) {
            int64_t s = lane < (int)(blockDim.x >> 5) ? warp_sums[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int64_t y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            warp_sums[lane] = s;
        }
        __syncthreads();
        const int64_t incl = x + (wid > 0 ? warp_sums[wid - 1] : 0) + carry;
        if (t < G) ptr[t + 1] = incl;
        __syncthreads();
        if (threadIdx.x == blockDim.x - 1) carry = incl;
        __syncthreads();
    }
}

__device__ __forceinline__ int64_t owner(const int64_t* __restrict__ ptr, int64_t G, int64_t v) {
    // last g in [0, G) with ptr[g] <= v
    int64_t lo = 0, hi = G - 1;
    while (lo < hi) {
        const int64_t mid = (lo + hi + 1) >> 1;
        if (ptr[mid] <= v) lo = mid; else hi = mid - 1;
    }
    return lo;
}

__global__ void collate_edges(int64_t G, const int64_t* __restrict__ num_nodes, const int64_t* __restrict__ edge_ptr,
                              const int64_t* __restrict__ node_ptr, const int64_t* __restrict__ local, int64_t Et,
                              int64_t* ei, int* flag) {
    GRID_STRIDE(e, Et) {
        const int64_t g = owner(edge_ptr, G, e);
        const int64_t off = node_ptr[g], ng = num_nodes[g];
        const int64_t s = local[e], d = local[Et + e];
        if (flag && (s < 0 || s >= ng || d < 0 || d >= ng)) *flag = 1;
        ei[e] = s + off;  // block-diagonal offset
        ei[Et + e] = d + off;
    }
}

__global__ void collate_batch(int64_t G, const int64_t* __restrict__ node_ptr, int64_t Nt, int64_t* batch) {
    GRID_STRIDE(v, Nt) batch[v] = owner(node_ptr, G, v);  // assignment vector
}

__global__ void collate_check(int64_t G, const int64_t* edge_ptr, const int64_t* node_ptr, int64_t Et,
                              int64_t Nt, int* flag) {
    if (edge_ptr[0] != 0) *flag = 2;
    if (edge_ptr[G] != Et || node_ptr[G] != Nt) *flag = 2;
    for (int64_t g = 0; g < G; ++g)
        if (edge_ptr[g + 1] < edge_ptr[g]) *flag = 2;
}

}  // namespace

#define LAUNCH_CHECK()                  \
    do {                                \
        PYG_LAUNCHED();                 \
        PYG_CUDA(cudaGetLastError());   \
    } while (0)

pyg_status_t xi_block(const float* x, int64_t ldx, int F, int64_t n, const int64_t* rowptr, const int32_t* perm,
                      const int32_t* deg, const int32_t* first, int reduce, float* out, int64_t ldo, int64_t* arg,
                      int64_t lda, int64_t E, cudaStream_t s) {
    if (n <= 0 || F <= 0) return PYG_OK;
    xi_kernel<<<grid_for(n * F), 256, 0, s>>>(x, ldx, F, n, rowptr, perm, deg, first, reduce, out, ldo, arg, lda, E);
    LAUNCH_CHECK();
    return PYG_OK;
}

pyg_status_t edge_gather_grad(const float* g, int64_t ldg, const int64_t* index, int64_t E, int F, int reduce,
                              const int64_t* arg, int64_t lda, const int32_t* deg, float* out, int64_t ldo,
                              cudaStream_t s) {
    if (E <= 0 || F <= 0) return PYG_OK;
    edge_gather_grad_kernel<<<grid_for(E * F), 256, 0, s>>>(g, ldg, index, E, F, reduce, arg, lda, deg, out, ldo);
    LAUNCH_CHECK();
    return PYG_OK;
}

pyg_status_t xdst_grad(const float* g, int64_t ldg, int F, int64_t n, const int32_t* deg, const int64_t* arg,
                       int64_t lda, int64_t E, int reduce, float* out, int64_t ldo, cudaStream_t s) {
    if (n <= 0 || F <= 0) return PYG_OK;
    xdst_grad_kernel<<<grid_for(n * F), 256, 0, s>>>(g, ldg, F, n, deg, arg, lda, E, reduce, out, ldo);
    LAUNCH_CHECK();
    return PYG_OK;
}

__global__ void gather_by_index_kernel(const float* __restrict__ v, const int32_t* __restrict__ idx, int64_t n,
                                       float* __restrict__ out) {
    for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x)
        out[p] = __ldg(v + __ldg(idx + p));
}

pyg_status_t gather_by_index(const float* v, const int32_t* idx, int64_t n, float* out, cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    gather_by_index_kernel<<<grid_for(n), 256, 0, s>>>(v, idx, n, out);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t max_route_grad(const float* g, int64_t ldg, const int64_t* arg, int64_t lda, int F, int64_t n_dst,
                            const int64_t* src, const float* w, int64_t E, float* gx, int64_t ldgx, cudaStream_t s) {
    if (n_dst <= 0 || F <= 0) return PYG_OK;
    max_route_kernel<<<grid_for(n_dst * F), 256, 0, s>>>(g, ldg, arg, lda, F, n_dst, src, w, E, gx, ldgx);
    LAUNCH_CHECK();
    return PYG_OK;
}

pyg_status_t edge_weight_grad(const float* x, int64_t ldx, const float* g, int64_t ldg, const int64_t* arg,
                              int64_t lda, const int64_t* ei, int64_t E, int F, int reduce, const int32_t* deg,
                              float* gw, cudaStream_t s) {
    if (E <= 0) return PYG_OK;
    edge_weight_grad_kernel<<<grid_for(E * 32), 256, 0, s>>>(x, ldx, g, ldg, arg, lda, ei, E, F, reduce, deg, gw);
    LAUNCH_CHECK();
    return PYG_OK;
}

pyg_status_t fill_rows(float* out, int64_t ldo, int ncols, int64_t n, cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return PYG_OK;
    PYG_CUDA(cudaMemset2DAsync(out, ldo * 4, 0, (size_t)ncols * 4, (size_t)n, s));
    return PYG_OK;
}

pyg_status_t validate_index(const int64_t* idx, int64_t n, int64_t lo, int64_t hi, cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    validate_kernel<<<grid_for(n), 256, 0, s>>>(idx, n, lo, hi, validate_flag_dev());
    LAUNCH_CHECK();
    return PYG_OK;
}

// ---- GCN norm / collate host entry points (declared in api.cu via extern "C") ----------

pyg_status_t gcn_norm_impl(const int64_t* ei, int64_t E, int64_t N, const float* w, int64_t* eo, float* wo,
                           int64_t* E_out, void* ws, size_t bytes, cudaStream_t s, size_t* need) {
    Carver cv(ws, bytes);
    int32_t* missing = cv.take<int32_t>((size_t)std::max<int64_t>(N, 1));
    int32_t* scan = cv.take<int32_t>((size_t)std::max<int64_t>(N, 1));
    double* deg = cv.take<double>((size_t)std::max<int64_t>(N, 1));
    int64_t* total = cv.take<int64_t>(1);
    size_t cub_bytes = 0;
    cub::DeviceScan::ExclusiveSum(nullptr, cub_bytes, missing, scan, (int)std::max<int64_t>(N, 1));
    void* cub_tmp = cv.take<char>(cub_bytes);
    if (need) { *need = cv.off; return PYG_OK; }
    if (!ws || !cv.ok()) return fail(PYG_ERR_NO_MEMORY, "gcn_norm workspace too small");
    if (N > 0) {
        fill_i32<<<grid_for(N), 256, 0, s>>>(missing, N, 1);
        LAUNCH_CHECK();
        PYG_CUDA(cudaMemsetAsync(deg, 0, (size_t)N * sizeof(double), s));
    }
    if (E > 0) {
        gcn_mark_loops<<<grid_for(E), 256, 0, s>>>(ei, E, N, missing);
        LAUNCH_CHECK();
    }
    if (N > 0) {
        PYG_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, cub_bytes, missing, scan, (int)N, s));
        PYG_LAUNCHED();
    }
    gcn_total<<<1, 1, 0, s>>>(missing, scan, N, E, total);
    LAUNCH_CHECK();
    if (E + N > 0) {
        gcn_write_edges<<<grid_for(E + N), 256, 0, s>>>(ei, E, N, w, missing, scan, total, eo, wo, deg);
        LAUNCH_CHECK();
        gcn_weights<<<grid_for(E + N), 256, 0, s>>>(eo, total, deg, wo);
        LAUNCH_CHECK();
    }
    PYG_CUDA(cudaMemcpyAsync(E_out, total, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    PYG_CUDA(cudaStreamSynchronize(s));
    return PYG_OK;
}

pyg_status_t collate_impl(int64_t G, const int64_t* num_nodes, const int64_t* edge_ptr, const int64_t* local,
                          int64_t Et, int64_t Nt, uint32_t flags, int64_t* ei, int64_t* batch, int64_t* node_ptr,
                          cudaStream_t s) {
    if (flags & PYG_VALIDATE) validate_begin();
    int* flag = (flags & PYG_VALIDATE) ? validate_flag_dev() : nullptr;
    scan_ptr_kernel<<<1, 1024, 0, s>>>(num_nodes, G, node_ptr, flag);
    LAUNCH_CHECK();
    if (flags & PYG_VALIDATE) {
        collate_check<<<1, 1, 0, s>>>(G, edge_ptr, node_ptr, Et, Nt, flag);
        LAUNCH_CHECK();
        pyg_status_t st = validate_flag_check(s, "collate: sizes");
        if (st != PYG_OK) return PYG_ERR_DIMENSION;
    }
    if (Et > 0) {
        collate_edges<<<grid_for(Et), 256, 0, s>>>(G, num_nodes, edge_ptr, node_ptr, local, Et, ei, flag);
        LAUNCH_CHECK();
    }
    if (Nt > 0) {
        collate_batch<<<grid_for(Nt), 256, 0, s>>>(G, node_ptr, Nt, batch);
        LAUNCH_CHECK();
    }
    if (flags & PYG_VALIDATE) return validate_flag_check(s, "collate: local node id outside [0, N_g)");
    return PYG_OK;
}

}  // namespace pyg

// ---- global pooling readout (NEXT-3) -----------------------------------------------
// out[g] = BOX over the contiguous node segment [node_ptr[g], node_ptr[g+1]) of x.  The readout
// has few, long segments (64 point clouds x 1,024 nodes): a thread-block CLUSTER of 8 CTAs shares
// each segment, every CTA reducing one eighth of its rows (256 threads = 4 row stripes x 64
// columns), and the cluster's rank-0 CTA combines the 8 partials through distributed shared memory
// in rank order (fp64 for sum/mean; strict > for max, so ties keep the lowest node id).  One kernel,
// no workspace, deterministic.
#include <cooperative_groups.h>

namespace pyg {
namespace {

namespace cg = cooperative_groups;
constexpr int kPoolCluster = 8;
constexpr int kPoolCols = 64;      // columns per column tile (threads per row stripe)
constexpr int kPoolStripes = 4;    // row stripes per CTA

template <int RED>
__global__ void __cluster_dims__(1, kPoolCluster, 1) __launch_bounds__(256)
    pool_kernel(const float* __restrict__ x, int64_t ldx, int F, const int64_t* __restrict__ node_ptr,
                float* out, int64_t ldo, int64_t* arg, int64_t N) {
    cg::cluster_group cluster = cg::this_cluster();
    __shared__ double s_part[kPoolCols];   // this CTA's partial of the current column tile
    __shared__ float s_val[kPoolStripes][kPoolCols];
    __shared__ int64_t s_arg[kPoolStripes][kPoolCols];
    __shared__ int64_t s_parg[kPoolCols];
    const int g = blockIdx.x;
    const int rank = (int)cluster.block_rank();
    const int col_in = threadIdx.x % kPoolCols, stripe = threadIdx.x / kPoolCols;
    const int64_t b = node_ptr[g], e = node_ptr[g + 1];
    const int64_t len = e - b, chunk = (len + kPoolCluster - 1) / kPoolCluster;
    const int64_t cb = b + min(len, (int64_t)rank * chunk), ce = b + min(len, (int64_t)(rank + 1) * chunk);
    for (int c0 = 0; c0 < F; c0 += kPoolCols) {
        const int c = c0 + col_in;
        // 1. stripe partial over this CTA's rows
        float acc = RED == PYG_MAX ? -INFINITY : 0.0f;
        int64_t best = -1;
        if (c < F) {
            for (int64_t r = cb + stripe; r < ce; r += kPoolStripes) {
                const float v = __ldg(x + r * ldx + c);
                if (RED == PYG_MAX) {
                    if (v > acc) { acc = v; best = r; }  // rows ascend: strict > keeps the lowest id (Q4)
                } else {
                    acc += v;
                }
            }
        }
        s_val[stripe][col_in] = acc;
        s_arg[stripe][col_in] = best;
        __syncthreads();
        // 2. the CTA partial (stripes combined in order)
        if (stripe == 0) {
            if (RED == PYG_MAX) {
                float bv = s_val[0][col_in];
                int64_t ba = s_arg[0][col_in];
                for (int q = 1; q < kPoolStripes; ++q) {
                    const float v = s_val[q][col_in];
                    const int64_t av = s_arg[q][col_in];
                    if (av >= 0 && (ba < 0 || v > bv || (v == bv && av < ba))) { bv = v; ba = av; }
                }
                s_part[col_in] = bv;
                s_parg[col_in] = ba;
            } else {
                double t = 0.0;
                for (int q = 0; q < kPoolStripes; ++q) t += (double)s_val[q][col_in];
                s_part[col_in] = t;
            }
        }
        cluster.sync();  // every CTA's partial of this tile is visible cluster-wide
        // 3. rank 0 combines the cluster's partials in rank order (distributed shared memory)
        if (rank == 0 && stripe == 0 && c < F) {
            double t = 0.0, bv = 0.0;
            int64_t ba = -1;
            for (int q = 0; q < kPoolCluster; ++q) {
                const double v = *cluster.map_shared_rank(&s_part[col_in], q);
                if (RED == PYG_MAX) {
                    const int64_t av = *cluster.map_shared_rank(&s_parg[col_in], q);
                    if (av >= 0 && (ba < 0 || v > bv || (v == bv && av < ba))) { bv = v; ba = av; }
                } else {
                    t += v;
                }
            }
            float r;
            if (RED == PYG_MAX) {
                r = ba >= 0 ? (float)bv : 0.0f;
                arg[(int64_t)g * ldo + c] = ba >= 0 ? ba : N;
            } else if (RED == PYG_MEAN) {
                r = len > 0 ? (float)(t / (double)len) : 0.0f;
            } else {
                r = (float)t;
            }
            out[(int64_t)g * ldo + c] = r;
        }
        cluster.sync();  // rank 0 is done reading before the partials are overwritten / CTAs exit
    }
}

}  // namespace

pyg_status_t global_pool_impl(const float* x, int64_t ldx, int F, const int64_t* node_ptr, int64_t G, int reduce,
                              float* out, int64_t ldo, int64_t* arg, int64_t N, cudaStream_t s) {
    if (G <= 0 || F <= 0) return PYG_OK;
    if (G > 0x7fffffff) return fail(PYG_ERR_UNSUPPORTED, "global_pool: too many graphs");
    const dim3 grid((unsigned)G, kPoolCluster);
    switch (reduce) {
        case PYG_SUM: pool_kernel<PYG_SUM><<<grid, 256, 0, s>>>(x, ldx, F, node_ptr, out, ldo, arg, N); break;
        case PYG_MEAN: pool_kernel<PYG_MEAN><<<grid, 256, 0, s>>>(x, ldx, F, node_ptr, out, ldo, arg, N); break;
        default: pool_kernel<PYG_MAX><<<grid, 256, 0, s>>>(x, ldx, F, node_ptr, out, ldo, arg, N); break;
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
