// segment.cu -- CSR (target-sorted) segment-reduce: the deterministic strategy for
// the scatter-reduce BOX of Eq. (1), fused with the gather of x_j and phi
// (Fig. 1) so the E x F edge space is never materialised.
//
// Mapping (sm_100a, 148 SMs, HBM-bound):
//   * one group of `lpr` lanes (4..32, power of two) owns one target row;
//     lane l owns vector chunks q = l + ch*lpr (ch < NCH) of V floats each, so a
//     row of F floats is covered by lpr*NCH*V columns per column tile
//     (blockIdx.y tiles wider rows);
//   * the group loads the row's (gathered id, edge id, scale) for lpr positions
//     at once, coalesced, and broadcasts them with shuffles;
//   * U consecutive edges' row vectors are loaded before any is accumulated, so
//     each lane keeps U*NCH independent 8/16-byte loads in flight (memory-level
//     parallelism is what an HBM-bound random-row gather needs);
//   * accumulation is sequential in sorted position order => deterministic, and
//     for MAX the strict '>' keeps the lowest edge id among equal maxima (Q4);
//   * rows longer than kHeavyThreshold (R-MAT hubs) are split into chunks whose
//     fp32 partials are combined in fp64 by a second kernel (reading Q12).
#include "kernels.cuh"

namespace pyg {

namespace {

template <int NCH>
struct Unroll { static constexpr int U = NCH <= 2 ? 4 : (NCH <= 5 ? 2 : 1); };

__device__ __forceinline__ unsigned group_mask(int lpr) {
    if (lpr >= 32) return 0xffffffffu;
    int lane = threadIdx.x & 31;
    return ((1u << lpr) - 1u) << (lane & ~(lpr - 1));
}

// Accumulate positions [beg, end) of one segment into registers.
template <int V, int NCH, int RED>
__device__ __forceinline__ void seg_accumulate(const SegArgs& a, int64_t beg, int64_t end, int l,
                                               int lpr, unsigned mask, int c0,
                                               float (&acc)[NCH][V], int (&bi)[NCH][V]) {
    constexpr int U = Unroll<NCH>::U;
    const bool scaled = (a.w != nullptr) || (a.gdeg != nullptr);
    // the edge id is only needed for weights, argmax or edge-space rows
    const bool need_e = (RED == PYG_MAX) || (a.w != nullptr) || (a.gidx == nullptr);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int t = 0; t < V; ++t) {
            acc[ch][t] = (RED == PYG_MAX) ? -INFINITY : 0.0f;
            bi[ch][t] = -1;
        }
    bool cv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) cv[ch] = (c0 + (l + ch * lpr) * V) < a.ncols;

    for (int64_t base = beg; base < end; base += lpr) {
        const int n = (int)min((int64_t)lpr, end - base);
        int mg = 0, me = 0;
        float ms = 1.0f;
        if (l < n) {
            const int64_t p = base + l;
            me = (a.eid && need_e) ? __ldg(a.eid + p) : (int)p;
            mg = a.gidx ? __ldg(a.gidx + p) : me;
            if (a.w) ms = __ldg(a.w + me);
            if (a.gdeg) ms = ms / (float)__ldg(a.gdeg + mg);
        }
        int t = 0;
        for (; t + U <= n; t += U) {
            float v[U][NCH][V];
            float sv[U];
            int ev[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = __shfl_sync(mask, mg, t + u, lpr);
                sv[u] = __shfl_sync(mask, ms, t + u, lpr);
                ev[u] = __shfl_sync(mask, me, t + u, lpr);
                const float* row = a.X + (int64_t)g * a.ldx + c0;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    if (cv[ch]) ldv<V>(v[u][ch], row + (l + ch * lpr) * V);
                    else {
#pragma unroll
                        for (int q = 0; q < V; ++q) v[u][ch][q] = 0.0f;
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        if (RED == PYG_MAX) {
                            const float m = scaled ? __fmul_rn(sv[u], v[u][ch][q]) : v[u][ch][q];
                            if (bi[ch][q] < 0 || m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = ev[u]; }
                        } else {
                            acc[ch][q] = scaled ? fmaf(sv[u], v[u][ch][q], acc[ch][q])
                                                : acc[ch][q] + v[u][ch][q];
                        }
                    }
        }
        for (; t < n; ++t) {
            const int g = __shfl_sync(mask, mg, t, lpr);
            const float sc = __shfl_sync(mask, ms, t, lpr);
            const int e = __shfl_sync(mask, me, t, lpr);
            const float* row = a.X + (int64_t)g * a.ldx + c0;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                if (!cv[ch]) continue;
                float v[V];
                ldv<V>(v, row + (l + ch * lpr) * V);
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    if (RED == PYG_MAX) {
                        const float m = scaled ? __fmul_rn(sc, v[q]) : v[q];
                        if (bi[ch][q] < 0 || m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = e; }
                    } else {
                        acc[ch][q] = scaled ? fmaf(sc, v[q], acc[ch][q]) : acc[ch][q] + v[q];
                    }
                }
            }
        }
    }
}

// mode 0: light rows (skip rows longer than heavy_threshold), write out/arg
// mode 1: chunks of split rows, write fp32 partials (+ int32 arg partials)
template <int V, int NCH, int RED>
__global__ void __launch_bounds__(256) seg_kernel(SegArgs a, int lpr, int mode,
                                                  const int32_t* __restrict__ heavy_rows,
                                                  const int64_t* __restrict__ item_ptr,
                                                  int64_t h_lo, int64_t h_hi, int64_t item_lo,
                                                  int64_t n_items, int64_t row_offset, int chunk,
                                                  float* __restrict__ part,
                                                  int32_t* __restrict__ part_arg, int64_t ldp,
                                                  int out_vec_ok) {
    const int groups = blockDim.x / lpr;
    const int64_t gid = (int64_t)blockIdx.x * groups + threadIdx.x / lpr;
    const int l = threadIdx.x & (lpr - 1);
    const int c0 = blockIdx.y * (lpr * NCH * V);
    const unsigned mask = group_mask(lpr);

    int64_t beg, end, row = -1, item = -1;
    if (mode == 0) {
        if (gid >= a.n_rows) return;
        row = gid;
        beg = __ldg(a.rowptr + row);
        end = __ldg(a.rowptr + row + 1);
        if (end - beg > a.heavy_threshold) return;  // handled by the split path
    } else {
        if (gid >= n_items) return;
        item = item_lo + gid;
        // heavy row h owning this item: last h with item_ptr[h] <= item
        int64_t lo = h_lo, hi = h_hi - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (__ldg(item_ptr + mid) <= item) lo = mid; else hi = mid - 1;
        }
        const int64_t r = (int64_t)__ldg(heavy_rows + lo) - row_offset;
        const int64_t c = item - __ldg(item_ptr + lo);
        const int64_t rb = __ldg(a.rowptr + r), re = __ldg(a.rowptr + r + 1);
        beg = rb + c * chunk;
        end = min(beg + chunk, re);
    }

    float acc[NCH][V];
    int bi[NCH][V];
    seg_accumulate<V, NCH, RED>(a, beg, end, l, lpr, mask, c0, acc, bi);

    if (mode == 0) {
        const int64_t dseg = end - beg;
        // accumulate passes (source-blocked plans) have nothing to add for empty segments
        if (a.accum && dseg == 0 && !(RED == PYG_MEAN && a.finalize)) return;
        const int64_t dtot = (RED == PYG_MEAN && a.deg_total) ? (int64_t)__ldg(a.deg_total + row) : dseg;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int col = c0 + (l + ch * lpr) * V;
            if (col >= a.ncols) continue;
            const int nv = min(V, a.ncols - col);
            float* o = a.out + row * a.ldo + col;
            if (RED != PYG_MAX) {
                float r[V];
#pragma unroll
                for (int q = 0; q < V; ++q) r[q] = acc[ch][q];
                if (a.accum) {
#pragma unroll
                    for (int q = 0; q < V; ++q) if (q < nv) r[q] += o[q];
                }
                if (RED == PYG_MEAN && a.finalize) {
#pragma unroll
                    for (int q = 0; q < V; ++q) r[q] = dtot > 0 ? r[q] / (float)dtot : 0.0f;
                }
                if (out_vec_ok) stv<V>(o, r, nv);
                else {
#pragma unroll
                    for (int q = 0; q < V; ++q) if (q < nv) o[q] = r[q];
                }
            } else {
                int64_t* ap = a.arg + row * a.lda + col;
                if (!a.accum) {
                    float r[V];
#pragma unroll
                    for (int q = 0; q < V; ++q) r[q] = bi[ch][q] >= 0 ? acc[ch][q] : 0.0f;
                    if (out_vec_ok) stv<V>(o, r, nv);
                    else {
#pragma unroll
                        for (int q = 0; q < V; ++q) if (q < nv) o[q] = r[q];
                    }
#pragma unroll
                    for (int q = 0; q < V; ++q)
                        if (q < nv) ap[q] = bi[ch][q] >= 0 ? (int64_t)bi[ch][q] : a.E_sentinel;
                } else {
                    // merge with the previous blocks: larger value wins, IEEE-equal values -> lower edge id (Q4)
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        if (q >= nv || bi[ch][q] < 0) continue;
                        const int64_t oa = ap[q];
                        const float ov = o[q];
                        if (oa == a.E_sentinel || acc[ch][q] > ov || (acc[ch][q] == ov && bi[ch][q] < oa)) {
                            o[q] = acc[ch][q];
                            ap[q] = bi[ch][q];
                        }
                    }
                }
            }
        }
    } else {
        float* pp = part + gid * ldp;
        int32_t* pa = part_arg ? part_arg + gid * ldp : nullptr;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int col = c0 + (l + ch * lpr) * V;
            if (col >= a.ncols) continue;
            const int nv = min(V, a.ncols - col);
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (q < nv) {
                    pp[col + q] = acc[ch][q];
                    if (RED == PYG_MAX) pa[col + q] = bi[ch][q];
                }
        }
    }
}

// fp64 combine of the chunk partials of each split row (deterministic order).
template <int RED>
__global__ void combine_kernel(SegArgs a, const int32_t* __restrict__ heavy_rows,
                               const int64_t* __restrict__ item_ptr, int64_t h_lo,
                               int64_t item_lo, int64_t row_offset,
                               const float* __restrict__ part, const int32_t* __restrict__ part_arg,
                               int64_t ldp) {
    const int64_t h = h_lo + blockIdx.x;
    const int64_t r = (int64_t)heavy_rows[h] - row_offset;
    const int64_t i0 = item_ptr[h] - item_lo, i1 = item_ptr[h + 1] - item_lo;
    const int64_t deg = a.deg_total ? (int64_t)a.deg_total[r] : a.rowptr[r + 1] - a.rowptr[r];
    for (int col = blockIdx.y * blockDim.x + threadIdx.x; col < a.ncols; col += gridDim.y * blockDim.x) {
        if (RED == PYG_MAX) {
            float best = 0.0f;
            int b = -1;
            for (int64_t it = i0; it < i1; ++it) {
                const int pb = part_arg[it * ldp + col];
                const float pv = part[it * ldp + col];
                if (pb >= 0 && (b < 0 || pv > best)) { best = pv; b = pb; }
            }
            float* o = a.out + r * a.ldo + col;
            int64_t* ap = a.arg + r * a.lda + col;
            if (!a.accum) {
                *o = b >= 0 ? best : 0.0f;
                *ap = b >= 0 ? (int64_t)b : a.E_sentinel;
            } else if (b >= 0 && (*ap == a.E_sentinel || best > *o || (best == *o && b < *ap))) {
                *o = best;
                *ap = b;
            }
        } else {
            double s = 0.0;
            for (int64_t it = i0; it < i1; ++it) s += (double)part[it * ldp + col];
            if (a.accum) s += (double)a.out[r * a.ldo + col];
            if (RED == PYG_MEAN && a.finalize) s = deg > 0 ? s / (double)deg : 0.0;
            a.out[r * a.ldo + col] = (float)s;
        }
    }
}

constexpr int kNch[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16};

template <int V, int RED>
pyg_status_t launch_v(const SegArgs& a, int nch, int lpr, int tiles, int mode, const pyg_plan* p,
                      int64_t n_items, float* part, int32_t* part_arg, int64_t ldp, int out_vec_ok,
                      cudaStream_t s) {
    const int threads = 256;
    const int groups = threads / lpr;
    const int64_t units = mode == 0 ? a.n_rows : n_items;
    if (units <= 0) return PYG_OK;
    dim3 grid((unsigned)cdiv(units, groups), (unsigned)tiles);
    const int32_t* hr = p ? p->heavy_rows : nullptr;
    const int64_t* ip = p ? p->heavy_item_ptr : nullptr;
    const int64_t h_lo = p ? p->h_lo : 0, h_hi = p ? p->h_hi : 0;
    const int64_t item_lo = p ? p->item_lo : 0, row_off = p ? p->row_offset : 0;
    const int chunk = p ? p->chunk : kChunk;
#define PYG_SEG_CASE(N)                                                                         \
    case N:                                                                                     \
        seg_kernel<V, N, RED><<<grid, threads, 0, s>>>(a, lpr, mode, hr, ip, h_lo, h_hi,        \
                                                        item_lo, n_items, row_off, chunk, part, \
                                                        part_arg, ldp, out_vec_ok);             \
        break;
    switch (nch) {
        PYG_SEG_CASE(1) PYG_SEG_CASE(2) PYG_SEG_CASE(3) PYG_SEG_CASE(4) PYG_SEG_CASE(5)
        PYG_SEG_CASE(6) PYG_SEG_CASE(8) PYG_SEG_CASE(10) PYG_SEG_CASE(12) PYG_SEG_CASE(16)
        default: return fail(PYG_ERR_INVALID_ARGUMENT, "internal: bad NCH %d", nch);
    }
#undef PYG_SEG_CASE
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

template <int RED>
pyg_status_t launch_red(const SegArgs& a, int V, int nch, int lpr, int tiles, int mode,
                        const pyg_plan* p, int64_t n_items, float* part, int32_t* part_arg,
                        int64_t ldp, int ovk, cudaStream_t s) {
    if (V == 4) return launch_v<4, RED>(a, nch, lpr, tiles, mode, p, n_items, part, part_arg, ldp, ovk, s);
    if (V == 2) return launch_v<2, RED>(a, nch, lpr, tiles, mode, p, n_items, part, part_arg, ldp, ovk, s);
    return launch_v<1, RED>(a, nch, lpr, tiles, mode, p, n_items, part, part_arg, ldp, ovk, s);
}

bool aligned(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

}  // namespace

size_t segment_ws_bytes(const pyg_plan* plan, int64_t ncols, int reduce) {
    if (!plan) return 0;
    if (!plan->parts.empty()) {
        size_t b = 0;
        for (const auto& p : plan->parts) b = std::max(b, segment_ws_bytes(&p, ncols, reduce));
        return b;
    }
    const int64_t items = plan->item_hi - plan->item_lo;
    if (items <= 0) return 0;
    const size_t ldp = align_up((size_t)ncols, 4);
    size_t b = align_up((size_t)items * ldp * sizeof(float), 256);
    if (reduce == PYG_MAX) b += align_up((size_t)items * ldp * sizeof(int32_t), 256);
    return b;
}

static pyg_status_t segment_reduce_one(const SegArgs& a0, int reduce, const pyg_plan* plan, void* ws,
                                       size_t ws_bytes, cudaStream_t s);

// Source-blocked plans: one pass per block of source rows (sized so the block of X stays
// L2-resident), accumulating into `out` in block order (deterministic); the last pass applies
// the mean division with the total in-degree.
pyg_status_t segment_reduce(const SegArgs& a0, int reduce, const pyg_plan* plan, void* ws,
                            size_t ws_bytes, cudaStream_t s) {
    if (!plan || plan->parts.empty()) return segment_reduce_one(a0, reduce, plan, ws, ws_bytes, s);
    const size_t nb = plan->parts.size();
    for (size_t b = 0; b < nb; ++b) {
        SegArgs a = a0;
        const pyg_plan& p = plan->parts[b];
        a.rowptr = p.rowptr;
        a.accum = b > 0;
        a.finalize = (b + 1 == nb);
        a.deg_total = plan->deg;
        a.heavy_threshold = p.heavy_threshold;
        PYG_TRY(segment_reduce_one(a, reduce, &p, ws, ws_bytes, s));
    }
    return PYG_OK;
}

static pyg_status_t segment_reduce_one(const SegArgs& a0, int reduce, const pyg_plan* plan, void* ws,
                                       size_t ws_bytes, cudaStream_t s) {
    SegArgs a = a0;
    if (a.n_rows <= 0 || a.ncols <= 0) return PYG_OK;
    // vector width: X rows (and optionally padded reads) must be V-aligned
    int V = 1;
    for (int cand : {4, 2}) {
        const bool cols_ok = (a.ncols % cand == 0) || (a.allow_pad_read && cand == 4 &&
                                                       a.ldx >= (int64_t)align_up(a.ncols, 4));
        if (cols_ok && a.ldx % cand == 0 && aligned(a.X, 4 * cand)) { V = cand; break; }
    }
    const int out_vec_ok = (a.ldo % V == 0) && aligned(a.out, 4 * V);
    const int64_t nvec = cdiv(a.ncols, V);
    int lpr, nch, tiles;
    if (nvec <= 32) {
        lpr = 4;
        while (lpr < nvec) lpr <<= 1;
        nch = 1;
        tiles = 1;
    } else {
        lpr = 32;
        int64_t need = cdiv(nvec, 32);
        tiles = (int)cdiv(need, 16);
        need = cdiv(nvec, 32 * (int64_t)tiles);
        nch = 16;
        for (int c : kNch) if (c >= need) { nch = c; break; }
    }
    if (a.heavy_threshold <= 0) a.heavy_threshold = INT64_MAX;
    const bool split = plan && (plan->item_hi > plan->item_lo);
    if (!split) a.heavy_threshold = INT64_MAX;

    // light rows
    switch (reduce) {
        case PYG_SUM: PYG_TRY(launch_red<PYG_SUM>(a, V, nch, lpr, tiles, 0, plan, 0, nullptr, nullptr, 0, out_vec_ok, s)); break;
        case PYG_MEAN: PYG_TRY(launch_red<PYG_MEAN>(a, V, nch, lpr, tiles, 0, plan, 0, nullptr, nullptr, 0, out_vec_ok, s)); break;
        default: PYG_TRY(launch_red<PYG_MAX>(a, V, nch, lpr, tiles, 0, plan, 0, nullptr, nullptr, 0, out_vec_ok, s)); break;
    }
    if (!split) return PYG_OK;

    // split hub rows: chunk partials then fp64 combine
    const int64_t n_items = plan->item_hi - plan->item_lo;
    const int64_t ldp = (int64_t)align_up((size_t)a.ncols, 4);
    Carver cv(ws, ws_bytes);
    float* part = cv.take<float>((size_t)n_items * ldp);
    int32_t* part_arg = reduce == PYG_MAX ? cv.take<int32_t>((size_t)n_items * ldp) : nullptr;
    if (!ws || !cv.ok())
        return fail(PYG_ERR_NO_MEMORY, "workspace too small for %lld split-row chunks (need %zu bytes)",
                    (long long)n_items, segment_ws_bytes(plan, a.ncols, reduce));
    switch (reduce) {
        case PYG_SUM: PYG_TRY(launch_red<PYG_SUM>(a, V, nch, lpr, tiles, 1, plan, n_items, part, part_arg, ldp, out_vec_ok, s)); break;
        case PYG_MEAN: PYG_TRY(launch_red<PYG_MEAN>(a, V, nch, lpr, tiles, 1, plan, n_items, part, part_arg, ldp, out_vec_ok, s)); break;
        default: PYG_TRY(launch_red<PYG_MAX>(a, V, nch, lpr, tiles, 1, plan, n_items, part, part_arg, ldp, out_vec_ok, s)); break;
    }
    const int64_t n_heavy = plan->h_hi - plan->h_lo;
    dim3 grid((unsigned)n_heavy, (unsigned)cdiv(a.ncols, 256));
    switch (reduce) {
        case PYG_SUM: combine_kernel<PYG_SUM><<<grid, 256, 0, s>>>(a, plan->heavy_rows, plan->heavy_item_ptr, plan->h_lo, plan->item_lo, plan->row_offset, part, part_arg, ldp); break;
        case PYG_MEAN: combine_kernel<PYG_MEAN><<<grid, 256, 0, s>>>(a, plan->heavy_rows, plan->heavy_item_ptr, plan->h_lo, plan->item_lo, plan->row_offset, part, part_arg, ldp); break;
        default: combine_kernel<PYG_MAX><<<grid, 256, 0, s>>>(a, plan->heavy_rows, plan->heavy_item_ptr, plan->h_lo, plan->item_lo, plan->row_offset, part, part_arg, ldp); break;
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
