// attention.cu -- NEXT-1: segment softmax and the GAT attention-weighted
// aggregation, "our own optimized sparse softmax kernels" of P:239 (GAT; S:161-169,
// S:421-429), on the same CSR plans as the segment-reduce.
//
// Every per-row kernel comes in two shapes over the plan's rows: a WARP per light row (rows of
// <= heavy_threshold positions, visited in the plan's degree-bucket order, longest first) and a
// 256-thread CTA per split hub row (power-law graphs: a 300k-position row would otherwise serialise
// one warp), with the same per-thread position assignment in both passes.
//
//   softmax_fwd_kernel   pass 1: online (max, sum of exp) per head over the row's logits (all H
//                        heads per position from one vector load of s_src[j]); a fixed-tree group
//                        reduction of the (max, sum) pairs; pass 2: alpha = exp(l - max) / sum,
//                        written per ORIGINAL edge id ([E x H], the backward needs it).  Logits are
//                        GAT's leaky_relu(s_src[j] + s_dst[i]) or caller-given values.
//   alpha-weighted sum   the segment-reduce kernels in mode kRedHeadW (weights alpha[eid][c / C]):
//                        forward (z over the forward plan) and grad_z (grad_out over the transposed
//                        plan) inherit the hub split, the fp64 combine and the tuned geometry.
//   softmax_bwd_kernel   pass A: d_alpha per edge (GAT: the SDDMM grad_out[i] . z[j] per head,
//                        thread per edge, grad_out[i] staged in shared memory) and
//                        t = sum alpha d_alpha; pass B: dL/dlogit = alpha (d_alpha - t) (times
//                        leaky_relu'(pre) for GAT), grad_s_dst = row sum.  grad_s_src is a segment
//                        sum of dL/dlogit over the transposed plan (gathered by edge id).
// All deterministic (fixed per-row order and reduction trees).
#include "kernels.cuh"

namespace pyg {

namespace {

constexpr int kMaxHeads = 8;
constexpr int64_t kShortRow = 16;  // softmax rows up to this length use 8-lane groups

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// (max, sum-of-exp) pair merge; an empty side is (-inf, 0)
__device__ __forceinline__ void ms_merge(float& m, float& s, float m2, float s2) {
    const float M = fmaxf(m, m2);
    if (M == -INFINITY) return;
    s = s * expf(m - M) + s2 * expf(m2 - M);
    m = M;
}

// Group of G threads (32: one warp; 256: one CTA) reducing per-head values in a fixed tree.
template <int G>
struct Group {
    float* red;  // G == 256: shared scratch of 8 warps x kMaxHeads x 2 floats
    __device__ __forceinline__ void sum(float (&v)[kMaxHeads], int H) {
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) {
            if (h >= H) continue;
            if constexpr (G >= 32) {
                v[h] = warp_sum(v[h]);
            } else {
#pragma unroll
                for (int o = G / 2; o > 0; o >>= 1) v[h] += __shfl_xor_sync(0xffffffffu, v[h], o);
            }
        }
        if constexpr (G > 32) {
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            __syncthreads();
            if (lane == 0)
                for (int h = 0; h < H; ++h) red[w * kMaxHeads + h] = v[h];
            __syncthreads();
            for (int h = 0; h < H; ++h) {
                float t = 0.0f;
                for (int q = 0; q < G / 32; ++q) t += red[q * kMaxHeads + h];
                v[h] = t;
            }
        }
    }
    __device__ __forceinline__ void max_sum(float (&m)[kMaxHeads], float (&s)[kMaxHeads], int H) {
#pragma unroll
        for (int o = (G >= 32 ? 16 : G / 2); o > 0; o >>= 1)
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
                if (h >= H) continue;
                const float m2 = __shfl_xor_sync(0xffffffffu, m[h], o);
                const float s2 = __shfl_xor_sync(0xffffffffu, s[h], o);
                ms_merge(m[h], s[h], m2, s2);
            }
        if constexpr (G > 32) {
            const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
            __syncthreads();
            if (lane == 0)
                for (int h = 0; h < H; ++h) {
                    red[(w * kMaxHeads + h) * 2] = m[h];
                    red[(w * kMaxHeads + h) * 2 + 1] = s[h];
                }
            __syncthreads();
            for (int h = 0; h < H; ++h) {
                float mm = -INFINITY, ss = 0.0f;
                for (int q = 0; q < G / 32; ++q) ms_merge(mm, ss, red[(q * kMaxHeads + h) * 2], red[(q * kMaxHeads + h) * 2 + 1]);
                m[h] = mm;
                s[h] = ss;
            }
        }
    }
};

// the H (<= 8) per-head values of row `row` of a packed [n x H] array (vector loads when H is 2, 4, 8)
__device__ __forceinline__ void load_heads(float (&v)[kMaxHeads], const float* base, int64_t row, int H) {
    const float* p = base + row * H;
    if (H == 8) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
    } else if (H == 4) {
        const float4 a = __ldg(reinterpret_cast<const float4*>(p));
        v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
    } else {
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) v[h] = h < H ? __ldg(p + h) : 0.0f;
    }
}
__device__ __forceinline__ void store_heads(float* base, int64_t row, int H, const float (&v)[kMaxHeads]) {
    float* p = base + row * H;
    if (H == 8) {
        reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
        reinterpret_cast<float4*>(p)[1] = make_float4(v[4], v[5], v[6], v[7]);
    } else if (H == 4) {
        reinterpret_cast<float4*>(p)[0] = make_float4(v[0], v[1], v[2], v[3]);
    } else {
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < H) p[h] = v[h];
    }
}

struct RowSet {
    const int64_t* rowptr;      // this plan's rows (offset for slices)
    int64_t n_rows;
    const int32_t* order;       // light rows: root ids in degree-bucket order (or null: 0..n_rows)
    int64_t order_len, order_offset;
    int64_t thr;                // rows longer than this are hub rows
    int64_t dlo, dhi;           // light-row kernels: rows with dlo < degree <= dhi (and <= thr)
    const int32_t* heavy_rows;  // hub rows: root ids
    int64_t h_lo, h_hi, row_offset;
};

// the row a group works on in unit u (light: warp-granular; heavy: CTA-granular); -1: skip
template <int G>
__device__ __forceinline__ int64_t row_of(const RowSet& rs, int64_t u) {
    if constexpr (G <= 32) {
        int64_t r;
        if (rs.order) {
            if (u >= rs.order_len) return -2;
            r = (int64_t)rs.order[u] - rs.order_offset;
            if (r < 0 || r >= rs.n_rows) return -1;
        } else {
            if (u >= rs.n_rows) return -2;
            r = u;
        }
        const int64_t d = rs.rowptr[r + 1] - rs.rowptr[r];
        return (d == 0 || d > rs.thr || d <= rs.dlo || d > rs.dhi) ? -1 : r;
    } else {
        if (u >= rs.h_hi - rs.h_lo) return -2;
        return (int64_t)rs.heavy_rows[rs.h_lo + u] - rs.row_offset;
    }
}

struct SoftmaxArgs {
    const int32_t* col;   // GAT: source of each position
    const int32_t* eid;   // edge id per position (null -> position)
    const float* src;     // values mode: [E x H] stride lds
    int64_t lds;
    const float* s_src;   // GAT: [n_src x H] packed
    const float* s_dst;   // GAT: [n_rows x H] packed
    int H;
    float slope;
    float* alpha;         // [E x H] stride lda
    int64_t lda;
};

template <bool GAT>
__device__ __forceinline__ void logits(const SoftmaxArgs& a, int64_t p, int64_t k, const float (&sd)[kMaxHeads],
                                       float (&l)[kMaxHeads]) {
    if constexpr (GAT) {
        load_heads(l, a.s_src, a.col[p], a.H);
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) {
            const float pre = l[h] + sd[h];
            l[h] = pre > 0.0f ? pre : a.slope * pre;
        }
    } else {
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) l[h] = h < a.H ? __ldg(a.src + k * a.lds + h) : 0.0f;
    }
}

template <int G, bool GAT>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(SoftmaxArgs a, RowSet rs) {
    __shared__ float red[8 * kMaxHeads * 2];
    Group<G> grp{red};
    // G < 32: 32 / G rows per warp (short rows); the row loop stays warp-uniform (a group without a
    // row joins the shuffles with an empty range) because the reductions shuffle across the warp
    constexpr int GPW = G < 32 ? 32 / G : 1;
    const int t = G <= 32 ? (threadIdx.x & (G - 1)) : threadIdx.x;
    const int64_t units = G <= 32 ? (((int64_t)gridDim.x * blockDim.x) >> 5) : gridDim.x;
    int64_t u = G <= 32 ? (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) : blockIdx.x;
    for (;; u += units) {
        const int64_t r = row_of<G>(rs, G < 32 ? u * GPW + ((threadIdx.x & 31) / G) : u);
        if constexpr (G < 32) {
            if (__all_sync(0xffffffffu, r == -2)) break;
            if (__all_sync(0xffffffffu, r < 0)) continue;
        } else {
            if (r == -2) break;
            if (r < 0) continue;
        }
        const int64_t b = r >= 0 ? rs.rowptr[r] : 0, e = r >= 0 ? rs.rowptr[r + 1] : 0;
        float sd[kMaxHeads];
        if (GAT && r >= 0) load_heads(sd, a.s_dst, r, a.H);
        float m[kMaxHeads], s[kMaxHeads], l[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) { m[h] = -INFINITY; s[h] = 0.0f; }
        // (PU = 2 / 4 positions per step measured slower on R-MAT: softmax 21 -> 27 ms at PU = 4, the
        // register growth cost more warps than the extra gathers in flight gained; gpurun_out/r2h)
        constexpr int PU = 1;
        for (int64_t p0 = b + t; p0 < e; p0 += (int64_t)G * PU) {
            float lv[PU][kMaxHeads];
#pragma unroll
            for (int j = 0; j < PU; ++j) {
                const int64_t p = p0 + (int64_t)j * G;
                if (p < e) logits<GAT>(a, p, a.eid ? (int64_t)a.eid[p] : p, sd, lv[j]);
            }
#pragma unroll
            for (int j = 0; j < PU; ++j) {
                if (p0 + (int64_t)j * G >= e) continue;
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) {
                    if (h >= a.H) continue;
                    if (lv[j][h] > m[h]) { s[h] = s[h] * expf(m[h] - lv[j][h]) + 1.0f; m[h] = lv[j][h]; }
                    else s[h] += expf(lv[j][h] - m[h]);
                }
            }
        }
        grp.max_sum(m, s, a.H);
        for (int64_t p0 = b + t; p0 < e; p0 += (int64_t)G * PU) {
            float lv[PU][kMaxHeads];
            int64_t kv[PU];
#pragma unroll
            for (int j = 0; j < PU; ++j) {
                const int64_t p = p0 + (int64_t)j * G;
                kv[j] = p < e ? (a.eid ? (int64_t)a.eid[p] : p) : -1;
                if (p < e) logits<GAT>(a, p, kv[j], sd, lv[j]);
            }
#pragma unroll
            for (int j = 0; j < PU; ++j) {
                if (kv[j] < 0) continue;
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) l[h] = h < a.H ? expf(lv[j][h] - m[h]) / s[h] : 0.0f;
                if (a.lda == a.H) {
                    store_heads(a.alpha, kv[j], a.H, l);
                } else {
                    for (int h = 0; h < a.H; ++h) a.alpha[kv[j] * a.lda + h] = l[h];
                }
            }
        }
    }
}

struct SoftmaxBwdArgs {
    const int32_t* col;     // GAT: source per position
    const int32_t* eid;     // edge id per position (null -> position)
    int H, C, F;
    const float* alpha;     // [E x H] stride lda (values mode: the softmax output)
    int64_t lda;
    const float* grad;      // values mode: dL/dout [E x H] stride ldg; GAT: dL/dout [n_rows x F] stride ldg
    int64_t ldg;
    const float* z;         // GAT: [n_src x F] stride ldz
    int64_t ldz;
    const float* s_src;
    const float* s_dst;
    float slope;
    int vec;                // GAT: float4 dot products (F, C, ldz % 4 == 0, aligned)
    float* dlogit;          // [E x H] stride ldd (GAT: also the d_alpha scratch of pass A)
    int64_t ldd;
    float* grad_s_dst;      // GAT: [n_rows x H]
    const float* rs;        // GAT with factored alpha: alpha[k][h] / rs[row][h] is the coefficient (or null)
};

// the row's 1 / rs factors (all 1 when alpha is normalised), applied to every alpha load of the row
__device__ __forceinline__ void row_scale(float (&inv)[kMaxHeads], const float* rs, int64_t r, int H) {
    if (rs) {
        load_heads(inv, rs, r, H);
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) inv[h] = h < H ? 1.0f / inv[h] : 1.0f;
    } else {
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) inv[h] = 1.0f;
    }
}

template <int G, bool GAT>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(SoftmaxBwdArgs a, RowSet rs) {
    __shared__ float red[8 * kMaxHeads * 2];
    extern __shared__ float s_g[];  // GAT: grad_out row of the group's target, F floats per group
    Group<G> grp{red};
    const int t = G == 32 ? (threadIdx.x & 31) : threadIdx.x;
    float* sg = s_g + (G == 32 ? (int64_t)(threadIdx.x >> 5) * a.F : 0);
    const int64_t units = G == 32 ? (((int64_t)gridDim.x * blockDim.x) >> 5) : gridDim.x;
    int64_t u = G == 32 ? (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) : blockIdx.x;
    for (;; u += units) {
        const int64_t r = row_of<G>(rs, u);
        if (r == -2) break;
        if (r < 0) continue;
        const int64_t b = rs.rowptr[r], e = rs.rowptr[r + 1];
        float sd[kMaxHeads], inv[kMaxHeads];
        row_scale(inv, GAT ? a.rs : nullptr, r, a.H);
        if (GAT) {
            load_heads(sd, a.s_dst, r, a.H);
            if (G == 32) __syncwarp(); else __syncthreads();
            for (int c = t; c < a.F; c += G) sg[c] = a.grad[r * a.ldg + c];
            if (G == 32) __syncwarp(); else __syncthreads();
        }
        float tp[kMaxHeads], al[kMaxHeads], da[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) tp[h] = 0.0f;
        // pass A: d_alpha per edge and head, t = sum alpha * d_alpha
        for (int64_t p = b + t; p < e; p += G) {
            const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
            if constexpr (GAT) {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) da[h] = 0.0f;
                const float* zr = a.z + (int64_t)a.col[p] * a.ldz;
                if (a.vec) {
                    for (int c = 0; c < a.F; c += 4) {
                        const float4 zv = __ldg(reinterpret_cast<const float4*>(zr + c));
                        const int hh = c / a.C;
                        float d = sg[c] * zv.x;
                        d = fmaf(sg[c + 1], zv.y, d);
                        d = fmaf(sg[c + 2], zv.z, d);
                        d = fmaf(sg[c + 3], zv.w, d);
#pragma unroll
                        for (int h = 0; h < kMaxHeads; ++h)
                            if (h == hh) da[h] += d;
                    }
                } else {
                    for (int c = 0; c < a.F; ++c) {
                        const int hh = c / a.C;
                        const float d = sg[c] * __ldg(zr + c);
#pragma unroll
                        for (int h = 0; h < kMaxHeads; ++h)
                            if (h == hh) da[h] += d;
                    }
                }
                store_heads(a.dlogit, k, a.H, da);  // scratch, re-read by this thread in pass B
            } else {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) da[h] = h < a.H ? __ldg(a.grad + k * a.ldg + h) : 0.0f;
            }
            if (a.lda == a.H) {
                load_heads(al, a.alpha, k, a.H);
            } else {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) al[h] = h < a.H ? __ldg(a.alpha + k * a.lda + h) : 0.0f;
            }
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) al[h] *= inv[h];
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) tp[h] = fmaf(al[h], da[h], tp[h]);
        }
        grp.sum(tp, a.H);
        // pass B: dL/dlogit = alpha * (d_alpha - t) (* leaky_relu' for GAT); grad_s_dst = row sum
        float gs[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) gs[h] = 0.0f;
        for (int64_t p = b + t; p < e; p += G) {
            const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
            if constexpr (GAT) {
                float ss[kMaxHeads];
                load_heads(da, a.dlogit, k, a.H);
                load_heads(al, a.alpha, k, a.H);
                load_heads(ss, a.s_src, a.col[p], a.H);
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) {
                    float d = al[h] * inv[h] * (da[h] - tp[h]);
                    if (!(ss[h] + sd[h] > 0.0f)) d *= a.slope;
                    da[h] = d;
                    gs[h] += d;
                }
                store_heads(a.dlogit, k, a.H, da);
            } else {
                for (int h = 0; h < a.H; ++h)
                    a.dlogit[k * a.ldd + h] = __ldg(a.alpha + k * a.lda + h) * (__ldg(a.grad + k * a.ldg + h) - tp[h]);
            }
        }
        if constexpr (GAT) {
            grp.sum(gs, a.H);
            if (t == 0)
                for (int h = 0; h < a.H; ++h) a.grad_s_dst[r * a.H + h] = gs[h];
        }
        if (G > 32) __syncthreads();  // shared scratch reused by the next row
    }
}

// GAT backward, warp-cooperative SDDMM (C % 4 == 0 and C a power of two <= 128 or a multiple of
// 128; float4-aligned z / grad_out): a warp walks 32-position windows of its row, loading U z rows
// at a time with lane l holding float4 chunk (l + 32 ch) of a row (coalesced), dotted with the
// lane's chunk of grad_out[i] (registers, loaded once per row) and reduced over the C/4 lanes of
// each head by a butterfly; the per-(position, head) d_alpha goes through shared memory to the
// lane owning the position, which continues exactly like softmax_bwd_kernel (same position
// assignment, so pass B is shared).
template <int G, int NCH>
__global__ void __launch_bounds__(256) gat_bwd_coop_kernel(SoftmaxBwdArgs a, RowSet rs) {
    // G = 8: 8-lane subgroups, one short row each (4 rows per warp); G = 32: a warp per row;
    // G = 256: a CTA per hub row, each warp a subgroup walking every 8th 32-position window.
    constexpr int LS = G >= 32 ? 32 : G;       // lanes per subgroup (one window = LS positions)
    constexpr int GPW = G < 32 ? 32 / G : 1;   // rows per warp
    __shared__ float red[8 * kMaxHeads * 2];
    __shared__ float sda[8][32 * kMaxHeads];
    constexpr int U = NCH >= 8 ? 1 : 8 / NCH;
    Group<G> grp{red};
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    const int sl = lane & (LS - 1);            // lane within the subgroup
    const int sbase = lane & ~(LS - 1);        // first lane of the subgroup
    const int t = G <= 32 ? sl : threadIdx.x;
    float* sd_w = sda[wib] + sbase * kMaxHeads;
    const int CL = a.C >= 4 * LS ? LS : a.C / 4;  // lanes sharing a head inside one chunk row
    int hch[NCH];
    bool cvalid[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int c = 4 * (sl + LS * ch);
        cvalid[ch] = c < a.F;
        hch[ch] = cvalid[ch] ? c / a.C : 0;
    }
    const bool leader = (sl % CL) == 0;
    const int64_t units = G <= 32 ? (((int64_t)gridDim.x * blockDim.x) >> 5) : gridDim.x;
    int64_t u = G <= 32 ? (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) : blockIdx.x;
    for (;; u += units) {
        // warp-uniform row loop (the subgroups of a warp shuffle together)
        const int64_t r = row_of<G>(rs, G < 32 ? u * GPW + lane / LS : u);
        if constexpr (G < 32) {
            if (__all_sync(0xffffffffu, r == -2)) break;
            if (__all_sync(0xffffffffu, r < 0)) continue;
        } else {
            if (r == -2) break;
            if (r < 0) continue;
        }
        const bool rok = r >= 0;
        const int64_t b = rok ? rs.rowptr[r] : 0, e = rok ? rs.rowptr[r + 1] : 0;
        float sd[kMaxHeads], inv[kMaxHeads];
        if (rok) load_heads(sd, a.s_dst, r, a.H);
        row_scale(inv, rok ? a.rs : nullptr, r, a.H);
        float4 gv[NCH];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            gv[ch] = (rok && cvalid[ch]) ? __ldg(reinterpret_cast<const float4*>(a.grad + r * a.ldg) + sl + LS * ch)
                                         : make_float4(0.f, 0.f, 0.f, 0.f);
        float tp[kMaxHeads], al[kMaxHeads], da[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) tp[h] = 0.0f;
        // pass A: windows of LS positions; this thread owns position w + sl
        const int64_t w_first = b + (G > 32 ? 32 * wib : 0);
        for (int64_t w = w_first; __any_sync(0xffffffffu, w < e); w += (G > 32 ? G : LS)) {
            const int64_t p = w + sl;
            const bool valid = p < e;
            const int j = valid ? a.col[p] : 0;
            const int64_t k = valid ? (a.eid ? (int64_t)a.eid[p] : p) : 0;
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) sd_w[sl * kMaxHeads + h] = 0.0f;
            __syncwarp();
            const int n = w < e ? (int)min((int64_t)LS, e - w) : 0;
            // warp-uniform trip count: the longest window of the warp's subgroups
            int nmax = n;
            if constexpr (G < 32) {
#pragma unroll
                for (int o = LS; o < 32; o <<= 1) nmax = max(nmax, __shfl_xor_sync(0xffffffffu, nmax, o));
            }
            for (int t0 = 0; t0 < nmax; t0 += U) {
                float4 zc[U][NCH];
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
                    const int jt = __shfl_sync(0xffffffffu, j, sbase + ((t0 + uu) & (LS - 1)));
                    const float4* zr = reinterpret_cast<const float4*>(a.z + (int64_t)jt * a.ldz);
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch)
                        zc[uu][ch] = (cvalid[ch] && t0 + uu < n) ? __ldg(zr + sl + LS * ch)
                                                                 : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int uu = 0; uu < U; ++uu) {
#pragma unroll
                    for (int ch = 0; ch < NCH; ++ch) {
                        float d = gv[ch].x * zc[uu][ch].x;
                        d = fmaf(gv[ch].y, zc[uu][ch].y, d);
                        d = fmaf(gv[ch].z, zc[uu][ch].z, d);
                        d = fmaf(gv[ch].w, zc[uu][ch].w, d);
                        for (int o = 1; o < CL; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                        if (leader && cvalid[ch] && t0 + uu < n) sd_w[(t0 + uu) * kMaxHeads + hch[ch]] += d;
                    }
                }
            }
            __syncwarp();
            if (valid) {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) da[h] = sd_w[sl * kMaxHeads + h];
                store_heads(a.dlogit, k, a.H, da);  // scratch, re-read by this thread in pass B
                load_heads(al, a.alpha, k, a.H);
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) tp[h] = fmaf(al[h] * inv[h], da[h], tp[h]);
            }
            __syncwarp();
        }
        grp.sum(tp, a.H);
        // pass B (as softmax_bwd_kernel): position p = b + t + i*G' is this thread's in both passes
        // (G' = LS for subgroups, G for the CTA)
        float gs[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) gs[h] = 0.0f;
        for (int64_t p = b + t; p < e; p += (G > 32 ? G : LS)) {
            const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
            float ss[kMaxHeads];
            load_heads(da, a.dlogit, k, a.H);
            load_heads(al, a.alpha, k, a.H);
            load_heads(ss, a.s_src, a.col[p], a.H);
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
                float d = al[h] * inv[h] * (da[h] - tp[h]);
                if (!(ss[h] + sd[h] > 0.0f)) d *= a.slope;
                da[h] = d;
                gs[h] += d;
            }
            store_heads(a.dlogit, k, a.H, da);
        }
        grp.sum(gs, a.H);
        if (t == 0 && rok)
            for (int h = 0; h < a.H; ++h) a.grad_s_dst[r * a.H + h] = gs[h];
        if (G > 32) __syncthreads();
    }
}

RowSet row_set(const pyg_plan* p) {
    RowSet rs;
    rs.rowptr = p->rowptr;
    rs.n_rows = p->n_rows;
    rs.order = p->row_order;
    rs.order_len = p->row_order ? p->order_len : p->n_rows;
    rs.order_offset = p->row_offset;
    const bool split = p->item_hi > p->item_lo && p->heavy_rows;
    rs.thr = split ? p->heavy_threshold : INT64_MAX;
    rs.dlo = 0;
    rs.dhi = INT64_MAX;
    rs.heavy_rows = p->heavy_rows;
    rs.h_lo = split ? p->h_lo : 0;
    rs.h_hi = split ? p->h_hi : 0;
    rs.row_offset = p->row_offset;
    return rs;
}

int warp_grid(int64_t units) { return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(units, 8), 148 * 8)); }
int cta_grid(int64_t units) { return (int)std::max<int64_t>(1, std::min<int64_t>(units, 148 * 8)); }

}  // namespace

pyg_status_t attention_softmax(const pyg_plan* plan, const int32_t* col, const int32_t* eid, const float* src,
                               int64_t lds, const float* s_src, const float* s_dst, int H, float slope, float* alpha,
                               int64_t lda, cudaStream_t s) {
    if (plan->n_rows <= 0 || H <= 0) return PYG_OK;
    if (H > kMaxHeads) return fail(PYG_ERR_UNSUPPORTED, "softmax: at most %d heads / columns", kMaxHeads);
    SoftmaxArgs a{col, eid, src, lds, s_src, s_dst, H, slope, alpha, lda};
    const RowSet rs = row_set(plan);
    const int64_t light = rs.order_len, heavy = rs.h_hi - rs.h_lo;
    // rows of <= kShortRow positions: 8-lane groups (4 rows per warp); longer light rows: a warp
    RowSet rs_short = rs, rs_long = rs;
    rs_short.dhi = kShortRow;
    rs_long.dlo = kShortRow;
    if (s_src) {
        softmax_fwd_kernel<8, true><<<warp_grid(cdiv(light, 4)), 256, 0, s>>>(a, rs_short);
        softmax_fwd_kernel<32, true><<<warp_grid(light), 256, 0, s>>>(a, rs_long);
        if (heavy > 0) { softmax_fwd_kernel<256, true><<<cta_grid(heavy), 256, 0, s>>>(a, rs); PYG_LAUNCHED(); }
    } else {
        softmax_fwd_kernel<8, false><<<warp_grid(cdiv(light, 4)), 256, 0, s>>>(a, rs_short);
        softmax_fwd_kernel<32, false><<<warp_grid(light), 256, 0, s>>>(a, rs_long);
        if (heavy > 0) { softmax_fwd_kernel<256, false><<<cta_grid(heavy), 256, 0, s>>>(a, rs); PYG_LAUNCHED(); }
    }
    PYG_LAUNCHED();
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t attention_softmax_bwd(const pyg_plan* plan, const int32_t* col, const int32_t* eid, int H, int C, int F,
                                   const float* alpha, int64_t lda, const float* grad, int64_t ldg, const float* z,
                                   int64_t ldz, const float* s_src, const float* s_dst, float slope, float* dlogit,
                                   int64_t ldd, float* grad_s_dst, cudaStream_t s, const float* row_sums) {
    if (plan->n_rows <= 0 || H <= 0) return PYG_OK;
    if (H > kMaxHeads) return fail(PYG_ERR_UNSUPPORTED, "softmax backward: at most %d heads / columns", kMaxHeads);
    SoftmaxBwdArgs a;
    a.rs = row_sums;
    a.col = col; a.eid = eid;
    a.H = H; a.C = C; a.F = F; a.alpha = alpha; a.lda = lda; a.grad = grad; a.ldg = ldg;
    a.z = z; a.ldz = ldz; a.s_src = s_src; a.s_dst = s_dst; a.slope = slope;
    a.vec = z && (F % 4 == 0) && (C % 4 == 0) && (ldz % 4 == 0) && !(reinterpret_cast<uintptr_t>(z) & 15);
    a.dlogit = dlogit; a.ldd = ldd; a.grad_s_dst = grad_s_dst;
    const RowSet rs = row_set(plan);
    const int64_t light = rs.order_len, heavy = rs.h_hi - rs.h_lo;
    const bool pow2 = C > 0 && (C & (C - 1)) == 0;
    const bool coop = z && a.vec && (ldg % 4 == 0) && !(reinterpret_cast<uintptr_t>(grad) & 15) &&
                      ((pow2 && C >= 4 && C <= 128) || C % 128 == 0) && F <= 1024;
    if (coop) {
        if (ldd != H || lda != H) return fail(PYG_ERR_INVALID_ARGUMENT, "internal: GAT backward arrays must be packed");
        const int nch = (int)cdiv(F, 128);
        // short rows (<= kShortRow positions) on 8-lane subgroups when a head's columns tile an
        // 8-lane chunk row (C a power of two <= 32 or a multiple of 32) and F <= 256
        const bool short8 = ((pow2 && C <= 32) || C % 32 == 0) && F <= 256;
        RowSet rs_long = rs;
        if (short8) {
            RowSet rs_short = rs;
            rs_short.dhi = kShortRow;
            rs_long.dlo = kShortRow;
            const int n8 = (int)cdiv(F, 32);
            auto g8 = [&](auto k8) {
                k8<<<warp_grid(cdiv(light, 4)), 256, 0, s>>>(a, rs_short);
                PYG_LAUNCHED();
            };
            if (n8 <= 1) g8(gat_bwd_coop_kernel<8, 1>);
            else if (n8 <= 2) g8(gat_bwd_coop_kernel<8, 2>);
            else if (n8 <= 4) g8(gat_bwd_coop_kernel<8, 4>);
            else g8(gat_bwd_coop_kernel<8, 8>);
        }
        auto go = [&](auto kl, auto kh) {
            kl<<<warp_grid(light), 256, 0, s>>>(a, rs_long);
            PYG_LAUNCHED();
            if (heavy > 0) { kh<<<cta_grid(heavy), 256, 0, s>>>(a, rs); PYG_LAUNCHED(); }
        };
        if (nch == 1) go(gat_bwd_coop_kernel<32, 1>, gat_bwd_coop_kernel<256, 1>);
        else if (nch == 2) go(gat_bwd_coop_kernel<32, 2>, gat_bwd_coop_kernel<256, 2>);
        else if (nch <= 4) go(gat_bwd_coop_kernel<32, 4>, gat_bwd_coop_kernel<256, 4>);
        else go(gat_bwd_coop_kernel<32, 8>, gat_bwd_coop_kernel<256, 8>);
    } else if (z) {
        if (ldd != H || lda != H) return fail(PYG_ERR_INVALID_ARGUMENT, "internal: GAT backward arrays must be packed");
        const size_t smem_w = (size_t)8 * F * sizeof(float), smem_c = (size_t)F * sizeof(float);
        if (smem_w > 48 * 1024)
            PYG_CUDA(cudaFuncSetAttribute(softmax_bwd_kernel<32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem_w));
        softmax_bwd_kernel<32, true><<<warp_grid(light), 256, smem_w, s>>>(a, rs);
        PYG_LAUNCHED();
        if (heavy > 0) { softmax_bwd_kernel<256, true><<<cta_grid(heavy), 256, smem_c, s>>>(a, rs); PYG_LAUNCHED(); }
    } else {
        softmax_bwd_kernel<32, false><<<warp_grid(light), 256, 0, s>>>(a, rs);
        PYG_LAUNCHED();
        if (heavy > 0) { softmax_bwd_kernel<256, false><<<cta_grid(heavy), 256, 0, s>>>(a, rs); PYG_LAUNCHED(); }
    }
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
