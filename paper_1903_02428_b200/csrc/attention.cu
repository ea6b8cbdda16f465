// attention.cu -- NEXT-1: segment softmax and the GAT attention-weighted
// aggregation, "our own optimized sparse softmax kernels" of P:239 (GAT; S:161-169,
// S:421-429), on the same CSR plans as the segment-reduce.
//
//   softmax_fwd_kernel   one warp per target row: per head, max, sum of exp, alpha = exp / sum
//                        (three passes over the row's logits; logits are GAT's
//                        leaky_relu(s_src[j] + s_dst[i]) or caller-given values); alpha is written
//                        per ORIGINAL edge id ([E x H]) because the backward needs it.
//   headw_kernel         one warp per row: out[r] = sum_p alpha[eid_p][head(c)] * X[gidx_p][c],
//                        the alpha window of 32 positions staged in shared memory; fp32 partial
//                        sums per 32-position window added into the row accumulator (chains of
//                        <= max(32, deg/32) terms, reading Q12).  Forward (X = z over the forward
//                        plan) and grad_z (X = grad_out over the transposed plan) alike.
//   softmax_bwd_kernel   one warp per target row: d_alpha per edge (GAT: the SDDMM
//                        grad_out[i] . z[j] per head, lane per edge, grad_out[i] staged in shared
//                        memory), t = sum alpha d_alpha, dL/dlogit = alpha (d_alpha - t), times
//                        leaky_relu' for GAT; grad_s_dst = row sum.  grad_s_src is a segment sum of
//                        dL/dlogit over the transposed plan (segment_reduce, gathered by edge id).
// All deterministic (fixed per-row order, fixed warp-reduction trees).  HBM/L2-bound like the
// segment-reduce: the z-row gather dominates (4*H*C bytes per edge).
#include "kernels.cuh"

namespace pyg {

namespace {

constexpr int kMaxHeads = 8;

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

struct SoftmaxArgs {
    const int64_t* rowptr;
    int64_t n_rows;
    const int32_t* col;   // GAT: source of each position
    const int32_t* eid;   // edge id per position (null -> position)
    const float* src;     // values mode: [E x H] stride lds
    int64_t lds;
    const float* s_src;   // GAT: [n_src x H]
    const float* s_dst;   // GAT: [n_rows x H]
    int H;
    float slope;
    float* alpha;         // [E x H] stride lda
    int64_t lda;
};

template <bool GAT>
__device__ __forceinline__ float logit(const SoftmaxArgs& a, int64_t r, int64_t p, int h) {
    if constexpr (GAT) {
        const float pre = __ldg(a.s_src + (int64_t)a.col[p] * a.H + h) + __ldg(a.s_dst + r * a.H + h);
        return pre > 0.0f ? pre : a.slope * pre;
    } else {
        const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
        return __ldg(a.src + k * a.lds + h);
    }
}

template <bool GAT>
__global__ void __launch_bounds__(256) softmax_fwd_kernel(SoftmaxArgs a) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n_rows; r += nw) {
        const int64_t b = a.rowptr[r], e = a.rowptr[r + 1];
        if (b == e) continue;
        for (int h = 0; h < a.H; ++h) {
            float m = -INFINITY;
            for (int64_t p = b + lane; p < e; p += 32) m = fmaxf(m, logit<GAT>(a, r, p, h));
            m = warp_max(m);
            float s = 0.0f;
            for (int64_t p = b + lane; p < e; p += 32) s += expf(logit<GAT>(a, r, p, h) - m);
            s = warp_sum(s);
            for (int64_t p = b + lane; p < e; p += 32) {
                const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
                a.alpha[k * a.lda + h] = expf(logit<GAT>(a, r, p, h) - m) / s;
            }
        }
    }
}

struct HeadwArgs {
    const int64_t* rowptr;
    int64_t n_rows;
    const int32_t* gidx;  // gathered row per position
    const int32_t* eid;   // edge id per position (null -> position)
    const float* X;
    int64_t ldx;
    int F, C, H;
    const float* alpha;   // [E x H] packed
    float* out;
    int64_t ldo;
};

// V floats per lane access (4: float4 when F % 4 == 0 and rows are 16-byte aligned; else 1);
// lane l owns columns [V*(l + 32*ch), +V) for ch < NCH.
template <int V, int NCH>
__global__ void __launch_bounds__(256) headw_kernel(HeadwArgs a) {
    __shared__ float s_alpha[8][32 * kMaxHeads];
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float* sa = s_alpha[wib];
    int hd[NCH][V];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const int c = V * (lane + 32 * ch) + q;
            hd[ch][q] = c < a.F ? c / a.C : 0;
        }
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n_rows; r += nw) {
        const int64_t b = a.rowptr[r], e = a.rowptr[r + 1];
        float acc[NCH][V];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) acc[ch][q] = 0.0f;
        for (int64_t w = b; w < e; w += 32) {
            const int64_t p = w + lane;
            int g = 0;
            if (p < e) {
                g = a.gidx[p];
                const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
                for (int h = 0; h < a.H; ++h) sa[lane * kMaxHeads + h] = __ldg(a.alpha + k * a.H + h);
            }
            __syncwarp();
            const int n = (int)min((int64_t)32, e - w);
            float wacc[NCH][V];
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int q = 0; q < V; ++q) wacc[ch][q] = 0.0f;
            for (int t = 0; t < n; ++t) {
                const int j = __shfl_sync(0xffffffffu, g, t);
                const float* xr = a.X + (int64_t)j * a.ldx;
                const float* at = sa + t * kMaxHeads;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const int c = V * (lane + 32 * ch);
                    if (c >= a.F) continue;
                    float v[V];
                    ldv<V>(v, xr + c);
#pragma unroll
                    for (int q = 0; q < V; ++q) wacc[ch][q] = fmaf(at[hd[ch][q]], v[q], wacc[ch][q]);
                }
            }
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int q = 0; q < V; ++q) acc[ch][q] += wacc[ch][q];
            __syncwarp();
        }
        float* o = a.out + r * a.ldo;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int c = V * (lane + 32 * ch);
            if (c < a.F) stv<V>(o + c, acc[ch], min(V, a.F - c));
        }
    }
}

struct SoftmaxBwdArgs {
    const int64_t* rowptr;
    int64_t n_rows;
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
};

template <bool GAT>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(SoftmaxBwdArgs a) {
    extern __shared__ float s_g[];  // GAT: grad_out row of the warp's target, F floats per warp
    const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
    float* sg = s_g + (GAT ? (int64_t)wib * a.F : 0);
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; r < a.n_rows; r += nw) {
        const int64_t b = a.rowptr[r], e = a.rowptr[r + 1];
        if (GAT) {
            __syncwarp();
            for (int c = lane; c < a.F; c += 32) sg[c] = a.grad[r * a.ldg + c];
            __syncwarp();
        }
        float tp[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) tp[h] = 0.0f;
        // pass A: d_alpha per edge and head, t = sum alpha * d_alpha
        for (int64_t p = b + lane; p < e; p += 32) {
            const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
            float da[kMaxHeads];
            if constexpr (GAT) {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) da[h] = 0.0f;
                const float* zr = a.z + (int64_t)a.col[p] * a.ldz;
                if (a.vec) {
                    for (int c = 0; c < a.F; c += 4) {
                        const float4 zv = __ldg(reinterpret_cast<const float4*>(zr + c));
                        const int hh = c / a.C;
                        float d = 0.0f;
                        d = fmaf(sg[c], zv.x, d);
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
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h)
                    if (h < a.H) a.dlogit[k * a.ldd + h] = da[h];
            } else {
#pragma unroll
                for (int h = 0; h < kMaxHeads; ++h) da[h] = h < a.H ? __ldg(a.grad + k * a.ldg + h) : 0.0f;
            }
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h)
                if (h < a.H) tp[h] = fmaf(__ldg(a.alpha + k * a.lda + h), da[h], tp[h]);
        }
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h)
            if (h < a.H) tp[h] = warp_sum(tp[h]);
        __syncwarp();  // pass A's d_alpha stores visible to the lanes re-reading them
        // pass B: dL/dlogit = alpha * (d_alpha - t) (* leaky_relu' for GAT); grad_s_dst = row sum
        float gs[kMaxHeads];
#pragma unroll
        for (int h = 0; h < kMaxHeads; ++h) gs[h] = 0.0f;
        for (int64_t p = b + lane; p < e; p += 32) {
            const int64_t k = a.eid ? (int64_t)a.eid[p] : p;
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
                if (h >= a.H) continue;
                const float da = GAT ? a.dlogit[k * a.ldd + h] : __ldg(a.grad + k * a.ldg + h);
                float d = __ldg(a.alpha + k * a.lda + h) * (da - tp[h]);
                if constexpr (GAT) {
                    const float pre = __ldg(a.s_src + (int64_t)a.col[p] * a.H + h) + __ldg(a.s_dst + r * a.H + h);
                    if (!(pre > 0.0f)) d *= a.slope;
                    gs[h] += d;
                }
                a.dlogit[k * a.ldd + h] = d;
            }
        }
        if constexpr (GAT) {
#pragma unroll
            for (int h = 0; h < kMaxHeads; ++h) {
                if (h >= a.H) continue;
                const float v = warp_sum(gs[h]);
                if (lane == 0) a.grad_s_dst[r * a.H + h] = v;
            }
        }
    }
}

int warp_grid(int64_t rows) {
    return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(rows, 8), 148 * 8));
}

template <int V>
pyg_status_t launch_headw(const HeadwArgs& a, cudaStream_t s) {
    const int nch = (int)cdiv(a.F, 32 * V);
    const int grid = warp_grid(a.n_rows);
    switch (nch) {
        case 1: headw_kernel<V, 1><<<grid, 256, 0, s>>>(a); break;
        case 2: headw_kernel<V, 2><<<grid, 256, 0, s>>>(a); break;
        case 3: headw_kernel<V, 3><<<grid, 256, 0, s>>>(a); break;
        case 4: headw_kernel<V, 4><<<grid, 256, 0, s>>>(a); break;
        case 5: headw_kernel<V, 5><<<grid, 256, 0, s>>>(a); break;
        case 6: headw_kernel<V, 6><<<grid, 256, 0, s>>>(a); break;
        case 7: headw_kernel<V, 7><<<grid, 256, 0, s>>>(a); break;
        case 8: headw_kernel<V, 8><<<grid, 256, 0, s>>>(a); break;
        default: return fail(PYG_ERR_UNSUPPORTED, "attention: feature width %d too large", a.F);
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace

pyg_status_t attention_headw(const int64_t* rowptr, int64_t n_rows, const int32_t* gidx, const int32_t* eid,
                             const float* X, int64_t ldx, int F, int C, int H, const float* alpha, float* out,
                             int64_t ldo, cudaStream_t s) {
    if (n_rows <= 0 || F <= 0) return PYG_OK;
    HeadwArgs a{rowptr, n_rows, gidx, eid, X, ldx, F, C, H, alpha, out, ldo};
    const bool v4 = (F % 4 == 0) && (ldx % 4 == 0) && (ldo % 4 == 0) && !(reinterpret_cast<uintptr_t>(X) & 15) &&
                    !(reinterpret_cast<uintptr_t>(out) & 15);
    if (v4) return launch_headw<4>(a, s);
    return launch_headw<1>(a, s);
}

pyg_status_t attention_softmax(const int64_t* rowptr, int64_t n_rows, const int32_t* col, const int32_t* eid,
                               const float* src, int64_t lds, const float* s_src, const float* s_dst, int H,
                               float slope, float* alpha, int64_t lda, cudaStream_t s) {
    if (n_rows <= 0 || H <= 0) return PYG_OK;
    SoftmaxArgs a{rowptr, n_rows, col, eid, src, lds, s_src, s_dst, H, slope, alpha, lda};
    if (s_src) softmax_fwd_kernel<true><<<warp_grid(n_rows), 256, 0, s>>>(a);
    else softmax_fwd_kernel<false><<<warp_grid(n_rows), 256, 0, s>>>(a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t attention_softmax_bwd(const int64_t* rowptr, int64_t n_rows, const int32_t* col, const int32_t* eid,
                                   int H, int C, int F, const float* alpha, int64_t lda, const float* grad, int64_t ldg,
                                   const float* z, int64_t ldz, const float* s_src, const float* s_dst, float slope,
                                   float* dlogit, int64_t ldd, float* grad_s_dst, cudaStream_t s) {
    if (n_rows <= 0 || H <= 0) return PYG_OK;
    SoftmaxBwdArgs a;
    a.rowptr = rowptr; a.n_rows = n_rows; a.col = col; a.eid = eid;
    a.H = H; a.C = C; a.F = F; a.alpha = alpha; a.lda = lda; a.grad = grad; a.ldg = ldg;
    a.z = z; a.ldz = ldz; a.s_src = s_src; a.s_dst = s_dst; a.slope = slope;
    a.vec = z && (F % 4 == 0) && (C % 4 == 0) && (ldz % 4 == 0) && !(reinterpret_cast<uintptr_t>(z) & 15);
    a.dlogit = dlogit; a.ldd = ldd; a.grad_s_dst = grad_s_dst;
    const int grid = warp_grid(n_rows);
    if (z) {
        const size_t smem = (size_t)8 * F * sizeof(float);
        if (smem > 48 * 1024)
            PYG_CUDA(cudaFuncSetAttribute(softmax_bwd_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          (int)smem));
        softmax_bwd_kernel<true><<<grid, 256, smem, s>>>(a);
    } else {
        softmax_bwd_kernel<false><<<grid, 256, 0, s>>>(a);
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
