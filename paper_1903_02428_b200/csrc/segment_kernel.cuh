// segment_kernel.cuh -- the CSR (target-sorted) segment-reduce kernel: the deterministic
// strategy for the scatter-reduce BOX of Eq. (1), fused with the gather of x_j
// and phi (Fig. 1) so the E x F edge space is never materialised.
//
// Mapping (sm_100a, 148 SMs, HBM/L2-bound):
//   * a group of LPR lanes (4..32, compile-time) owns one target row; lane l owns the
//     vector chunks q = l + ch*LPR (ch < NCH) of V floats (V = 1, 2, 4 or 8 -> 4..32-byte
//     loads; V = 8 is the sm_100 256-bit LDG.E.ENL2.256), so one column tile is
//     LPR*NCH*V floats wide (blockIdx.y tiles wider rows) and every chunk address is
//     `row base + compile-time offset`;
//   * the group loads the (gathered id, edge id, scale) of LPR positions at once,
//     coalesced, and broadcasts them with shuffles (scale / edge id only when used);
//   * U consecutive edges' rows are loaded before any is accumulated: U*NCH independent
//     loads in flight per lane (memory-level parallelism for a latency-bound gather);
//   * accumulation is sequential in sorted position order => deterministic; for MAX the
//     strict '>' keeps the lowest edge id among IEEE-equal maxima (reading Q4);
//   * rows longer than kHeavyThreshold (power-law hubs) are split into chunks whose fp32
//     partials are combined in fp64 by combine_kernel (reading Q12);
//   * accum/finalize let source-blocked plans add pass after pass into `out`.
#pragma once

#include <type_traits>

#include "kernels.cuh"

namespace pyg {
namespace seg {

template <int V>
__device__ __forceinline__ void ld(float (&r)[V], const float* p) {
    if constexpr (V == 8) {
        asm("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                     : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]),
                       "=f"(r[7])
                     : "l"(p));
    } else {
        ldv<V>(r, p);
    }
}

template <int V>
__device__ __forceinline__ void st(float* p, const float (&r)[V], int n, int vec_ok) {
    if constexpr (V == 8) {
        if (vec_ok && n == 8) {
            reinterpret_cast<float4*>(p)[0] = make_float4(r[0], r[1], r[2], r[3]);
            reinterpret_cast<float4*>(p)[1] = make_float4(r[4], r[5], r[6], r[7]);
            return;
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) if (q < n) p[q] = r[q];
    } else {
        if (vec_ok) {
            stv<V>(p, r, n);
            return;
        }
#pragma unroll
        for (int q = 0; q < V; ++q) if (q < n) p[q] = r[q];
    }
}

// edges whose rows are loaded before accumulation: ~40 floats of loads in flight per lane
template <int V, int NCH, int LPR>
struct Unroll {
    static constexpr int T0 = (V == 8 ? 32 : 40) / (NCH * V);
    static constexpr int T = T0 < 1 ? 1 : (T0 > 8 ? 8 : T0);
    static constexpr int U = T < LPR ? T : LPR;
};

template <int LPR>
__device__ __forceinline__ unsigned group_mask() {
    if constexpr (LPR >= 32) {
        return 0xffffffffu;
    } else {
        const int lane = threadIdx.x & 31;
        return ((1u << LPR) - 1u) << (lane & ~(LPR - 1));
    }
}

#ifndef PYG_MAX_PACK
#define PYG_MAX_PACK 1
#endif
#ifndef PYG_SEG_PERSIST
#define PYG_SEG_PERSIST 0
#endif
#if PYG_SEG_PERSIST
#define PYG_SEG_SKIP continue
#else
#define PYG_SEG_SKIP return
#endif
#ifndef PYG_MAX_U
#define PYG_MAX_U 1
#endif
#ifndef PYG_MAX_FRONT
#define PYG_MAX_FRONT 1
#endif

// MAX of a wide segment (17-20 floats per lane, e.g. Reddit's 602 columns) with the argmax kept as a
// 16-bit position inside the segment, two per register (segments are <= 2048 positions: light rows
// and 512-position hub chunks), so U edges can be in flight per lane at the SUM instantiation's
// occupancy; the positions become edge ids once, at the end.  With 10 registers freed the plain
// (unweighted) MAX instantiation also drops the x1 multiply without spilling (Reddit max, 11 passes:
// 23.8 -> 22.6 ms, gpurun_out/r2u; more edges in flight per lane measured slower: U = 2 at 2 CTAs/SM
// 27.3 ms, U = 3 37.2 ms; splitting the 602 columns over 2 / 3 column tiles of 12 / 8 floats per lane
// with U = 2 measured 27.9 / 32.9 ms, gpurun_out/r2ac).
template <int V, int NCH, int RED, int LPR>
__device__ __forceinline__ void accumulate_max_packed(const SegArgs& a, int64_t beg, int64_t end, int l, int c0,
                                                      float (&acc)[NCH][V], int (&bi)[NCH][V]) {
    static_assert(V % 2 == 0, "packed positions pair up vector elements");
    constexpr int U = PYG_MAX_U;
    const unsigned mask = group_mask<LPR>();
    const int32_t* __restrict__ gidx = a.gidx;
    const int32_t* __restrict__ eid = a.eid;
    const float* __restrict__ w = a.w;
    uint32_t bp[NCH][V / 2];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
#pragma unroll
        for (int q = 0; q < V; ++q) acc[ch][q] = -INFINITY;
#pragma unroll
        for (int q = 0; q < V / 2; ++q) bp[ch][q] = 0xffffffffu;
    }
    const int lane_off = c0 + l * V;
    bool cv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) cv[ch] = lane_off + ch * LPR * V < a.ncols;
    const char* __restrict__ Xl = reinterpret_cast<const char*>(a.X + lane_off);
    const uint32_t row_bytes = (uint32_t)(a.ldx * 4);
    float v[U][NCH][V];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) v[u][ch][q] = 0.0f;
    auto take = [&](const float (&vv)[NCH][V], float sc, uint32_t pos) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) {
                const float m = RED == kRedMaxW ? __fmul_rn(sc, vv[ch][q]) : vv[ch][q];
                if (m > acc[ch][q]) {  // acc starts at -inf (Q5: finite inputs); strict > keeps the lowest id
                    acc[ch][q] = m;
                    // one byte permute (PRMT) inserts pos into the element's 16-bit half
                    bp[ch][q / 2] = __byte_perm(bp[ch][q / 2], pos, (q & 1) ? 0x5410u : 0x3254u);
                }
            }
    };
    // all chunks but the last are full for every lane when the tile reaches that far (Reddit: 4 of 5):
    // a compile-time-true load predicate for them, so the loop does not rematerialise per-chunk column
    // checks under the 80-register cap
    const bool front_full = PYG_MAX_FRONT && (a.ncols >= c0 + (NCH - 1) * LPR * V);
    auto run = [&](auto front) {
    constexpr bool FRONT = decltype(front)::value;
    for (int64_t base = beg; base < end; base += LPR) {
        const int n = (int)min((int64_t)LPR, end - base);
        int mg = 0;
        float ms = 1.0f;
        if (l < n) {
            const int64_t p = base + l;
            mg = __ldg(gidx + p);
            if (RED == kRedMaxW) ms = __ldg(w + (eid ? (int64_t)__ldg(eid + p) : p));
        }
        const uint32_t pos0 = (uint32_t)(base - beg);
        int t = 0;
        for (; t + U <= n; t += U) {
            float sv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = __shfl_sync(mask, mg, t + u, LPR);
                sv[u] = RED == kRedMaxW ? __shfl_sync(mask, ms, t + u, LPR) : 1.0f;
                const float* row = reinterpret_cast<const float*>(Xl + (uint64_t)(uint32_t)g * row_bytes);
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    if ((FRONT && ch < NCH - 1) || cv[ch]) ld<V>(v[u][ch], row + ch * LPR * V);
            }
#pragma unroll
            for (int u = 0; u < U; ++u) take(v[u], sv[u], pos0 + (uint32_t)(t + u));
        }
        for (; t < n; ++t) {
            const int g = __shfl_sync(mask, mg, t, LPR);
            const float sc = RED == kRedMaxW ? __shfl_sync(mask, ms, t, LPR) : 1.0f;
            const float* row = reinterpret_cast<const float*>(Xl + (uint64_t)(uint32_t)g * row_bytes);
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if ((FRONT && ch < NCH - 1) || cv[ch]) ld<V>(v[0][ch], row + ch * LPR * V);
            take(v[0], sc, pos0 + (uint32_t)t);
        }
    }
    };
    if (front_full) run(std::true_type{});
    else run(std::false_type{});
    // positions -> edge ids (0xffff: no edge yet)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < V; ++q) {
            const uint32_t pos = (bp[ch][q / 2] >> (16 * (q & 1))) & 0xffffu;
            const int64_t p = beg + (int64_t)pos;
            bi[ch][q] = pos == 0xffffu ? -1 : (eid ? __ldg(eid + p) : (int)p);
        }
}

// Accumulate positions [beg, end) of one segment into registers.
template <int V, int NCH, int RED, int LPR>
__device__ __forceinline__ void accumulate(const SegArgs& a, int64_t beg, int64_t end, int l, int c0,
                                           float (&acc)[NCH][V], int (&bi)[NCH][V]) {
    if constexpr (PYG_MAX_PACK && (RED == PYG_MAX || RED == kRedMaxW) && V % 2 == 0 && V * NCH > 16 &&
                  V * NCH <= 20) {
        // 16-bit positions (0xffff = none): plans split rows above 2,048 positions (segment_reduce_one
        // refuses MAX without a plan), so a segment is always shorter
        accumulate_max_packed<V, NCH, RED, LPR>(a, beg, end, l, c0, acc, bi);
        return;
    }
    // MAX keeps an edge id per element besides the value: for 17-20 floats per lane one edge in flight per
    // lane keeps the kernel at the SUM instantiation's resident CTAs (wider shapes would spill) (Reddit max: 29.8 -> 23.8 ms, gpurun_out/r2e;
    // occupancy beats per-warp memory-level parallelism for this L2-latency-bound gather)
    constexpr bool IS_MAX = RED == PYG_MAX || RED == kRedMaxW;
    constexpr int U = (IS_MAX && V * NCH > 16 && V * NCH <= 20) ? 1 : Unroll<V, NCH, LPR>::U;
    const unsigned mask = group_mask<LPR>();
    const float* __restrict__ X = a.X;
    const int64_t ldx = a.ldx;
    const int32_t* __restrict__ gidx = a.gidx;
    const int32_t* __restrict__ eid = a.eid;
    const float* __restrict__ w = a.w;
    const int32_t* __restrict__ gdeg = a.gdeg;
    const bool scaled = (w != nullptr) || (gdeg != nullptr);
    // the edge id is only needed for weights, argmax or edge-space rows
    const bool need_e = IS_MAX || (RED == kRedHeadW) || (w != nullptr) || (gidx == nullptr);
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
        for (int q = 0; q < V; ++q) {
            acc[ch][q] = IS_MAX ? -INFINITY : 0.0f;
            bi[ch][q] = -1;
        }
    const int lane_off = c0 + l * V;
    bool cv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) cv[ch] = lane_off + ch * LPR * V < a.ncols;
    // kRedHeadW: the head of each chunk (a V-chunk never straddles heads: hC % V == 0)
    int hch[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) hch[ch] = (RED == kRedHeadW && cv[ch]) ? (lane_off + ch * LPR * V) / a.hC : 0;
    const float* __restrict__ hw = a.hw;
    const int64_t hH = a.hH;
    // row address = base + g * row_bytes as one 32x32->64 IMAD.WIDE (row_bytes < 2^32, g < 2^31);
    // chunk offsets are compile-time immediates
    const char* __restrict__ Xl = reinterpret_cast<const char*>(X + lane_off);
    const uint32_t row_bytes = (uint32_t)(ldx * 4);
    // Loads of invalid chunks (columns >= ncols) are predicated off; their registers keep stale
    // values that only ever reach accumulators of columns that are never stored.
    float v[U][NCH][V];
#pragma unroll
    for (int u = 0; u < U; ++u)
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) v[u][ch][q] = 0.0f;

    for (int64_t base = beg; base < end; base += LPR) {
        const int n = (int)min((int64_t)LPR, end - base);
        int mg = 0, me = 0;
        float ms = 1.0f;
        if (l < n) {
            const int64_t p = base + l;
            me = (eid && need_e) ? __ldg(eid + p) : (int)p;
            mg = gidx ? __ldg(gidx + p) : me;
            if (w) ms = __ldg(w + me);
            if (gdeg) ms = ms / (float)__ldg(gdeg + mg);
        }
        int t = 0;
        for (; t + U <= n; t += U) {
            float sv[U];
            int ev[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int g = __shfl_sync(mask, mg, t + u, LPR);
                sv[u] = scaled ? __shfl_sync(mask, ms, t + u, LPR) : 1.0f;
                ev[u] = (IS_MAX || RED == kRedHeadW) ? __shfl_sync(mask, me, t + u, LPR) : 0;
                const float* row = reinterpret_cast<const float*>(Xl + (uint64_t)(uint32_t)g * row_bytes);
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    if (cv[ch]) ld<V>(v[u][ch], row + ch * LPR * V);
            }
#pragma unroll
            for (int u = 0; u < U; ++u)
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    const float hwv = (RED == kRedHeadW) ? __ldg(hw + (int64_t)ev[u] * hH + hch[ch]) : 1.0f;
#pragma unroll
                    for (int q = 0; q < V; ++q) {
                        if (IS_MAX) {
                            // m = w * x_j (s = 1 without weights: exact).  Dropping the multiply for the
                            // unweighted case was measured SLOWER on Reddit (27.7 vs 23.8 ms: ptxas then
                            // spills 208 instead of 72 bytes at 3 CTAs / SM), so both cases multiply
                            const float m = __fmul_rn(sv[u], v[u][ch][q]);
                            if (m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = ev[u]; }  // acc starts at -inf (Q5: finite inputs)
                        } else if (RED == kRedHeadW) {
                            acc[ch][q] = fmaf(hwv, v[u][ch][q], acc[ch][q]);
                        } else {
                            acc[ch][q] = fmaf(sv[u], v[u][ch][q], acc[ch][q]);  // s = 1 -> plain add
                        }
                    }
                }
        }
        for (; t < n; ++t) {
            const int g = __shfl_sync(mask, mg, t, LPR);
            const float sc = scaled ? __shfl_sync(mask, ms, t, LPR) : 1.0f;
            const int e = (IS_MAX || RED == kRedHeadW) ? __shfl_sync(mask, me, t, LPR) : 0;
            const float* row = reinterpret_cast<const float*>(Xl + (uint64_t)(uint32_t)g * row_bytes);
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if (cv[ch]) ld<V>(v[0][ch], row + ch * LPR * V);
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const float hwv = (RED == kRedHeadW) ? __ldg(hw + (int64_t)e * hH + hch[ch]) : 1.0f;
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    if (IS_MAX) {
                        const float m = __fmul_rn(sc, v[0][ch][q]);
                        if (m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = e; }
                    } else if (RED == kRedHeadW) {
                        acc[ch][q] = fmaf(hwv, v[0][ch][q], acc[ch][q]);
                    } else {
                        acc[ch][q] = fmaf(sc, v[0][ch][q], acc[ch][q]);
                    }
                }
            }
        }
    }
}

struct HeavyArgs {
    const int32_t* heavy_rows = nullptr;
    const int64_t* item_ptr = nullptr;
    int64_t h_lo = 0, h_hi = 0, item_lo = 0, n_items = 0, row_offset = 0;
    int chunk = 0;
    float* part = nullptr;
    int32_t* part_arg = nullptr;
    int64_t ldp = 0;
};

// mode 0: light rows (skip rows longer than heavy_threshold), write / accumulate out, arg
// mode 1: chunks of split rows, write fp32 partials (+ int32 arg partials)
// resident CTAs per SM requested from ptxas (caps registers at 65536 / (256 * MINB)): 3 (24 warps)
// measured best for the V*NCH <= 24 float/lane shapes; wider shapes get fewer to avoid spills
#ifndef PYG_SEG_MINB
#define PYG_SEG_MINB 3
#endif
#ifndef PYG_MAX_MINB
#define PYG_MAX_MINB 3
#endif
template <int V, int NCH, int RED>
struct MinBlocks {
    static constexpr bool packed_max =
        PYG_MAX_PACK && (RED == PYG_MAX || RED == kRedMaxW) && V % 2 == 0 && V * NCH > 16 && V * NCH <= 20;
    static constexpr int base = packed_max ? PYG_MAX_MINB : (V * NCH <= 24 ? PYG_SEG_MINB : (V * NCH <= 48 ? 2 : 1));
    // the head-weighted sum keeps a head index per chunk, narrow MAX an arg id per element: one CTA fewer
    static constexpr int value =
        (!packed_max && (RED == kRedHeadW || ((RED == PYG_MAX || RED == kRedMaxW) && !(V * NCH > 16 && V * NCH <= 20))) &&
         base > 1)
            ? base - 1
            : base;
};
// Epilogue of a light row (mode 0): write / accumulate into `out` (and `arg`), apply the mean divide,
// the GCN / APPNP extras and, for MAX over several passes, the packed-key merge / decode.  Shared by
// seg_kernel and the bulk-copy pipeline (segment_bulk.cuh).
template <int V, int NCH, int RED, int LPR>
__device__ __forceinline__ void row_epilogue(const SegArgs& a, int64_t row, int64_t dseg, int l, int c0,
                                             const float (&acc)[NCH][V], const int (&bi)[NCH][V], int out_vec_ok) {
    constexpr bool IS_MAX = RED == PYG_MAX || RED == kRedMaxW;
    // accumulate passes (source-blocked plans) have nothing to add for empty segments
    // the GCN / APPNP epilogue extras exist only in the kRedSumEpi instantiation, so the plain
    // SUM / MEAN kernels keep their register budget
    constexpr bool EPI = RED == kRedSumEpi;
    // MAX over several passes keeps packed (value, edge id) keys in `arg` until the last pass decodes
    // them, so the final pass visits every row too
    if (a.accum && dseg == 0 &&
        !((RED == PYG_MEAN || IS_MAX || (EPI && (a.blend || a.col_bias))) && a.finalize))
        return;
    const float rsc = (EPI && a.row_scale && a.finalize) ? __ldg(a.row_scale + row) : 1.0f;
    const int64_t dtot = (RED == PYG_MEAN && a.deg_total) ? (int64_t)__ldg(a.deg_total + row) : dseg;
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int col = c0 + l * V + ch * LPR * V;
        if (col >= a.ncols) continue;
        const int nv = min(V, a.ncols - col);
        float* o = a.out + row * a.ldo + col;
        if (!IS_MAX) {
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
            if (EPI && a.row_scale && a.finalize) {
#pragma unroll
                for (int q = 0; q < V; ++q) r[q] *= rsc;
            }
            if (EPI && a.blend && a.finalize) {
                const float* hb = a.blend + row * a.ldb + col;
#pragma unroll
                for (int q = 0; q < V; ++q) if (q < nv) r[q] = fmaf(a.blend_b, hb[q], a.blend_a * r[q]);
            }
            if (EPI && a.col_bias && a.finalize) {
#pragma unroll
                for (int q = 0; q < V; ++q) if (q < nv) r[q] += __ldg(a.col_bias + col + q);
            }
            st<V>(o, r, nv, out_vec_ok);
        } else {
            int64_t* ap = a.arg + row * a.lda + col;
            if (!a.accum && a.finalize) {  // one pass: write (value, arg)
                float r[V];
#pragma unroll
                for (int q = 0; q < V; ++q) r[q] = bi[ch][q] >= 0 ? acc[ch][q] : 0.0f;
                st<V>(o, r, nv, out_vec_ok);
#pragma unroll
                for (int q = 0; q < V; ++q)
                    if (q < nv) ap[q] = bi[ch][q] >= 0 ? (int64_t)bi[ch][q] : a.E_sentinel;
            } else {
                // several passes (source-blocked plans): the arg buffer holds the packed key
                // (ord(value) << 32 | ~edge id; 0 = no edge yet) so each pass merges with ONE 8-byte
                // read-modify-write -- larger value wins, IEEE-equal -> lower edge id (Q4) -- and the
                // last pass decodes it into (value, arg)
                unsigned long long* kp = reinterpret_cast<unsigned long long*>(ap);
#pragma unroll
                for (int q = 0; q < V; ++q) {
                    if (q >= nv) continue;
                    const unsigned long long nk = bi[ch][q] >= 0 ? max_key(acc[ch][q], (uint32_t)bi[ch][q]) : 0ull;
                    unsigned long long k = nk;
                    if (a.accum) {
                        const unsigned long long old = kp[q];
                        k = old > nk ? old : nk;
                        if (!a.finalize && k == old) continue;
                    }
                    if (a.finalize) {
                        o[q] = k ? ord2f((uint32_t)(k >> 32)) : 0.0f;
                        ap[q] = k ? (int64_t)(0xffffffffu - (uint32_t)(k & 0xffffffffu)) : a.E_sentinel;
                    } else {
                        kp[q] = k;
                    }
                }
            }
        }
    }
}

template <int V, int NCH, int RED, int LPR>
__global__ void __launch_bounds__(256, (MinBlocks<V, NCH, RED>::value)) seg_kernel(SegArgs a, int mode, HeavyArgs h,
                                                                                  int out_vec_ok) {
    constexpr int groups = 256 / LPR;
    const int l = threadIdx.x & (LPR - 1);
    const int c0 = blockIdx.y * (LPR * NCH * V);
    // PYG_SEG_PERSIST (A/B builds only; measured no gain on Reddit, gpurun_out/r2v): a grid of resident
    // CTAs whose groups stride over the rows; the default is one row per group
#if PYG_SEG_PERSIST
    const int64_t gstride = (int64_t)gridDim.x * groups;
    for (int64_t gid = (int64_t)blockIdx.x * groups + threadIdx.x / LPR;; gid += gstride) {
#else
    {
    const int64_t gid = (int64_t)blockIdx.x * groups + threadIdx.x / LPR;
#endif
    int64_t beg, end, row = -1;
    if (mode == 0) {
        if (a.row_order) {
            if (gid >= a.order_len) return;
            row = (int64_t)__ldg(a.row_order + gid) - a.order_offset;
            if (row < 0 || row >= a.n_rows) { PYG_SEG_SKIP; }  // a slice visits only its own rows
        } else {
            if (gid >= a.n_rows) return;
            row = gid;
        }
        beg = __ldg(a.rowptr + row);
        end = __ldg(a.rowptr + row + 1);
        if (end - beg > a.heavy_threshold) { PYG_SEG_SKIP; }  // handled by the split path
    } else {
        if (gid >= h.n_items) return;
        const int64_t item = h.item_lo + gid;
        // heavy row owning this item: last hr with item_ptr[hr] <= item
        int64_t lo = h.h_lo, hi = h.h_hi - 1;
        while (lo < hi) {
            const int64_t mid = (lo + hi + 1) >> 1;
            if (__ldg(h.item_ptr + mid) <= item) lo = mid; else hi = mid - 1;
        }
        const int64_t r = (int64_t)__ldg(h.heavy_rows + lo) - h.row_offset;
        const int64_t c = item - __ldg(h.item_ptr + lo);
        const int64_t rb = __ldg(a.rowptr + r), re = __ldg(a.rowptr + r + 1);
        beg = rb + c * h.chunk;
        end = min(beg + h.chunk, re);
    }

    constexpr bool IS_MAX = RED == PYG_MAX || RED == kRedMaxW;
    float acc[NCH][V];
    int bi[NCH][V];
    accumulate<V, NCH, RED, LPR>(a, beg, end, l, c0, acc, bi);

    if (mode == 0) {
        row_epilogue<V, NCH, RED, LPR>(a, row, end - beg, l, c0, acc, bi, out_vec_ok);
    } else {
        float* pp = h.part + gid * h.ldp;
        int32_t* pa = h.part_arg ? h.part_arg + gid * h.ldp : nullptr;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int col = c0 + l * V + ch * LPR * V;
            if (col >= a.ncols) continue;
            const int nv = min(V, a.ncols - col);
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (q < nv) {
                    pp[col + q] = acc[ch][q];
                    if (IS_MAX) pa[col + q] = bi[ch][q];
                }
        }
    }
    if (!PYG_SEG_PERSIST) return;
    }
}

template <int V, int NCH, int RED, int LPR>
inline pyg_status_t launch_one(const SegArgs& a, int tiles, int mode, const HeavyArgs& h, int ovk,
                               cudaStream_t s) {
    constexpr int groups = 256 / LPR;
    const int64_t units = mode == 0 ? (a.row_order ? a.order_len : a.n_rows) : h.n_items;
    if (units <= 0) return PYG_OK;
    int64_t blocks = cdiv(units, groups);
    if (PYG_SEG_PERSIST) blocks = std::min<int64_t>(blocks, 148LL * MinBlocks<V, NCH, RED>::value * PYG_SEG_PERSIST);
    dim3 grid((unsigned)blocks, (unsigned)tiles);
    seg_kernel<V, NCH, RED, LPR><<<grid, 256, 0, s>>>(a, mode, h, ovk);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

template <int V, int RED>
inline pyg_status_t launch_red(const SegArgs& a, int nch, int lpr, int tiles, int mode, const HeavyArgs& h,
                               int ovk, cudaStream_t s) {
    if (nch == 1) {
        switch (lpr) {
            case 4: return launch_one<V, 1, RED, 4>(a, tiles, mode, h, ovk, s);
            case 8: return launch_one<V, 1, RED, 8>(a, tiles, mode, h, ovk, s);
            case 16: return launch_one<V, 1, RED, 16>(a, tiles, mode, h, ovk, s);
            default: return launch_one<V, 1, RED, 32>(a, tiles, mode, h, ovk, s);
        }
    }
    switch (nch) {
        case 2: return launch_one<V, 2, RED, 32>(a, tiles, mode, h, ovk, s);
        case 3: return launch_one<V, 3, RED, 32>(a, tiles, mode, h, ovk, s);
        case 4: return launch_one<V, 4, RED, 32>(a, tiles, mode, h, ovk, s);
        case 5: return launch_one<V, 5, RED, 32>(a, tiles, mode, h, ovk, s);
        case 6: return launch_one<V, 6, RED, 32>(a, tiles, mode, h, ovk, s);
        case 8: return launch_one<V, 8, RED, 32>(a, tiles, mode, h, ovk, s);
        case 12: return launch_one<V, 12, RED, 32>(a, tiles, mode, h, ovk, s);
        case 16: return launch_one<V, 16, RED, 32>(a, tiles, mode, h, ovk, s);
        default: return fail(PYG_ERR_INVALID_ARGUMENT, "internal: bad NCH %d", nch);
    }
}

// explicit per-V entry points (one translation unit per V for parallel builds)
template <int V>
pyg_status_t launch(const SegArgs& a, int reduce, int nch, int lpr, int tiles, int mode, const HeavyArgs& h,
                    int ovk, cudaStream_t s) {
    switch (reduce) {
        case PYG_SUM: return launch_red<V, PYG_SUM>(a, nch, lpr, tiles, mode, h, ovk, s);
        case PYG_MEAN: return launch_red<V, PYG_MEAN>(a, nch, lpr, tiles, mode, h, ovk, s);
        case kRedHeadW: return launch_red<V, kRedHeadW>(a, nch, lpr, tiles, mode, h, ovk, s);
        case kRedSumEpi: return launch_red<V, kRedSumEpi>(a, nch, lpr, tiles, mode, h, ovk, s);
        case kRedMaxW: return launch_red<V, kRedMaxW>(a, nch, lpr, tiles, mode, h, ovk, s);
        default: return launch_red<V, PYG_MAX>(a, nch, lpr, tiles, mode, h, ovk, s);
    }
}

}  // namespace seg
}  // namespace pyg
