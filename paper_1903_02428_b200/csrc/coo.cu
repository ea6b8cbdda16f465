// coo.cu -- atomic COO scatter: the strategy of P:270-271 ("parallelization over
// *all* elements and making use of atomic operations") rebuilt for sm_100a.
//
//   * a group of `lpr` lanes walks a contiguous run of `epg` edges in input order,
//     fusing the gather of x_j and phi;
//   * warp-aggregated atomics: each batch of lpr edges is matched on its targets
//     (__match_any_sync) and visited in grouped order, so edges with equal targets --
//     consecutive (target-sorted, "coalesced" input) or not (unsorted input) --
//     are summed in registers and flushed with ONE vector red.global.add.v{2,4}.f32
//     (REDG.E.ADD.F32x4) per distinct target; for unsorted input with distinct
//     targets this is one RED per element, the paper's scheme ("GS is always
//     fast, nevertheless of the input being coalesced");
//   * hub rows (in-degree > kHeavyThreshold) would otherwise be one fp32 atomic chain
//     of up to ~306k terms (R-MAT), which breaks the tolerance (reading Q12).  Their
//     edges are routed to slots of at most kCooSlot = 2048 entries each (a per-hub counter,
//     warp-aggregated, hands out positions; slot = position / kCooSlot), the slot
//     partials live in an L2-sized workspace, and hub_combine_kernel sums them in
//     fp64 -- every fp32 chain stays <= 2048 terms on the atomic strategy too (the same bound as the
//     plan path); a 1-bit-per-row hub bitmap (1.25 MB for 10M rows, L2-resident) keeps the
//     per-edge hub test off DRAM;
//   * MAX uses 64-bit atomicMax on a packed key (order-preserving value bits in
//     the high word, 0xffffffff - edge id in the low word), so the result is
//     deterministic and ties go to the lowest edge id (Q4) without a second pass
//     over the edges; the keys live in the caller's arg_out buffer and are
//     decoded in place.  A key is only sent to the L2 atomic unit when it beats the
//     key currently stored (keys only grow, so a stale read is never too high):
//     after the first few edges of a segment almost every element is a plain read,
//     which saves the dirty-line write-back of the atomic.
#include <type_traits>

#include "kernels.cuh"

namespace pyg {

namespace {

constexpr int kBatches = 8;   // batches of lpr edges per group (epg = kBatches * lpr)
constexpr int kCooSlot = 2048;  // entries per hub slot (fp32 chain bound of the atomic path, = Q12's 2048)

template <int NCH>
struct Unroll { static constexpr int U = NCH <= 2 ? 4 : (NCH <= 5 ? 2 : 1); };

__device__ __forceinline__ unsigned group_mask(int lpr) {
    if (lpr >= 32) return 0xffffffffu;
    int lane = threadIdx.x & 31;
    return ((1u << lpr) - 1u) << (lane & ~(lpr - 1));
}

template <int V, int NCH, int RED>
__device__ __forceinline__ void flush(const CooArgs& a, int64_t cur, int l, int lpr, int c0,
                                      const bool (&cv)[NCH], float (&acc)[NCH][V],
                                      int (&bi)[NCH][V], int out_vec_ok) {
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        if (!cv[ch]) continue;
        const int col = c0 + (l + ch * lpr) * V;
        const int nv = min(V, a.ncols - col);
        if (RED == PYG_MAX) {
            unsigned long long* kp = a.keys + cur * a.ldk + col;
            unsigned long long have[V];
            if (V >= 2 && nv == V && (reinterpret_cast<uintptr_t>(kp) & 15) == 0) {
#pragma unroll
                for (int q = 0; q < V; q += 2) {
                    const ulonglong2 t = __ldcg(reinterpret_cast<const ulonglong2*>(kp + q));
                    have[q] = t.x;
                    if (q + 1 < V) have[q + 1] = t.y;
                }
            } else {
#pragma unroll
                for (int q = 0; q < V; ++q) have[q] = q < nv ? __ldcg(kp + q) : ~0ull;
            }
#pragma unroll
            for (int q = 0; q < V; ++q) {
                if (q < nv && bi[ch][q] >= 0) {
                    const unsigned long long k = max_key(acc[ch][q], (uint32_t)bi[ch][q]);
                    if (k > have[q]) atomicMax(kp + q, k);
                }
            }
        } else {
            float* op = cur < a.n_out ? a.out + cur * a.ldo + col : a.part + (cur - a.n_out) * a.ldp + col;
            if (out_vec_ok) redv<V>(op, acc[ch], nv);
            else {
#pragma unroll
                for (int q = 0; q < V; ++q) if (q < nv) atomicAdd(op + q, acc[ch][q]);
            }
        }
    }
}

template <int V, int NCH, int RED>
__global__ void __launch_bounds__(256) coo_kernel(CooArgs a, int lpr, int epg, int out_vec_ok) {
    constexpr int U = Unroll<NCH>::U;
    const int groups = blockDim.x / lpr;
    const int64_t gid = (int64_t)blockIdx.x * groups + threadIdx.x / lpr;
    const int l = threadIdx.x & (lpr - 1);
    const int gbase = (threadIdx.x & 31) & ~(lpr - 1);  // first lane of the group in its warp
    const int c0 = blockIdx.y * (lpr * NCH * V);
    const unsigned mask = group_mask(lpr);
    const int64_t e0 = gid * epg;
    if (e0 >= a.E) return;
    const int64_t e1 = min(a.E, e0 + epg);
    const bool scaled = (a.w != nullptr) || (a.gdeg != nullptr);

    bool cv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) cv[ch] = (c0 + (l + ch * lpr) * V) < a.ncols;
    float acc[NCH][V];
    int bi[NCH][V];
    auto reset = [&]() {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) { acc[ch][q] = RED == PYG_MAX ? -INFINITY : 0.0f; bi[ch][q] = -1; }
    };
    reset();
    int64_t cur = -1;

    auto consume = [&](int64_t i, int e, float sc, const float (&v)[NCH][V]) {
        if (i != cur) {
            if (cur >= 0) flush<V, NCH, RED>(a, cur, l, lpr, c0, cv, acc, bi, out_vec_ok);
            cur = i;
            reset();
        }
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < V; ++q) {
                if (RED == PYG_MAX) {
                    const float m = scaled ? __fmul_rn(sc, v[ch][q]) : v[ch][q];
                    if (bi[ch][q] < 0 || m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = e; }
                } else {
                    acc[ch][q] = scaled ? fmaf(sc, v[ch][q], acc[ch][q]) : acc[ch][q] + v[ch][q];
                }
            }
    };

    // hub rows: each hub edge's entry position comes from the hub's counter (warp-aggregated: one atomic
    // per hub and batch) and its target becomes the slot's virtual row n_out + slot.  The counters of
    // ALL the group's batches are fetched up front, so their L2 round trips overlap instead of stalling
    // every batch; the resulting targets wait in shared memory.
    __shared__ long long s_tgt[kBatches][256];
    if (RED != PYG_MAX && a.hub_base) {
        int hb[kBatches], got[kBatches];
        unsigned hm[kBatches];
#pragma unroll
        for (int j = 0; j < kBatches; ++j) {
            const int64_t p = e0 + (int64_t)j * lpr + l;
            long long t = -1 - (long long)l;
            hb[j] = -1;
            if (p < e1) {
                t = __ldcs(a.sidx + p);
                if ((__ldg(a.hub_bits + (t >> 5)) >> (t & 31)) & 1u) hb[j] = __ldg(a.hub_base + t);
            }
            s_tgt[j][threadIdx.x] = t;
            hm[j] = 0u;
            got[j] = 0;
            if (__any_sync(mask, hb[j] >= 0)) {
                hm[j] = __match_any_sync(mask, hb[j] >= 0 ? t : -1 - (long long)l);
                if (hb[j] >= 0 && (int)(threadIdx.x & 31) == __ffs(hm[j]) - 1)
                    got[j] = atomicAdd(a.hub_cursor + (int64_t)hb[j] * gridDim.y + blockIdx.y, __popc(hm[j]));
            }
        }
#pragma unroll
        for (int j = 0; j < kBatches; ++j) {
            if (hm[j] == 0u) continue;  // group-uniform: no hub in this batch
            const int lead = __ffs(hm[j]) - 1;  // absolute lane of the member group's first lane
            const int b = __shfl_sync(mask, got[j], lead - gbase, lpr);
            const int rank = __popc(hm[j] & ((1u << (threadIdx.x & 31)) - 1u));
            if (hb[j] >= 0) s_tgt[j][threadIdx.x] = a.n_out + hb[j] + (b + rank) / kCooSlot;
        }
    }

    for (int64_t base = e0; base < e1; base += lpr) {
        const int n = (int)min((int64_t)lpr, e1 - base);
        long long mi = -1 - (long long)l, mg = 0;  // unique keys for lanes without an edge
        float ms = 1.0f;
        if (l < n) {
            const int64_t p = base + l;
            mi = (RED != PYG_MAX && a.hub_base) ? s_tgt[(base - e0) / lpr][threadIdx.x] : __ldcs(a.sidx + p);
            mg = a.gidx ? __ldcs(a.gidx + p) : p;
            if (a.w) ms = __ldcs(a.w + p);
            if (a.gdeg) ms = ms / (float)__ldg(a.gdeg + mg);
        }
        // warp-aggregated atomics: visit the batch grouped by target (first-occurrence order)
        const unsigned gm = __match_any_sync(mask, mi) >> gbase;  // group-relative member mask
        const int lo = __ffs(gm) - 1;
        const bool contiguous = (((gm >> lo) & ((gm >> lo) + 1u)) == 0u);
        const bool permute = !__all_sync(mask, contiguous);
        int pos = l;
        if (permute) {
            int v = (lo == l) ? __popc(gm) : 0;
            for (int d = 1; d < lpr; d <<= 1) {
                const int t = __shfl_up_sync(mask, v, d, lpr);
                if (l >= d) v += t;
            }
            const int incl = __shfl_sync(mask, v, lo, lpr);
            pos = incl - __popc(gm) + __popc(gm & ((1u << l) - 1u));
        }
        auto src_of = [&](int t) -> int {
            return permute ? (__ffs(__ballot_sync(mask, pos == t)) - 1 - gbase) : t;
        };
        int t = 0;
        for (; t + U <= n; t += U) {
            float v[U][NCH][V];
            float sv[U];
            long long iv[U];
            int ev[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int sl = src_of(t + u);
                const long long g = __shfl_sync(mask, mg, sl, lpr);
                sv[u] = __shfl_sync(mask, ms, sl, lpr);
                iv[u] = __shfl_sync(mask, mi, sl, lpr);
                ev[u] = (int)(base + sl);
                const float* row = a.X + g * a.ldx + c0;
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
            for (int u = 0; u < U; ++u) consume(iv[u], ev[u], sv[u], v[u]);
        }
        for (; t < n; ++t) {
            const int sl = src_of(t);
            const long long g = __shfl_sync(mask, mg, sl, lpr);
            const float sc = __shfl_sync(mask, ms, sl, lpr);
            const long long i = __shfl_sync(mask, mi, sl, lpr);
            float v[NCH][V];
            const float* row = a.X + g * a.ldx + c0;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                if (cv[ch]) ldv<V>(v[ch], row + (l + ch * lpr) * V);
                else {
#pragma unroll
                    for (int q = 0; q < V; ++q) v[ch][q] = 0.0f;
                }
            }
            consume(i, (int)(base + sl), sc, v);
        }
    }
    if (cur >= 0) flush<V, NCH, RED>(a, cur, l, lpr, c0, cv, acc, bi, out_vec_ok);
}

// ---------------------------------------------------------------- warp-batched tile kernel
// coo_tile_kernel<LPR, RED>: the atomic strategy for float4-capable rows whose column tile is
// W = 4 * LPR floats (LPR in {4, 8, 16}; one tile = the whole row for F <= 64, else the L2 column
// tiles of l2_tile_cols).  Rows of 65-128 floats that are not L2-tiled (R-MAT: out 5 GB, DRAM read-
// modify-write bound) stay on coo_kernel, whose up-front hub-counter prefetch measured faster there
// (R-MAT sum 34.4 vs 36.0 ms, max 63.5 vs 70.5 ms, gpurun_out/r3e).  A WARP takes 32 edges at a time (one coalesced, streaming load of
// source, target and weight per lane) and its 32 / LPR lane groups split them:
//   * warp-aggregated atomics with ONE full-warp __match_any_sync per 32 edges: if any target repeats
//     (sorted input, hubs, small graphs), the batch is visited in grouped order (leaders in lane order,
//     members after their leader, positions from a shuffle scan, inverted through shared memory), so a
//     group sums the run of equal targets it holds in registers and sends one red.global.add.v4.f32 per
//     run; for distinct targets (the common case on large uniform graphs) the identity order costs
//     nothing;
//   * U = 8 rows in flight per lane before any is consumed (the generic coo_kernel spends ~26 warp
//     instructions per edge on per-group matching, 64-bit index arithmetic and runtime lane counts;
//     ncu on the L2-tiled Reddit pass: 50% issue-busy at 2.0 IPC, MATCH/WARPSYNC the top stalls,
//     gpurun_out/r3d);
//   * hub rows (SUM / MEAN) take slot positions from their per-(slot, tile) counter exactly as in
//     coo_kernel (one atomic per hub and batch) and become the virtual rows n_out + slot;
//   * MAX: packed 64-bit keys, a group's run keeps the lowest edge id (grouped order is ascending edge
//     id within a target), atomicMax only when the stored key is smaller.
template <int LPR, int RED>
__global__ void __launch_bounds__(256, 3) coo_tile_kernel(CooArgs a, int64_t chunk, int out_vec_ok) {
    constexpr int PER = LPR;     // grouped positions per group per batch (G * PER = 32)
    constexpr int U = PER < 8 ? PER : 8;
    const unsigned full = 0xffffffffu;
    const int lane = threadIdx.x & 31, grp = lane / LPR, l = lane % LPR;
    const int wib = threadIdx.x >> 5;
    __shared__ int s_inv[8][32];
    const int col = blockIdx.y * (4 * LPR) + 4 * l;
    const int nv = max(0, min(4, a.ncols - col));
    const bool full_ld = nv == 4 || (nv > 0 && a.allow_pad_read);
    const int64_t e0 = ((int64_t)blockIdx.x * 8 + wib) * chunk;
    if (e0 >= a.E) return;
    const int64_t e1 = min(a.E, e0 + chunk);
    const bool scaled = (a.w != nullptr) || (a.gdeg != nullptr);
    const unsigned lt = (1u << lane) - 1u;
    // no hub row at all (the common case; the count is on the device, written by hub_assign_kernel):
    // skip the per-edge bitmap test
    const bool hubs = RED != PYG_MAX && a.hub_base && __ldg(a.hub_count) > 0;
    // 32-bit row offsets (one IMAD.WIDE.U32 per address) when every byte offset fits
    const float* __restrict__ Xc = a.X + col;
    const uint32_t xrb = (uint32_t)(a.ldx * 4), orb = (uint32_t)(a.ldo * 4);
    const bool off32 = (uint64_t)a.ldx * 4 * (uint64_t)(a.n_src > 0 ? a.n_src : a.E) < (1ull << 32) &&
                       (RED == PYG_MAX || (uint64_t)a.ldo * 4 * (uint64_t)a.n_out < (1ull << 32));
    char* __restrict__ Oc = reinterpret_cast<char*>(a.out + col);
    const bool keys16 = RED == PYG_MAX && (a.ldk % 2 == 0) && !(reinterpret_cast<uintptr_t>(a.keys) & 15);
    const bool red4_ok = out_vec_ok && nv == 4;

    // the next batch's (target, source, weight) are loaded while this batch is processed: the index
    // stream comes from DRAM, and its latency would otherwise open every batch
    long long nt = 0, ng = 0;
    float nw = 1.0f;
    auto fetch = [&](int64_t b) {
        const int64_t q = b + lane;
        if (q < e1) {
            nt = __ldcs(a.sidx + q);
            ng = a.gidx ? __ldcs(a.gidx + q) : q;
            if (a.w) nw = __ldcs(a.w + q);
        }
    };
    fetch(e0);
    for (int64_t base = e0; base < e1; base += 32) {
        const int n = (int)min((int64_t)32, e1 - base);
        const bool valid = lane < n;
        int t = valid ? (int)nt : -1 - lane;
        int g = valid ? (int)ng : 0;
        float s = a.w ? nw : 1.0f;
        if (base + 32 < e1) fetch(base + 32);
        if (valid && a.gdeg) s = s / (float)__ldg(a.gdeg + g);
        bool hub_batch = false;
        if (hubs) {
            int hb = -1;
            if (valid && ((__ldg(a.hub_bits + (t >> 5)) >> (t & 31)) & 1u)) hb = __ldg(a.hub_base + t);
            if (__any_sync(full, hb >= 0)) {
                const unsigned hm = __match_any_sync(full, hb >= 0 ? t : -1 - lane);
                const int lead = __ffs(hm) - 1;
                int got = 0;
                if (hb >= 0 && lane == lead)
                    got = atomicAdd(a.hub_cursor + (int64_t)hb * (a.n_tiles ? a.n_tiles : (int)gridDim.y) +
                                        (a.n_tiles ? a.tile_y : (int)blockIdx.y), __popc(hm));
                got = __shfl_sync(full, got, lead);
                if (hb >= 0) t = (int)a.n_out + hb + (got + __popc(hm & lt)) / kCooSlot;
                hub_batch = true;
            }
        }
        const unsigned m = __match_any_sync(full, t);
        const bool dup = __any_sync(full, m != (1u << lane));
        if (RED == PYG_MAX && n == 32 && !dup && off32) {
            // 32 distinct targets: every edge is its own run; the stored keys of 4 edges are loaded
            // together (one dependent L2 round trip per 4 edges instead of per edge), and a key is only
            // sent to the atomic unit when it beats the stored one
#pragma unroll
            for (int k0 = 0; k0 < PER; k0 += 4) {
                float v[4][4];
                unsigned long long kh[4][4];
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int gg = __shfl_sync(full, g, grp * PER + k0 + u);
                    const float* row = reinterpret_cast<const float*>(reinterpret_cast<const char*>(Xc) +
                                                                     (uint64_t)(uint32_t)gg * xrb);
                    if (full_ld) {
                        const float4 x = __ldg(reinterpret_cast<const float4*>(row));
                        v[u][0] = x.x; v[u][1] = x.y; v[u][2] = x.z; v[u][3] = x.w;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) v[u][c] = c < nv ? __ldg(row + c) : 0.0f;
                    }
                    const int tu = __shfl_sync(full, t, grp * PER + k0 + u);
                    const unsigned long long* kp = a.keys + (int64_t)tu * a.ldk + col;
                    if (nv == 4 && keys16) {
                        const ulonglong2 x0 = __ldcg(reinterpret_cast<const ulonglong2*>(kp));
                        const ulonglong2 x1 = __ldcg(reinterpret_cast<const ulonglong2*>(kp + 2));
                        kh[u][0] = x0.x; kh[u][1] = x0.y; kh[u][2] = x1.x; kh[u][3] = x1.y;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) kh[u][c] = c < nv ? __ldcg(kp + c) : ~0ull;
                    }
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const int sl = grp * PER + k0 + u;
                    const int tu = __shfl_sync(full, t, sl);
                    const float su = scaled ? __shfl_sync(full, s, sl) : 1.0f;
                    unsigned long long* kp = a.keys + (int64_t)tu * a.ldk + col;
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        const float mv = scaled ? __fmul_rn(su, v[u][c]) : v[u][c];
                        const unsigned long long k = max_key(mv, (uint32_t)(base + sl));
                        if (c < nv && k > kh[u][c]) atomicMax(kp + c, k);
                    }
                }
            }
            continue;
        }
        if (RED != PYG_MAX && LPR < 32 && n == 32 && dup && off32 && __all_sync(full, m == full)) {
            // 32 edges into ONE target (target-sorted input, high in-degree: Fig. 3's coalesced case):
            // each group sums its positions, a butterfly over the groups adds them up, one RED
            float acc[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
            for (int k0 = 0; k0 < PER; k0 += U) {
                float v[U][4];
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const int gg = __shfl_sync(full, g, grp * PER + k0 + u);
                    const float* row = reinterpret_cast<const float*>(reinterpret_cast<const char*>(Xc) +
                                                                     (uint64_t)(uint32_t)gg * xrb);
                    if (full_ld) {
                        const float4 x = __ldg(reinterpret_cast<const float4*>(row));
                        v[u][0] = x.x; v[u][1] = x.y; v[u][2] = x.z; v[u][3] = x.w;
                    } else {
#pragma unroll
                        for (int c = 0; c < 4; ++c) v[u][c] = c < nv ? __ldg(row + c) : 0.0f;
                    }
                }
#pragma unroll
                for (int u = 0; u < U; ++u) {
                    const float su = scaled ? __shfl_sync(full, s, grp * PER + k0 + u) : 1.0f;
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[c] = scaled ? fmaf(su, v[u][c], acc[c]) : acc[c] + v[u][c];
                }
            }
#pragma unroll
            for (int off = 16; off >= LPR; off >>= 1)
#pragma unroll
                for (int c = 0; c < 4; ++c) acc[c] += __shfl_xor_sync(full, acc[c], off);
            const int t0 = t;  // every lane holds the batch's one target
            if (grp == 0) {
                float* op = t0 < a.n_out ? reinterpret_cast<float*>(Oc + (uint64_t)(uint32_t)t0 * orb)
                                         : a.part + (int64_t)(t0 - a.n_out) * a.ldp + col;
                if (red4_ok) redv<4>(op, acc, 4);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) if (c < nv) atomicAdd(op + c, acc[c]);
                }
            }
            __syncwarp();  // s_inv was written for this batch
            continue;
        }
        if (RED != PYG_MAX && n == 32 && !dup && !hub_batch && off32) {
            // 32 distinct real targets (uniform graphs: almost every batch): every edge is its own run,
            // so no run tracking -- per edge and lane one shuffle, one row load, one RED
#pragma unroll
            for (int k0 = 0; k0 < PER; k0 += U) {
            float v[U][4];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int gg = __shfl_sync(full, g, grp * PER + k0 + u);
                const float* row = reinterpret_cast<const float*>(reinterpret_cast<const char*>(Xc) +
                                                                 (uint64_t)(uint32_t)gg * xrb);
                if (full_ld) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(row));
                    v[u][0] = x.x; v[u][1] = x.y; v[u][2] = x.z; v[u][3] = x.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[u][c] = c < nv ? __ldg(row + c) : 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int tu = __shfl_sync(full, t, grp * PER + k0 + u);
                if (scaled) {
                    const float su = __shfl_sync(full, s, grp * PER + k0 + u);
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[u][c] *= su;
                }
                float* op = reinterpret_cast<float*>(Oc + (uint64_t)(uint32_t)tu * orb);
                if (red4_ok) redv<4>(op, v[u], 4);
                else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) if (c < nv) atomicAdd(op + c, v[u][c]);
                }
            }
            }
            continue;
        }
        if (dup) {
            const int lead = __ffs(m) - 1;
            int v = lane == lead ? __popc(m) : 0;
#pragma unroll
            for (int d = 1; d < 32; d <<= 1) {
                const int y = __shfl_up_sync(full, v, d);
                if (lane >= d) v += y;
            }
            const int incl = __shfl_sync(full, v, lead);
            s_inv[wib][incl - __popc(m) + __popc(m & lt)] = lane;
            __syncwarp();
        }
        float acc[4];
        int bi[4];
        int cur = 0;
        bool have = false;
        auto flush = [&]() {
            if (!have || nv == 0) return;
            if (RED == PYG_MAX) {
                unsigned long long* kp = a.keys + (int64_t)cur * a.ldk + col;
                unsigned long long hv[4];
                if (nv == 4 && (reinterpret_cast<uintptr_t>(kp) & 15) == 0) {
                    const ulonglong2 x0 = __ldcg(reinterpret_cast<const ulonglong2*>(kp));
                    const ulonglong2 x1 = __ldcg(reinterpret_cast<const ulonglong2*>(kp + 2));
                    hv[0] = x0.x; hv[1] = x0.y; hv[2] = x1.x; hv[3] = x1.y;
                } else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) hv[q] = q < nv ? __ldcg(kp + q) : ~0ull;
                }
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (q < nv) {
                        const unsigned long long k = max_key(acc[q], (uint32_t)bi[q]);
                        if (k > hv[q]) atomicMax(kp + q, k);
                    }
                }
            } else {
                float* op = cur < a.n_out ? a.out + (int64_t)cur * a.ldo + col
                                          : a.part + (int64_t)(cur - a.n_out) * a.ldp + col;
                if (out_vec_ok) redv<4>(op, acc, nv);
                else {
#pragma unroll
                    for (int q = 0; q < 4; ++q) if (q < nv) atomicAdd(op + q, acc[q]);
                }
            }
        };
#pragma unroll
        for (int k0 = 0; k0 < PER; k0 += U) {
            // only the rows and their source lanes live across the loads (target and scale are
            // re-shuffled when consumed): 8 rows in flight per lane without spilling at 4 CTAs / SM
            float v[U][4];
            int slv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = grp * PER + k0 + u;
                const int sl = dup ? s_inv[wib][q] : q;
                slv[u] = sl;
                const int gg = __shfl_sync(full, g, sl);
                const float* row = a.X + (int64_t)gg * a.ldx + col;
                if (q < n && full_ld) {
                    const float4 x = __ldg(reinterpret_cast<const float4*>(row));
                    v[u][0] = x.x; v[u][1] = x.y; v[u][2] = x.z; v[u][3] = x.w;
                } else {
#pragma unroll
                    for (int c = 0; c < 4; ++c) v[u][c] = (q < n && c < nv) ? __ldg(row + c) : 0.0f;
                }
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int q = grp * PER + k0 + u;
                const int tu = __shfl_sync(full, t, slv[u]);
                const float su = scaled ? __shfl_sync(full, s, slv[u]) : 1.0f;
                if (q >= n) continue;  // (shuffles above stay warp-uniform)
                if (!have || tu != cur) {
                    flush();
                    cur = tu;
                    have = true;
#pragma unroll
                    for (int c = 0; c < 4; ++c) { acc[c] = RED == PYG_MAX ? -INFINITY : 0.0f; bi[c] = -1; }
                }
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    if (RED == PYG_MAX) {
                        const float mv = scaled ? __fmul_rn(su, v[u][c]) : v[u][c];
                        if (bi[c] < 0 || mv > acc[c]) { acc[c] = mv; bi[c] = (int)base + slv[u]; }
                    } else {
                        acc[c] = scaled ? fmaf(su, v[u][c], acc[c]) : acc[c] + v[u][c];
                    }
                }
            }
        }
        flush();
        if (dup) __syncwarp();  // s_inv is rewritten by the next batch
    }
}

template <int V, int RED>
pyg_status_t launch_v(const CooArgs& a, int nch, int lpr, int tiles, int epg, int ovk, cudaStream_t s) {
    const int threads = 256;
    const int groups = threads / lpr;
    const int64_t units = cdiv(a.E, epg);
    if (units <= 0) return PYG_OK;
    dim3 grid((unsigned)cdiv(units, groups), (unsigned)tiles);
#define PYG_COO_CASE(N) \
    case N: coo_kernel<V, N, RED><<<grid, threads, 0, s>>>(a, lpr, epg, ovk); break;
    switch (nch) {
        PYG_COO_CASE(1) PYG_COO_CASE(2) PYG_COO_CASE(3) PYG_COO_CASE(4) PYG_COO_CASE(5)
        PYG_COO_CASE(6) PYG_COO_CASE(8) PYG_COO_CASE(10) PYG_COO_CASE(12) PYG_COO_CASE(16)
        default: return fail(PYG_ERR_INVALID_ARGUMENT, "internal: bad NCH %d", nch);
    }
#undef PYG_COO_CASE
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

template <int RED>
pyg_status_t launch_red(const CooArgs& a, int V, int nch, int lpr, int tiles, int epg, int ovk,
                        cudaStream_t s) {
    if (V == 4) return launch_v<4, RED>(a, nch, lpr, tiles, epg, ovk, s);
    if (V == 2) return launch_v<2, RED>(a, nch, lpr, tiles, epg, ovk, s);
    return launch_v<1, RED>(a, nch, lpr, tiles, epg, ovk, s);
}

bool aligned(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

constexpr int kNch[] = {1, 2, 3, 4, 5, 6, 8, 10, 12, 16};

__global__ void degree_kernel(const int64_t* __restrict__ sidx, int64_t E, int32_t* deg, int32_t* first,
                              float* zero_out = nullptr, int64_t ldo = 0, int ncols = 0, int64_t n_rows = 0) {
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = t0; k < E; k += nt) {
        const int64_t i = sidx[k];
        if (deg) atomicAdd(deg + i, 1);
        if (first) atomicMin(first + i, (int32_t)k);
    }
    if (zero_out) {
        const int64_t total = n_rows * ncols;
        for (int64_t t = t0; t < total; t += nt) {
            const int64_t r = t / ncols;
            zero_out[r * ldo + (t - r * ncols)] = 0.0f;
        }
    }
}

// Compact column tiles: the tile kernel's gathers and REDs on a W-float slice of row-major X / out
// touch 128 bytes every ldx * 4 bytes, i.e. the slice's bytes spread over ldx / W times the address range
// -- beyond the TLB reach (scripts/l2red.cu: gather + RED into 32-float slices of 608-float rows 2.74 TB/s
// against 5.67 TB/s into a compact 30 MB table).  So each tile packs X's columns [c0, c0 + w) into a
// compact [n_src x W] scratch, accumulates into a compact [n_out x W] one and unpacks it into out
// (with the mean divide fused).
__global__ void pack_cols_kernel(const float* __restrict__ X, int64_t ldx, int64_t rows, int c0, int w, int W,
                                 int vec, float* __restrict__ Xs) {
    const int nq = W / 4;
    const int64_t total = rows * nq;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / nq;
        const int c = 4 * (int)(t - r * nq);
        const float* src = X + r * ldx + c0 + c;
        float4 v;
        if (vec && c + 4 <= w) {
            v = __ldg(reinterpret_cast<const float4*>(src));
        } else {
            v.x = c < w ? __ldg(src) : 0.0f;
            v.y = c + 1 < w ? __ldg(src + 1) : 0.0f;
            v.z = c + 2 < w ? __ldg(src + 2) : 0.0f;
            v.w = c + 3 < w ? __ldg(src + 3) : 0.0f;
        }
        reinterpret_cast<float4*>(Xs + r * W)[c / 4] = v;
    }
}

template <typename T>
__global__ void unpack_cols_kernel(const T* __restrict__ Os, int W, int64_t rows, T* __restrict__ out, int64_t ldo,
                                   int c0, int w, const int32_t* __restrict__ deg) {
    const int64_t total = rows * w;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = t / w;
        const int c = (int)(t - r * w);
        T v = Os[r * W + c];
        if constexpr (std::is_same<T, float>::value) {
            if (deg) {
                const int d = __ldg(deg + r);
                v = d > 0 ? v / (float)d : 0.0f;
            }
        }
        out[r * ldo + c0 + c] = v;
    }
}

// hub rows: deg > threshold -> ceil(deg / kCooSlot) consecutive slots, their counters zeroed
// (one per column tile); counters[0] = hubs, counters[1] = slots handed out
__global__ void hub_assign_kernel(const int32_t* __restrict__ deg, int64_t n, int threshold, int tiles,
                                  int32_t* hub_base, uint32_t* hub_bits, int32_t* hub_rows, int32_t* counters,
                                  int32_t* cursor, float* part, int64_t ldp) {
    // whole warps walk 32 consecutive rows so each bitmap word is one ballot
    const int64_t n32 = (n + 31) & ~(int64_t)31;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n32; i += (int64_t)gridDim.x * blockDim.x) {
        const int d = i < n ? deg[i] : 0;
        const bool hub = d > threshold;
        if (hub) {
            const int ns = (d + kCooSlot - 1) / kCooSlot;
            const int hb = atomicAdd(counters + 1, ns);
            hub_rows[atomicAdd(counters, 1)] = (int32_t)i;
            for (int t = 0; t < tiles; ++t) cursor[(int64_t)hb * tiles + t] = 0;
            hub_base[i] = hb;
            // the hub zeroes its own slot partials (no separate launch: small graphs are launch-bound)
            float4* ps = reinterpret_cast<float4*>(part + (int64_t)hb * ldp);
            for (int64_t q = 0; q < (int64_t)ns * (ldp / 4); ++q) ps[q] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
        const unsigned word = __ballot_sync(0xffffffffu, hub);
        if ((threadIdx.x & 31) == 0) hub_bits[i >> 5] = word;
    }
}

// out[hub] = fp64 sum of the hub's slot partials in slot order (/ deg for mean): Q12 on the
// atomic path
template <int RED>
__global__ void hub_combine_kernel(float* out, int64_t ldo, int ncols, const float* __restrict__ part, int64_t ldp,
                                   const int32_t* __restrict__ hub_rows, const int32_t* __restrict__ hub_base,
                                   const int32_t* __restrict__ deg, const int32_t* __restrict__ counters) {
    const int nh = counters[0];
    for (int h = blockIdx.x; h < nh; h += gridDim.x) {
        const int64_t r = hub_rows[h];
        const int d = deg[r];
        const int64_t b = hub_base[r];
        const int ns = (d + kCooSlot - 1) / kCooSlot;
        for (int c = threadIdx.x; c < ncols; c += blockDim.x) {
            double s = 0.0;
            for (int k = 0; k < ns; ++k) s += (double)part[(b + k) * ldp + c];
            if (RED == PYG_MEAN) s = d > 0 ? s / (double)d : 0.0;
            out[r * ldo + c] = (float)s;
        }
    }
}

__global__ void mean_div_kernel(float* out, int64_t ldo, int ncols, int64_t n, const int32_t* __restrict__ deg) {
    const int64_t total = n * ncols;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ncols;
        const int c = (int)(t - i * ncols);
        const int32_t d = deg[i];
        float* p = out + i * ldo + c;
        *p = d > 0 ? *p / (float)d : 0.0f;
    }
}

__global__ void max_decode_kernel(unsigned long long* keys, int64_t ldk, float* out, int64_t ldo, int ncols,
                                  int64_t n, int64_t E) {
    const int64_t total = n * ncols;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = t / ncols;
        const int c = (int)(t - i * ncols);
        unsigned long long* kp = keys + i * ldk + c;
        const unsigned long long key = *kp;
        if (key == 0ull) {
            out[i * ldo + c] = 0.0f;
            *reinterpret_cast<long long*>(kp) = E;
        } else {
            out[i * ldo + c] = ord2f((uint32_t)(key >> 32));
            *reinterpret_cast<long long*>(kp) = (long long)(0xffffffffu - (uint32_t)(key & 0xffffffffu));
        }
    }
}

int grid_for(int64_t work, int threads = 256) {
    int64_t b = cdiv(work, threads);
    return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 32));
}

// hub workspace capacity: at most E / (threshold + 1) hubs, and sum ceil(d / slot) <= E / slot + hubs
int64_t hub_cap(int64_t E) { return E / (kHeavyThreshold + 1) + 1; }
int64_t slot_cap(int64_t E) { return E / kCooSlot + hub_cap(E); }

// Column-tile width that keeps one tile's accumulation target (fp32 out or 64-bit MAX keys) and its
// gathered source rows inside the L2 budget (PYG_COO_L2_MB): without it a plan-free scatter into an
// output wider than L2 (Reddit: 561 MB) misses L2 on every red.global and pays a DRAM read-modify-
// write per element.  0: no tiling (everything fits already, or even 8 columns do not).
int l2_tile_cols(const CooArgs& a, int reduce) {
    // MAX: the keys are mostly only read (an atomicMax is sent only when the stored key is smaller), so
    // wider tiles pay off up to a larger footprint (Reddit max: 32-column tiles, 89 MB, 153 ms against
    // 16-column tiles 189 ms; SUM / MEAN: 32-column tiles, 60 MB; PubMed sum untiled at 79 MB 0.40 ms
    // against 64-column tiles 0.16 ms; gpurun_out/r3f)
    const int64_t budget = (int64_t)(reduce == PYG_MAX ? knobs().coo_l2_mb_max : knobs().coo_l2_mb) << 20;
    if (budget <= 0) return 0;
    const int64_t per_col = a.n_out * (reduce == PYG_MAX ? 8 : 4) + (a.gidx ? a.n_src * 4 : 0);
    if (per_col * a.ncols <= budget) return 0;
    for (int W : {64, 32, 16, 8})
        if (per_col * W <= budget && W < a.ncols) return W;
    return 0;
}

struct CooGeom {
    int V, lpr, nch, tiles, ovk;
    int tile_lpr;  // > 0: coo_tile_kernel<tile_lpr> (float4 rows), else coo_kernel
};

CooGeom coo_geometry(const CooArgs& a, int reduce) {
    CooGeom g{1, 4, 1, 1, 0, 0};
    for (int cand : {4, 2}) {
        const bool cols_ok = (a.ncols % cand == 0) || (a.allow_pad_read && cand == 4 &&
                                                       a.ldx >= (int64_t)align_up(a.ncols, 4));
        if (cols_ok && a.ldx % cand == 0 && aligned(a.X, 4 * cand)) { g.V = cand; break; }
    }
    g.ovk = (reduce != PYG_MAX) && (a.ldo % g.V == 0) && aligned(a.out, 4 * g.V) &&
            (!a.part || (a.ldp % g.V == 0 && aligned(a.part, 4 * g.V)));
    const int64_t nvec = cdiv(a.ncols, g.V);
    const int W = l2_tile_cols(a, reduce);
    if (g.V == 4 && knobs().coo_tile && a.E < (1LL << 31) && a.n_out + slot_cap(a.E) < (1LL << 31) &&
        (W >= 16 || (W == 0 && a.ncols <= (knobs().coo_tile == 2 ? 128 : 64)))) {
        int lpr = 4;
        while (4 * lpr < (W ? W : a.ncols)) lpr <<= 1;
        g.tile_lpr = lpr;
        g.tiles = (int)cdiv(a.ncols, 4 * lpr);
        return g;
    }
    if (W > 0 && W % g.V == 0) {
        // L2 column tiles: tile y's REDs (and gathers) stay inside an L2-resident slice; grid.y is the
        // slowest-varying block index, so tiles run one after another
        const int wv = W / g.V;
        g.lpr = std::min(32, wv);
        g.nch = wv / g.lpr;
        g.tiles = (int)cdiv(a.ncols, W);
    } else if (nvec <= 32) {
        while (g.lpr < nvec) g.lpr <<= 1;
    } else {
        g.lpr = 32;
        int64_t need = cdiv(nvec, 32);
        g.tiles = (int)cdiv(need, 16);
        need = cdiv(nvec, 32 * (int64_t)g.tiles);
        g.nch = 16;
        for (int c : kNch) if (c >= need) { g.nch = c; break; }
    }
    return g;
}

// edges per warp of coo_tile_kernel (PYG_COO_CHUNK, a multiple of 32; default 4 batches of 32:
// Reddit mean 81.8 ms against 83.8 ms at 8 and 86.5 ms at 64, gpurun_out/r3f)
int64_t tile_chunk() { return std::max<int64_t>(32, (int64_t)knobs().coo_chunk / 32 * 32); }

template <int RED>
pyg_status_t launch_tile(const CooArgs& a, const CooGeom& g, cudaStream_t s) {
    const int64_t chunk = tile_chunk();
    const int64_t blocks = cdiv(a.E, 8 * chunk);
    if (blocks <= 0) return PYG_OK;
    dim3 grid((unsigned)blocks, (unsigned)g.tiles);
    switch (g.tile_lpr) {
        case 4: coo_tile_kernel<4, RED><<<grid, 256, 0, s>>>(a, chunk, g.ovk); break;
        case 8: coo_tile_kernel<8, RED><<<grid, 256, 0, s>>>(a, chunk, g.ovk); break;
        case 16: coo_tile_kernel<16, RED><<<grid, 256, 0, s>>>(a, chunk, g.ovk); break;
        case 32: coo_tile_kernel<32, RED><<<grid, 256, 0, s>>>(a, chunk, g.ovk); break;
        default: return fail(PYG_ERR_INVALID_ARGUMENT, "internal: bad tile lanes %d", g.tile_lpr);
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

int64_t max_tiles(int64_t ncols) { return std::max<int64_t>(1, cdiv(ncols, 8)); }  // L2 tiles of >= 8 columns

}  // namespace

int64_t coo_tile_cols(int64_t n_out, int64_t n_src, int64_t ncols, int reduce) {
    CooArgs a;
    a.n_out = n_out;
    a.n_src = n_src;
    a.ncols = (int)ncols;
    static const int64_t dummy = 0;
    a.gidx = n_src > 0 ? &dummy : nullptr;
    return l2_tile_cols(a, reduce);
}

constexpr double kCompactSpan = 256.0 * (1 << 20);

// compact-tile scratch: [n_out x W] accumulation target (+ [n_src x W] gathered slice), 0 if untiled
static size_t compact_bytes(int64_t n_out, int64_t n_src, int64_t ncols, int reduce) {
    const int64_t W = coo_tile_cols(n_out, n_src, ncols, reduce);
    if (W <= 0) return 0;
    return (size_t)n_out * W * (reduce == PYG_MAX ? 8 : 4) + (size_t)n_src * W * 4 + 512;
}

size_t coo_ws_bytes(int64_t E, int64_t n_out, int64_t ncols, int reduce, int64_t n_src) {
    if (E <= 0) return 0;
    if (reduce == PYG_MAX) return compact_bytes(n_out, n_src, ncols, reduce);
    Carver cv(nullptr, 0);
    cv.take<int32_t>((size_t)std::max<int64_t>(n_out, 1) + 64);  // deg, then the 4 hub counters (one memset)
    if (E > kHeavyThreshold) {
        cv.take<int32_t>((size_t)n_out);                             // hub_base (valid for hubs only)
        cv.take<uint32_t>((size_t)cdiv(n_out, 32));                  // hub bitmap
        cv.take<int32_t>((size_t)hub_cap(E));                        // hub_rows
        cv.take<int32_t>((size_t)(slot_cap(E) * max_tiles(ncols)));  // cursors
        cv.take<float>((size_t)slot_cap(E) * align_up((size_t)ncols, 4));  // slot partials
    }
    return cv.off + 256 + compact_bytes(n_out, n_src, ncols, reduce);
}

pyg_status_t coo_reduce(const CooArgs& a0, int reduce, void* ws, size_t ws_bytes, cudaStream_t s) {
    CooArgs a = a0;
    if (a.n_out <= 0 || a.ncols <= 0) return PYG_OK;
    if (a.E <= 0) {  // outputs are overwritten (Q14): zeros, and arg = E for MAX
        if (reduce == PYG_MAX) {
            PYG_CUDA(cudaMemset2DAsync(a.keys, a.ldk * 8, 0, (size_t)a.ncols * 8, (size_t)a.n_out, s));
            PYG_TRY(max_decode(a.keys, a.ldk, a.out, a.ldo, a.ncols, a.n_out, a.E, s));
        } else {
            PYG_CUDA(cudaMemset2DAsync(a.out, a.ldo * 4, 0, (size_t)a.ncols * 4, (size_t)a.n_out, s));
        }
        return PYG_OK;
    }
    int32_t* deg = nullptr;
    int32_t* counters = nullptr;
    int32_t* hub_rows = nullptr;
    int32_t* hub_base = nullptr;
    const bool hubs = reduce != PYG_MAX && a.E > kHeavyThreshold;
    Carver cv(ws, ws_bytes);
    if (reduce != PYG_MAX) {
        const size_t n_deg = (size_t)std::max<int64_t>(a.n_out, 1);
        deg = cv.take<int32_t>(n_deg + 64);
        counters = deg + align_up(n_deg, 16);  // right behind deg: one memset zeroes both
        if (hubs) {
            hub_base = cv.take<int32_t>((size_t)a.n_out);
            a.hub_base = hub_base;
            a.hub_bits = cv.take<uint32_t>((size_t)cdiv(a.n_out, 32));
            hub_rows = cv.take<int32_t>((size_t)hub_cap(a.E));
            a.hub_cursor = cv.take<int32_t>((size_t)(slot_cap(a.E) * max_tiles(a.ncols)));
            a.hub_count = counters;
            a.ldp = (int64_t)align_up((size_t)a.ncols, 4);
            a.part = cv.take<float>((size_t)slot_cap(a.E) * a.ldp);
        }
        if (!ws || !cv.ok())
            return fail(PYG_ERR_NO_MEMORY, "atomic scatter: workspace too small (%zu < %zu bytes, see pyg_workspace_size)",
                        ws_bytes, coo_ws_bytes(a.E, a.n_out, a.ncols, reduce, a.gidx ? a.n_src : 0));
    }
    const CooGeom g = coo_geometry(a, reduce);
    // compact column tiles (see pack_cols_kernel) when the tile kernel runs several L2 tiles and the
    // workspace holds the scratch; otherwise the tiles address X / out in place
    const int W = 4 * g.tile_lpr;
    const int64_t xs_rows = a.gidx ? a.n_src : 0;
    float* Os = nullptr;
    unsigned long long* Ks = nullptr;
    float* Xs = nullptr;
    // (auto: only when the strided slices span more than kCompactSpan bytes -- PubMed's 39 MB X is within
    // TLB reach and its 8 tiles x 4 launches measured 0.51 ms compact against 0.14 ms in place, Reddit's
    // 1.1 GB span 54 ms against 82 ms; gpurun_out/r3k)
    const int cmode = knobs().coo_compact;
    const double span = 4.0 * ((double)a.n_out * (double)(reduce == PYG_MAX ? 2 * a.ldk : a.ldo) +
                               (a.gidx ? (double)a.n_src * (double)a.ldx : 0.0));
    if (g.tile_lpr && g.tiles > 1 && (cmode == 2 || (cmode == 1 && span > kCompactSpan)) &&
        (!a.gidx || a.n_src > 0)) {
        Carver c2 = cv;
        if (reduce == PYG_MAX) Ks = c2.take<unsigned long long>((size_t)a.n_out * W);
        else Os = c2.take<float>((size_t)a.n_out * W);
        if (xs_rows) Xs = c2.take<float>((size_t)xs_rows * W);
        if (!ws || !c2.ok()) Os = nullptr, Ks = nullptr, Xs = nullptr;
    }
    const bool compact = Os || Ks;
    bool out_zeroed = false;
    if (reduce != PYG_MAX) {
        if (a.deg) {
            if (hubs) PYG_CUDA(cudaMemsetAsync(counters, 0, 4 * sizeof(int32_t), s));
            deg = const_cast<int32_t*>(a.deg);
        } else {
            const size_t n_deg = (size_t)std::max<int64_t>(a.n_out, 1);
            PYG_CUDA(cudaMemsetAsync(deg, 0, (align_up(n_deg, 16) + 4) * sizeof(int32_t), s));
            // the degree pass also zeroes a small in-place target (one launch fewer: tiny graphs are launch-
            // bound; Fig. 3 atomic 25-29 -> 24-27 ms per 1,000 calls); large ones keep the memset (R-MAT's
            // 5 GB: 34.3 ms with it, 35.8 ms zeroed by the degree pass, gpurun_out/r3ah)
            out_zeroed = !compact && a.n_out * a.ncols <= (int64_t)(16 << 20);
            const int64_t work = std::max<int64_t>(a.E, out_zeroed ? a.n_out * a.ncols : 0);
            degree_kernel<<<grid_for(work), 256, 0, s>>>(a.sidx, a.E, deg, nullptr, out_zeroed ? a.out : nullptr,
                                                         a.ldo, a.ncols, a.n_out);
            PYG_LAUNCHED();
            PYG_CUDA(cudaGetLastError());
        }
    }
    if (!compact && !out_zeroed) {  // zero the accumulation target (outputs are overwritten, Q14)
        if (reduce == PYG_MAX)
            PYG_CUDA(cudaMemset2DAsync(a.keys, a.ldk * 8, 0, (size_t)a.ncols * 8, (size_t)a.n_out, s));
        else
            PYG_CUDA(cudaMemset2DAsync(a.out, a.ldo * 4, 0, (size_t)a.ncols * 4, (size_t)a.n_out, s));
    }
    if (hubs) {
        hub_assign_kernel<<<grid_for(a.n_out), 256, 0, s>>>(deg, a.n_out, kHeavyThreshold, g.tiles, hub_base,
                                                              const_cast<uint32_t*>(a.hub_bits), hub_rows, counters,
                                                              a.hub_cursor, a.part, a.ldp);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    const int epg = g.lpr * kBatches;
    if (compact) {
        const int vec = (a.ldx % 4 == 0) && aligned(a.X, 16);
        CooGeom g1 = g;
        g1.tiles = 1;
        for (int y = 0; y < g.tiles; ++y) {
            const int c0 = y * W;
            const int w = std::min(W, a.ncols - c0);
            CooArgs t = a;
            t.tile_y = y;
            t.n_tiles = g.tiles;
            t.ncols = w;
            if (Xs) {
                pack_cols_kernel<<<grid_for(xs_rows * (W / 4)), 256, 0, s>>>(a.X, a.ldx, xs_rows, c0, w, W, vec, Xs);
                PYG_LAUNCHED();
                t.X = Xs;
                t.ldx = W;
                t.allow_pad_read = 1;  // zero-padded to W
                t.n_src = xs_rows;
            } else {
                t.X = a.X + c0;
                t.allow_pad_read = a.allow_pad_read && (a.ldx >= (int64_t)align_up((size_t)a.ncols, 4));
            }
            if (hubs) t.part = a.part + c0;
            if (reduce == PYG_MAX) {
                PYG_CUDA(cudaMemsetAsync(Ks, 0, (size_t)a.n_out * W * 8, s));
                t.keys = Ks;
                t.ldk = W;
                PYG_TRY(launch_tile<PYG_MAX>(t, g1, s));
                unpack_cols_kernel<unsigned long long><<<grid_for(a.n_out * w), 256, 0, s>>>(
                    Ks, W, a.n_out, a.keys, a.ldk, c0, w, nullptr);
            } else {
                PYG_CUDA(cudaMemsetAsync(Os, 0, (size_t)a.n_out * W * 4, s));
                t.out = Os;
                t.ldo = W;
                g1.ovk = 1;
                PYG_TRY(launch_tile<PYG_SUM>(t, g1, s));
                unpack_cols_kernel<float><<<grid_for(a.n_out * w), 256, 0, s>>>(
                    Os, W, a.n_out, a.out, a.ldo, c0, w, reduce == PYG_MEAN ? deg : nullptr);
            }
            PYG_LAUNCHED();
            PYG_CUDA(cudaGetLastError());
        }
        if (reduce == PYG_MAX) return max_decode(a.keys, a.ldk, a.out, a.ldo, a.ncols, a.n_out, a.E, s);
    } else if (reduce == PYG_MAX) {
        if (g.tile_lpr) PYG_TRY(launch_tile<PYG_MAX>(a, g, s));
        else PYG_TRY(launch_red<PYG_MAX>(a, g.V, g.nch, g.lpr, g.tiles, epg, g.ovk, s));
        return max_decode(a.keys, a.ldk, a.out, a.ldo, a.ncols, a.n_out, a.E, s);
    } else {
        if (g.tile_lpr) PYG_TRY(launch_tile<PYG_SUM>(a, g, s));
        else PYG_TRY(launch_red<PYG_SUM>(a, g.V, g.nch, g.lpr, g.tiles, epg, g.ovk, s));
        if (reduce == PYG_MEAN) PYG_TRY(mean_divide(a.out, a.ldo, a.ncols, a.n_out, deg, s));
    }
    if (hubs) {
        const int ct = (int)std::min<int64_t>(256, align_up((size_t)a.ncols, 32));
        const int blocks = (int)std::min<int64_t>(hub_cap(a.E), 148 * 8);
        if (reduce == PYG_MEAN)
            hub_combine_kernel<PYG_MEAN><<<blocks, ct, 0, s>>>(a.out, a.ldo, a.ncols, a.part, a.ldp, hub_rows,
                                                              a.hub_base, deg, counters);
        else
            hub_combine_kernel<PYG_SUM><<<blocks, ct, 0, s>>>(a.out, a.ldo, a.ncols, a.part, a.ldp, hub_rows,
                                                             a.hub_base, deg, counters);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    return PYG_OK;
}

pyg_status_t coo_degree(const int64_t* sidx, int64_t E, int64_t n, int32_t* deg, int32_t* first,
                        cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    if (deg) PYG_CUDA(cudaMemsetAsync(deg, 0, (size_t)n * 4, s));
    if (first) PYG_CUDA(cudaMemsetAsync(first, 0x7f, (size_t)n * 4, s));
    if (E <= 0) return PYG_OK;
    degree_kernel<<<grid_for(E), 256, 0, s>>>(sidx, E, deg, first);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t mean_divide(float* out, int64_t ldo, int ncols, int64_t n, const int32_t* deg, cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return PYG_OK;
    mean_div_kernel<<<grid_for(n * ncols), 256, 0, s>>>(out, ldo, ncols, n, deg);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t max_decode(unsigned long long* keys, int64_t ldk, float* out, int64_t ldo, int ncols, int64_t n,
                        int64_t E, cudaStream_t s) {
    if (n <= 0 || ncols <= 0) return PYG_OK;
    max_decode_kernel<<<grid_for(n * ncols), 256, 0, s>>>(keys, ldk, out, ldo, ncols, n, E);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
