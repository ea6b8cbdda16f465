// segment_tma.cuh -- TMA-pipelined CSR segment-reduce for low-reuse graphs (power-law / R-MAT):
// the gather of x_j rows (Fig. 1) is issued by the Tensor Memory Accelerator with
// `cp.async.bulk.tensor.2d.tile::gather4` (SASS UTMALDG.2D.GATHER4: 4 arbitrary rows per
// instruction) into a per-warp ring of S shared-memory stages, so each warp keeps (S-1)*4 rows in
// flight without spending registers on them -- what a DRAM-latency-bound random-row gather needs.
//
//   * work = plan-time tasks: runs of consecutive light rows with <= kTaskPositions positions
//     (contiguous position ranges), then one task per 512-position chunk of every split hub row;
//     the first task of a warp is static, the rest come from a global atomic counter;
//   * producer step (warp-uniform): positions advance 4 per stage; the gathered ids / row ids /
//     edge ids / scales come from 32-wide coalesced index windows (the next window is prefetched);
//     lanes 0..3 take their slot's values with ONE shuffle per field and store the slot metadata
//     (structure-of-arrays: 4 keys | 4 scales | 4 edge ids per stage); lane 0 arms the stage's
//     mbarrier (arrive.expect_tx) and issues one gather4 per column box;
//   * consumer step: wait on the mbarrier, accumulate the 4 rows in position order (same
//     arithmetic as seg_kernel => bitwise-identical results); a full stage inside the current row
//     takes an unrolled fast path; a row is flushed when the next slot's key differs (mean divides
//     by the count of accumulated positions = the degree, since tasks never split a light row);
//     hub-chunk tasks write fp32 partials for the fp64 combine instead;
//   * S (ring depth) is a template parameter so every stage address and count is compile-time;
//   * empty rows are zero-filled by `empty_rows_kernel`.
#pragma once

#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace pyg {
namespace tma {

struct Args {
    const int64_t* rowptr;  // ROOT rowptr
    const int32_t* pos_row; // ROOT row of each position
    const int64_t* task_pos;
    const int32_t* task_item;  // hub chunk tasks: split-row item id (partials), else -1
    int64_t n_tasks;
    unsigned long long* next;  // dynamic task counter (zeroed before the launch)
    float* part;               // [items x ldp] chunk partials (fp32), arg partials (MAX)
    int32_t* part_arg;
    int64_t ldp, item_lo;
    int64_t E_root;
    const int32_t* gidx;
    const int32_t* eid;     // null => identity
    const float* w;
    float* out;
    int64_t ldo;
    int64_t* arg;
    int64_t lda;
    int ncols;
    int box_w;              // floats per gather4 row (multiple of 8, <= 256)
    int nb;                 // column boxes per row
    int64_t row_lo, row_hi; // this plan's root rows; out row = r - row_lo
    int64_t E_sentinel;
    const float* row_scale; // GCN-layer epilogue: v *= row_scale[row], then + col_bias[c]
    const float* col_bias;
    const float* blend;     // APPNP epilogue (light rows): out = blend_a * v + blend_b * blend[row]
    int64_t ldb;
    float blend_a, blend_b;
    const float* hw;        // kRedHeadW: alpha [E x hH] by edge id, column c in head c / hC
    int hH, hC;
    int warp_bytes;         // shared memory per warp
    int data_off;           // offset of stage data inside the warp region
};

constexpr int kMetaBytes = 48;  // per stage: int keys[4] | float scales[4] | int eids[4]

__device__ __forceinline__ void bar_init(uint32_t bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar));
}
__device__ __forceinline__ void bar_expect(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " TMA_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra TMA_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* tmap, int c0, int r0, int r1, int r2, int r3,
                                        uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst),
        "l"(tmap), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void sts32(uint32_t addr, int v) {
    asm volatile("st.shared.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
__device__ __forceinline__ int4 lds128(uint32_t addr) {
    int4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
    return v;
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

template <int RED, int NCH, int S>
__global__ void __launch_bounds__(256) seg_tma_kernel(const __grid_constant__ CUtensorMap tmap, Args a) {
    constexpr bool EPI = RED == kRedSumEpi;        // SUM + row scale / blend / bias epilogue
    constexpr bool HW = RED == kRedHeadW;          // SUM with per-(edge, head) weights (GAT)
    constexpr bool MAXW = RED == kRedMaxW;         // MAX of weighted messages
    constexpr int RR = (EPI || HW) ? PYG_SUM : (MAXW ? PYG_MAX : RED);  // the reduction itself
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t region = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(warp * a.warp_bytes);
    const uint32_t bar0 = region;                 // S barriers (8 B each, <= 16)
    const uint32_t meta0 = region + 128;          // S x kMetaBytes
    const uint32_t data0 = region + (uint32_t)a.data_off;
    const int box_w = a.box_w, nb = a.nb;
    const uint32_t stage_bytes = (uint32_t)(16 * nb * box_w);
    const uint32_t row_bytes = (uint32_t)(4 * box_w);

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // per-lane byte offsets of its float4 chunks inside a stage (slot 0); slot i adds i*row_bytes
    uint32_t coff[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int c = 4 * (lane + 32 * ch);
        const int b = c / box_w, cc = c - b * box_w;
        coff[ch] = b < nb ? (uint32_t)(4 * (b * 4 * box_w + cc)) : 0u;
    }
    const bool need_e = (RR == PYG_MAX) || (a.w != nullptr) || HW;
    const bool weighted = RED != PYG_MAX && a.w != nullptr;  // PYG_MAX instantiation: unweighted
    int hch[NCH];  // kRedHeadW: head of each float4 chunk (hC % 4 == 0)
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) hch[ch] = HW ? min(4 * (lane + 32 * ch), a.ncols - 1) / a.hC : 0;
    // this plan's positions (slices restrict the root tasks)
    const int64_t plo = __ldg(a.rowptr + a.row_lo), phi = __ldg(a.rowptr + a.row_hi);
    const int64_t twarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;

    // ---------------- producer state (warp-uniform) ----------------
    int64_t pp = 0, pe = 0;  // position cursor / end of the current task range
    bool done = false;
    int64_t iwb = 0, nwb = -1;
    int wg = 0, wr = 0, we = 0, ng = 0, nr = 0, ne = 0;
    float ws = 1.0f, ns = 1.0f;
    int citem = -1;
    bool first = true;

    auto load_window = [&](int64_t base, int& g, int& r, int& e, float& sc) {
        const int64_t p = base + lane;
        g = 0; r = -1; e = 0; sc = 1.0f;
        if (p < a.E_root) {
            g = __ldg(a.gidx + p);
            r = __ldg(a.pos_row + p);
            if (need_e) e = a.eid ? __ldg(a.eid + p) : (int)p;
            if (weighted) sc = __ldg(a.w + e);
        }
    };
    auto set_window = [&](int64_t base) {
        if (base == nwb) {
            wg = ng; wr = nr; we = ne; ws = ns;
        } else {
            load_window(base, wg, wr, we, ws);
        }
        iwb = base;
        nwb = base + 32;  // speculative prefetch of the continuation
        load_window(nwb, ng, nr, ne, ns);
    };
    // every task comes from the global counter (a static first task would stall behind CTAs that
    // are not resident yet)
    (void)first;
    (void)twarps;
    auto next_task = [&]() -> bool {
        for (;;) {
            {
                unsigned long long t = 0;
                if (lane == 0) t = atomicAdd(a.next, 1ull);
                task = (int64_t)__shfl_sync(0xffffffffu, t, 0);
            }
            if (task >= a.n_tasks) return false;
            const int64_t t0 = max(__ldg(a.task_pos + 2 * task), plo);
            const int64_t t1 = min(__ldg(a.task_pos + 2 * task + 1), phi);
            const int it = a.task_item ? __ldg(a.task_item + task) : -1;
            if (t0 < t1 && (it < 0 || a.part)) {
                pp = t0;
                pe = t1;
                citem = it;
                return true;
            }
        }
    };
    if (next_task()) set_window(pp); else done = true;

    // fill stage s with the next (up to) 4 positions of the stream; returns the slot count
    auto fill = [&](int s) -> int {
        if (done) {  // mark the stage empty (the consumer stops at a stage without valid slots)
            if (lane < 4) sts32(meta0 + (uint32_t)(s * kMetaBytes) + 4u * (uint32_t)lane, -1);
            return 0;
        }
        if (pp - iwb >= 32) set_window(pp);
        const int j = (int)(pp - iwb);  // multiple of 4 within the window
        const int cnt = (int)min((int64_t)4, pe - pp);
        const int src = j + (lane & 3);
        const int g = __shfl_sync(0xffffffffu, wg, src);
        int key = __shfl_sync(0xffffffffu, wr, src);
        if (citem >= 0) key = -(citem + 2);  // hub chunk: its partial goes to `part`
        const uint32_t m = meta0 + (uint32_t)(s * kMetaBytes) + 4u * (uint32_t)lane;
        if (weighted) {
            const float sc = __shfl_sync(0xffffffffu, ws, src);
            if (lane < 4) sts32(m + 16, __float_as_int(sc));
        }
        if (need_e) {
            const int e = __shfl_sync(0xffffffffu, we, src);
            if (lane < 4) sts32(m + 32, e);
        }
        if (lane < 4) sts32(m, lane < cnt ? key : -1);
        const int g1 = __shfl_sync(0xffffffffu, g, cnt > 1 ? 1 : 0);
        const int g2 = __shfl_sync(0xffffffffu, g, cnt > 2 ? 2 : 0);
        const int g3 = __shfl_sync(0xffffffffu, g, cnt > 3 ? 3 : 0);
        if (lane == 0) {
            const uint32_t bar = bar0 + 8 * s;
            bar_expect(bar, stage_bytes);
            const uint32_t dst = data0 + (uint32_t)s * stage_bytes;
#pragma unroll
            for (int b = 0; b < NCH; ++b)
                if (b < nb) gather4(dst + (uint32_t)b * 4u * row_bytes, &tmap, b * box_w, g, g1, g2, g3, bar);
        }
        pp += cnt;
        if (pp >= pe) {
            if (next_task()) {
                if (pp != iwb + 32 && (pp < iwb || pp - iwb >= 32 || ((pp - iwb) & 3))) set_window(pp);
            } else {
                done = true;
            }
        }
        return cnt;
    };

    // ---------------- consumer ----------------
    float acc[NCH][4];
    int bi[NCH][4];
    int crow = -1, ccount = 0;
    auto reset = [&]() {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < 4; ++q) { acc[ch][q] = RR == PYG_MAX ? -INFINITY : 0.0f; bi[ch][q] = -1; }
    };
    auto flush = [&]() {
        if (crow < -1) {  // hub chunk: raw partial (+ arg) for the fp64 combine
            const int64_t it = (int64_t)(-crow - 2) - a.item_lo;
            float* pp_ = a.part + it * a.ldp;
            int32_t* pa = a.part_arg ? a.part_arg + it * a.ldp : nullptr;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const int col = 4 * (lane + 32 * ch);
                if (col >= a.ncols) continue;
                const int nv = min(4, a.ncols - col);
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (q >= nv) continue;
                    pp_[col + q] = acc[ch][q];
                    if (RR == PYG_MAX) pa[col + q] = bi[ch][q];
                }
            }
            return;
        }
        const int64_t orow = (int64_t)crow - a.row_lo;
        // epilogue extras (GCN row scale / APPNP blend / bias) behind one warp-uniform branch: the
        // kernel is issue-bound at F = 128, so the plain store path stays as short as before
        const bool extra = EPI && (a.row_scale || a.blend || a.col_bias);
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int col = 4 * (lane + 32 * ch);
            if (col >= a.ncols) continue;
            const int nv = min(4, a.ncols - col);
            float* o = a.out + orow * a.ldo + col;
            if (extra) {
                const float rsc = a.row_scale ? __ldg(a.row_scale + orow) : 1.0f;
                for (int q = 0; q < nv; ++q) {
                    float v = (RR == PYG_MEAN ? acc[ch][q] / (float)ccount : acc[ch][q]) * rsc;
                    if (a.blend) v = fmaf(a.blend_b, a.blend[orow * a.ldb + col + q], a.blend_a * v);
                    if (a.col_bias) v += __ldg(a.col_bias + col + q);
                    o[q] = v;
                }
                continue;
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q >= nv) continue;
                float v;
                if (RR == PYG_MAX) v = bi[ch][q] >= 0 ? acc[ch][q] : 0.0f;
                else if (RR == PYG_MEAN) v = acc[ch][q] / (float)ccount;
                else v = acc[ch][q];
                o[q] = v;
            }
            if (RR == PYG_MAX) {
                int64_t* ap = a.arg + orow * a.lda + col;
#pragma unroll
                for (int q = 0; q < 4; ++q) if (q < nv) ap[q] = bi[ch][q] >= 0 ? (int64_t)bi[ch][q] : a.E_sentinel;
            }
        }
    };
    auto slot = [&](uint32_t st, int i, float sc, int e) {
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            if constexpr (HW) sc = __ldg(a.hw + (int64_t)e * a.hH + hch[ch]);  // alpha of this chunk's head
            const float4 v = lds128f(st + coff[ch] + (uint32_t)i * row_bytes);
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (RR == PYG_MAX) {
                    const float mm = RED == PYG_MAX ? vv[q] : __fmul_rn(sc, vv[q]);
                    if (mm > acc[ch][q]) { acc[ch][q] = mm; bi[ch][q] = e; }  // acc starts at -inf (Q5: finite inputs)
                } else {
                    acc[ch][q] = fmaf(sc, vv[q], acc[ch][q]);
                }
            }
        }
    };

    // The ring loop is NOT unrolled: an S-times unrolled body overflows the instruction cache
    // (measured: S = 8 unrolled ran 2.6x slower than S = 2).  Slot counts live in shared memory
    // (keys of unused slots are -1).
#pragma unroll 1
    for (int s = 0; s < S; ++s) fill(s);
    __syncwarp();  // slot metadata of the prologue stages visible to every lane
    reset();
    uint32_t phase = 0;
#pragma unroll 1
    for (int s = 0;; s = (s + 1 == S) ? 0 : s + 1) {
        {
            const uint32_t m = meta0 + (uint32_t)(s * kMetaBytes);
            const int4 keys = lds128(m);
            const int c = (keys.x != -1) + (keys.y != -1) + (keys.z != -1) + (keys.w != -1);
            if (c == 0) break;
            bar_wait(bar0 + 8 * s, (phase >> s) & 1u);
            phase ^= 1u << s;
            const uint32_t st = data0 + (uint32_t)s * stage_bytes;
            float4 scs = make_float4(1.0f, 1.0f, 1.0f, 1.0f);
            int4 eids = make_int4(0, 0, 0, 0);
            if (weighted) scs = lds128f(m + 16);
            if (need_e) eids = lds128(m + 32);
            if (c == 4 && keys.x == crow && keys.w == crow) {
                // fast path: a full stage inside the current row (rows never interleave)
                slot(st, 0, scs.x, eids.x);
                slot(st, 1, scs.y, eids.y);
                slot(st, 2, scs.z, eids.z);
                slot(st, 3, scs.w, eids.w);
                ccount += 4;
            } else {
                const int kk[4] = {keys.x, keys.y, keys.z, keys.w};
                const float ss[4] = {scs.x, scs.y, scs.z, scs.w};
                const int ee[4] = {eids.x, eids.y, eids.z, eids.w};
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    if (i >= c) break;
                    if (kk[i] != crow) {
                        if (crow != -1) flush();
                        crow = kk[i];
                        ccount = 0;
                        reset();
                    }
                    ++ccount;
                    slot(st, i, ss[i], ee[i]);
                }
            }
            __syncwarp();  // every lane has read stage s before it is refilled
            fill(s);
        }
    }
    if (crow != -1) flush();
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn();

template <int RED, int NCH>
pyg_status_t launch_s(int S, int64_t want, int threads, int smem, cudaStream_t s, const CUtensorMap& tm,
                      const Args& t) {
    void (*k)(const CUtensorMap, Args) = nullptr;
    switch (S) {
        case 2: k = seg_tma_kernel<RED, NCH, 2>; break;
        case 3: k = seg_tma_kernel<RED, NCH, 3>; break;
        case 4: k = seg_tma_kernel<RED, NCH, 4>; break;
        case 6: k = seg_tma_kernel<RED, NCH, 6>; break;
        default: k = seg_tma_kernel<RED, NCH, 8>; break;
    }
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // Keep >= ~80 KB of the 256 KB unified L1/shared array as L1: the index windows are read
    // through L1, and a carveout that leaves it smaller made the same kernel 3x slower
    // (R-MAT sum: 213 KB of stages per SM -> 27.4 ms, 147 KB -> 8.9 ms; ncu long_scoreboard).
    const int kSmemPerSm = 150 * 1024;
    int dev = 0, sms = 148, per_sm = 1;
    PYG_CUDA(cudaGetDevice(&dev));
    PYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int cap = std::max(1, kSmemPerSm / (smem + 1024));
    const int carve = std::min(100, (int)cdiv((int64_t)cap * (smem + 1024) * 100, 228 * 1024));
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    PYG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, threads, smem));
    per_sm = std::min(per_sm, cap);
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1))));
    k<<<grid, threads, smem, s>>>(tm, t);
    return PYG_OK;
}

template <int RED>
pyg_status_t launch_nch(int nch, int S, int64_t want, int threads, int smem, cudaStream_t s, const CUtensorMap& tm,
                        const Args& t) {
    switch (nch) {
        case 1: return launch_s<RED, 1>(S, want, threads, smem, s, tm, t);
        case 2: return launch_s<RED, 2>(S, want, threads, smem, s, tm, t);
        case 3: return launch_s<RED, 3>(S, want, threads, smem, s, tm, t);
        case 4: return launch_s<RED, 4>(S, want, threads, smem, s, tm, t);
        case 5: return launch_s<RED, 5>(S, want, threads, smem, s, tm, t);
        case 6: return launch_s<RED, 6>(S, want, threads, smem, s, tm, t);
        case 7: return launch_s<RED, 7>(S, want, threads, smem, s, tm, t);
        case 8: return launch_s<RED, 8>(S, want, threads, smem, s, tm, t);
        default: return fail(PYG_ERR_INVALID_ARGUMENT, "internal: no TMA kernel for nch=%d", nch);
    }
}

}  // namespace tma
}  // namespace pyg
