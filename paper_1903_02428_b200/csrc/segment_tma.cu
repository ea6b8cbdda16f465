// segment_tma.cu -- TMA-pipelined CSR segment-reduce for low-reuse graphs (power-law / R-MAT):
// the gather of x_j rows (Fig. 1) is issued by the Tensor Memory Accelerator with
// `cp.async.bulk.tensor.2d.tile::gather4` (SASS UTMALDG.2D.GATHER4: 4 arbitrary rows per
// instruction) into a per-warp ring of shared-memory stages, so each warp keeps (S-1)*4 rows in
// flight without spending registers on them -- what a DRAM-latency-bound random-row gather needs.
//
//   * work = plan-time tasks: runs of consecutive light rows with <= kTaskPositions positions, i.e.
//     contiguous position ranges (balanced regardless of degree skew); a warp streams its tasks
//     back to back without draining the ring;
//   * producer step (warp-uniform): positions advance 4 per stage; the gathered ids, row ids,
//     scales and edge ids come from 32-wide coalesced index windows (the next window is
//     prefetched); lanes 0..3 take their slot's values with ONE shuffle per field and store the
//     slot metadata to shared memory; lane 0 issues one gather4 per column box on the stage's
//     mbarrier (arrive.expect_tx);
//   * consumer step: wait on the stage's mbarrier, accumulate the 4 rows in position order
//     (same arithmetic as seg_kernel => bitwise-identical results) and flush a row when the next
//     slot's row differs (mean divides by the count of accumulated positions = the degree, since
//     tasks never split a row);
//   * empty rows are zero-filled by `empty_rows_kernel`; rows longer than kHeavyThreshold keep the
//     split path (seg_kernel mode 1 + fp64 combine).
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
    float* part;              // [items x ldp] chunk partials (fp32), arg partials (MAX)
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
    int stages;             // ring depth per warp (<= 16)
    int64_t row_lo, row_hi; // this plan's root rows; out row = r - row_lo
    int64_t E_sentinel;
    int warp_bytes;         // shared memory per warp
    int data_off;           // offset of stage data inside the warp region
};

struct alignas(16) Meta {
    int row;
    float scale;
    int eid;
    int pad;
};

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

template <int RED, int NCH>
__global__ void __launch_bounds__(512) seg_tma_kernel(const __grid_constant__ CUtensorMap tmap, Args a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const int S = a.stages;
    unsigned char* region = smem + (size_t)warp * a.warp_bytes;
    const uint32_t bar0 = (uint32_t)__cvta_generic_to_shared(region);
    Meta* meta = reinterpret_cast<Meta*>(region + 128);  // after 16 barriers
    float* data = reinterpret_cast<float*>(region + a.data_off);
    const uint32_t data0 = (uint32_t)__cvta_generic_to_shared(data);
    const int stage_floats = 4 * a.nb * a.box_w;
    const uint32_t stage_bytes = (uint32_t)stage_floats * 4u;

    if (lane == 0) {
        for (int s = 0; s < S; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // per-lane smem offsets of its float4 chunks inside a stage (row 0); row i adds i*box_w
    int coff[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int c = 4 * (lane + 32 * ch);
        const int b = c / a.box_w, cc = c - b * a.box_w;
        coff[ch] = b < a.nb ? b * 4 * a.box_w + cc : 0;
    }
    const bool need_e = (RED == PYG_MAX) || (a.w != nullptr);
    // this plan's positions (slices restrict the root tasks)
    const int64_t plo = __ldg(a.rowptr + a.row_lo), phi = __ldg(a.rowptr + a.row_hi);

    const int64_t twarps = (int64_t)gridDim.x * (blockDim.x >> 5);
    int64_t task = (int64_t)blockIdx.x * (blockDim.x >> 5) + warp;

    // ---------------- producer state (warp-uniform) ----------------
    int64_t pp = 0, pe = 0;  // position cursor / end of the current task range
    bool done = false;
    // index windows: lane j holds gathered id / row / edge id / scale of position base + j
    int64_t iwb = 0, nwb = -1;
    int wg = 0, wr = 0, we = 0, ng = 0, nr = 0, ne = 0;
    float ws = 1.0f, ns = 1.0f;
    auto load_window = [&](int64_t base, int& g, int& r, int& e, float& sc) {
        const int64_t p = base + lane;
        g = 0; r = -1; e = 0; sc = 1.0f;
        if (p < a.E_root) {
            g = __ldg(a.gidx + p);
            r = __ldg(a.pos_row + p);
            if (need_e) e = a.eid ? __ldg(a.eid + p) : (int)p;
            if (a.w) sc = __ldg(a.w + e);
        }
    };
    int citem = -1;  // split-row item of the current task (hub chunk), or -1
    // first task static (warp id), later ones taken dynamically from a global counter: tasks differ
    // in cost (size, L2 locality), so static striding leaves a tail
    bool first = true;
    auto next_task = [&]() -> bool {
        for (;;) {
            if (!first) {
                unsigned long long t = 0;
                if (lane == 0) t = atomicAdd(a.next, 1ull);
                task = twarps + (int64_t)__shfl_sync(0xffffffffu, t, 0);
            }
            first = false;
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
        return false;
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
    if (next_task()) set_window(pp); else done = true;

    // fill stage s with the next (up to) 4 positions of the stream; returns the slot count
    auto fill = [&](int s) -> int {
        if (done) return 0;
        if (pp - iwb >= 32) set_window(pp);
        const int j = (int)(pp - iwb);           // multiple of 4 within the window
        const int cnt = (int)min((int64_t)4, pe - pp);
        const int src = j + (lane & 3);
        const int g = __shfl_sync(0xffffffffu, wg, src);
        const int r = __shfl_sync(0xffffffffu, wr, src);
        int e = 0;
        float sc = 1.0f;
        if (need_e) e = __shfl_sync(0xffffffffu, we, src);
        if (a.w) sc = __shfl_sync(0xffffffffu, ws, src);
        const int g0 = __shfl_sync(0xffffffffu, g, 0);
        const int g1 = __shfl_sync(0xffffffffu, g, cnt > 1 ? 1 : 0);
        const int g2 = __shfl_sync(0xffffffffu, g, cnt > 2 ? 2 : 0);
        const int g3 = __shfl_sync(0xffffffffu, g, cnt > 3 ? 3 : 0);
        // slot key: the root row, or -(item + 2) for a hub chunk (its partial goes to `part`)
        const int key = citem >= 0 ? -(citem + 2) : r;
        if (lane < 4) meta[s * 4 + lane] = Meta{lane < cnt ? key : -1, sc, e, 0};
        __syncwarp();
        if (lane == 0) {
            const uint32_t bar = bar0 + 8 * s;
            bar_expect(bar, stage_bytes);
            const uint32_t dst = data0 + (uint32_t)(s * stage_floats) * 4u;
            for (int b = 0; b < a.nb; ++b)
                gather4(dst + (uint32_t)(b * 4 * a.box_w) * 4u, &tmap, b * a.box_w, g0, g1, g2, g3, bar);
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
            for (int q = 0; q < 4; ++q) { acc[ch][q] = RED == PYG_MAX ? -INFINITY : 0.0f; bi[ch][q] = -1; }
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
                    if (RED == PYG_MAX) pa[col + q] = bi[ch][q];
                }
            }
            return;
        }
        const int64_t orow = (int64_t)crow - a.row_lo;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const int col = 4 * (lane + 32 * ch);
            if (col >= a.ncols) continue;
            const int nv = min(4, a.ncols - col);
            float* o = a.out + orow * a.ldo + col;
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                if (q >= nv) continue;
                float v;
                if (RED == PYG_MAX) v = bi[ch][q] >= 0 ? acc[ch][q] : 0.0f;
                else if (RED == PYG_MEAN) v = acc[ch][q] / (float)ccount;
                else v = acc[ch][q];
                o[q] = v;
            }
            if (RED == PYG_MAX) {
                int64_t* ap = a.arg + orow * a.lda + col;
#pragma unroll
                for (int q = 0; q < 4; ++q) if (q < nv) ap[q] = bi[ch][q] >= 0 ? (int64_t)bi[ch][q] : a.E_sentinel;
            }
        }
    };

    // prologue: fill the ring; the per-stage slot count is kept in a 16 x 3-bit register array
    uint64_t cnts = 0;
    for (int s = 0; s < S; ++s) cnts |= (uint64_t)fill(s) << (3 * s);
    uint32_t phase = 0;
    reset();
    for (int s = 0;;) {
        const int cnt = (int)((cnts >> (3 * s)) & 7u);
        if (cnt == 0) break;
        bar_wait(bar0 + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
        const float* st = data + s * stage_floats;
        const Meta* ms = meta + s * 4;
        auto slot = [&](const Meta& m, int i) {
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const float4 v = *reinterpret_cast<const float4*>(st + coff[ch] + i * a.box_w);
                const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (RED == PYG_MAX) {
                        const float mm = __fmul_rn(m.scale, vv[q]);
                        if (bi[ch][q] < 0 || mm > acc[ch][q]) { acc[ch][q] = mm; bi[ch][q] = m.eid; }
                    } else {
                        acc[ch][q] = fmaf(m.scale, vv[q], acc[ch][q]);
                    }
                }
            }
        };
        const Meta m0 = ms[0], m1 = ms[1], m2 = ms[2], m3 = ms[3];
        if (cnt == 4 && m0.row == crow && m3.row == crow) {
            // fast path: a full stage inside the current row (rows never interleave in the stream)
            slot(m0, 0); slot(m1, 1); slot(m2, 2); slot(m3, 3);
            ccount += 4;
        } else {
            for (int i = 0; i < cnt; ++i) {
                const Meta m = i == 0 ? m0 : (i == 1 ? m1 : (i == 2 ? m2 : m3));
                if (m.row != crow) {
                    if (crow != -1) flush();
                    crow = m.row;
                    ccount = 0;
                    reset();
                }
                ++ccount;
                slot(m, i);
            }
        }
        __syncwarp();  // every lane has read stage s before it is refilled
        const int nc = fill(s);
        cnts = (cnts & ~((uint64_t)7 << (3 * s))) | ((uint64_t)nc << (3 * s));
        s = (s + 1 == S) ? 0 : s + 1;
    }
    if (crow != -1) flush();
}

// one warp per empty row: out = 0 (float4 stores when aligned), arg = E
__global__ void empty_rows_kernel(const int32_t* __restrict__ order, int64_t begin, int64_t end, int64_t row_lo,
                                  int64_t row_hi, int ncols, float* out, int64_t ldo, int64_t* arg, int64_t lda,
                                  int64_t E, int vec_ok) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < end; k += warps) {
        const int64_t r = (int64_t)order[k];
        if (r < row_lo || r >= row_hi) continue;
        float* o = out + (r - row_lo) * ldo;
        if (vec_ok) {
            for (int c = 4 * lane; c < ncols; c += 128) *reinterpret_cast<float4*>(o + c) = make_float4(0, 0, 0, 0);
        } else {
            for (int c = lane; c < ncols; c += 32) o[c] = 0.0f;
        }
        if (arg) {
            int64_t* ap = arg + (r - row_lo) * lda;
            for (int c = lane; c < ncols; c += 32) ap[c] = E;
        }
    }
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
    static EncodeFn fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* p = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<EncodeFn>(p);
    });
    return fn;
}

}  // namespace tma

// Whether the TMA path applies: unblocked propagate plan with tasks, 16-byte rows, F in [64, 1024].
bool tma_eligible(const SegArgs& a, const pyg_plan* plan) {
    const char* env = getenv("PYG_SEG_TMA");  // unset: auto, 0: off, 1: whenever possible (tests)
    const int mode = env ? atoi(env) : -1;
    if (mode == 0 || (a.flags & PYG_NO_TMA) || !plan || !plan->parts.empty() || plan->n_tasks <= 0 ||
        !plan->task_pos || !plan->pos_row)
        return false;
    if (!a.gidx || a.gdeg || a.accum || a.deg_total) return false;
    if (a.ncols < 64 || a.ncols > 1024) return false;
    // enough tasks to keep every SM's warps streaming (small graphs are launch/latency-bound and
    // faster on the LDG kernel: PubMed-shaped measured 0.046 ms LDG vs 1.16 ms TMA)
    if (mode != 1 && plan->n_light_tasks < 1024) return false;
    if ((reinterpret_cast<uintptr_t>(a.X) & 15) || (a.ldx % 4)) return false;
    if (!tma::encode_fn()) return false;
    return true;
}

pyg_status_t segment_tma(const SegArgs& a, int reduce, const pyg_plan* plan, unsigned long long* counter,
                         float* part, int32_t* part_arg, int64_t ldp, cudaStream_t s) {
    if (!counter) return fail(PYG_ERR_NO_MEMORY, "TMA path needs workspace (see pyg_workspace_size)");
    PYG_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    using namespace tma;
    const int F = a.ncols;
    const int nb = (F + 255) / 256;
    const int box_w = (int)align_up((size_t)((F + nb - 1) / nb), 8);  // 128-byte aligned box destinations
    const int nch = (int)cdiv(nb * box_w, 128);
    const int stage_bytes = 16 * nb * box_w;
    static const int budget = [] {
        const char* e = getenv("PYG_TMA_WARP_KB");
        return (e ? atoi(e) : 8) * 1024;  // measured best on R-MAT F=128 (S = 4 stages of 2 KB)
    }();
    static const int warps = [] {
        const char* e = getenv("PYG_TMA_WARPS");
        const int w = e ? atoi(e) : 8;
        return (w == 2 || w == 4 || w == 8 || w == 16) ? w : 8;
    }();
    const int S = std::max(2, std::min(16, budget / stage_bytes));
    const int head = 128 + (int)align_up(sizeof(Meta) * 4 * 16, 128);
    const int warp_bytes = (int)align_up((size_t)(head + S * stage_bytes), 128);
    const int smem = warps * warp_bytes;

    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)F, (cuuint64_t)plan->n_cols};
    cuuint64_t gstr[1] = {(cuuint64_t)a.ldx * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_w, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult cr = encode_fn()(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(a.X), gdim, gstr, box, es,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (cr != CUDA_SUCCESS) return fail(PYG_ERR_CUDA, "cuTensorMapEncodeTiled failed (%d)", (int)cr);

    Args t;
    t.rowptr = plan->rowptr - plan->row_offset;
    t.pos_row = plan->pos_row;
    t.task_pos = plan->task_pos;
    t.n_tasks = part ? plan->n_tasks : plan->n_light_tasks;
    t.next = counter;
    t.task_item = plan->task_item;
    t.part = part;
    t.part_arg = part_arg;
    t.ldp = ldp;
    t.item_lo = plan->item_lo;
    t.E_root = plan->E;
    t.gidx = a.gidx;
    t.eid = a.eid;
    t.w = a.w;
    t.out = a.out;
    t.ldo = a.ldo;
    t.arg = a.arg;
    t.lda = a.lda;
    t.ncols = F;
    t.box_w = box_w;
    t.nb = nb;
    t.stages = S;
    t.row_lo = plan->row_offset;
    t.row_hi = plan->row_offset + plan->n_rows;
    t.E_sentinel = a.E_sentinel;
    t.warp_bytes = warp_bytes;
    t.data_off = head;

    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = cdiv(t.n_tasks, warps);
    const int per_sm = std::max(1, (220 * 1024) / smem);
    const unsigned grid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * per_sm));

#define PYG_TMA_CASE(R, N)                                                                    \
    if (reduce == R && nch == N) {                                                            \
        auto k = seg_tma_kernel<R, N>;                                                        \
        PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem)); \
        k<<<grid, warps * 32, smem, s>>>(tm, t);                                              \
        launched = true;                                                                      \
    }
    bool launched = false;
    PYG_TMA_CASE(PYG_SUM, 1) PYG_TMA_CASE(PYG_SUM, 2) PYG_TMA_CASE(PYG_SUM, 3) PYG_TMA_CASE(PYG_SUM, 4)
    PYG_TMA_CASE(PYG_SUM, 5) PYG_TMA_CASE(PYG_SUM, 6) PYG_TMA_CASE(PYG_SUM, 7) PYG_TMA_CASE(PYG_SUM, 8)
    PYG_TMA_CASE(PYG_MEAN, 1) PYG_TMA_CASE(PYG_MEAN, 2) PYG_TMA_CASE(PYG_MEAN, 3) PYG_TMA_CASE(PYG_MEAN, 4)
    PYG_TMA_CASE(PYG_MEAN, 5) PYG_TMA_CASE(PYG_MEAN, 6) PYG_TMA_CASE(PYG_MEAN, 7) PYG_TMA_CASE(PYG_MEAN, 8)
    PYG_TMA_CASE(PYG_MAX, 1) PYG_TMA_CASE(PYG_MAX, 2) PYG_TMA_CASE(PYG_MAX, 3) PYG_TMA_CASE(PYG_MAX, 4)
    PYG_TMA_CASE(PYG_MAX, 5) PYG_TMA_CASE(PYG_MAX, 6) PYG_TMA_CASE(PYG_MAX, 7) PYG_TMA_CASE(PYG_MAX, 8)
#undef PYG_TMA_CASE
    if (!launched) return fail(PYG_ERR_INVALID_ARGUMENT, "internal: no TMA kernel for nch=%d", nch);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());

    // zero-fill the empty rows of this plan
    const int64_t n_empty = plan->n_empty;
    if (n_empty > 0) {
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n_empty, 8), 148 * 16));
        const int vec_ok = (F % 4 == 0) && (a.ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
        empty_rows_kernel<<<blocks, 256, 0, s>>>(plan->row_order, plan->empty_begin, plan->empty_begin + n_empty,
                                                 plan->row_offset, plan->row_offset + plan->n_rows, F, a.out, a.ldo,
                                                 reduce == PYG_MAX ? a.arg : nullptr, a.lda, a.E_sentinel, vec_ok);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    return PYG_OK;
}

}  // namespace pyg
