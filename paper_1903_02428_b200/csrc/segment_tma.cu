// segment_tma.cu -- host side of the TMA gather4 pipeline (kernel in segment_tma.cuh; the
// kernel instantiations per reduction live in segment_tma_red{0,1,2}.cu so they compile in
// parallel): eligibility, ring geometry, tensor map, launch, empty-row fill.
#include "segment_tma.cuh"

namespace pyg {
namespace tma {

extern template pyg_status_t launch_nch<PYG_SUM>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
extern template pyg_status_t launch_nch<PYG_MEAN>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
extern template pyg_status_t launch_nch<PYG_MAX>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
extern template pyg_status_t launch_nch<kRedSumEpi>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
extern template pyg_status_t launch_nch<kRedHeadW>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
extern template pyg_status_t launch_nch<kRedMaxW>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);

// empty rows: out = 0 (or the APPNP teleport term / GCN bias), arg = E.  Flattened over the
// [empty rows x F] block so consecutive threads store consecutive 16 bytes (the stores stream instead of
// waiting on one row index per warp; R-MAT: 5M empty rows, 2.5 GB of zeros + 5 GB of int64 args)
__global__ void empty_rows_kernel(const int32_t* __restrict__ order, int64_t begin, int64_t end, int64_t row_lo,
                                  int64_t row_hi, int ncols, float* out, int64_t ldo, int64_t* arg, int64_t lda,
                                  int64_t E, int vec_ok, const float* blend, int64_t ldb, float blend_b,
                                  const float* col_bias) {
    const bool vec = vec_ok && !blend && !col_bias;
    const int per = vec ? ncols / 4 : ncols;  // out units per row (float4 or float)
    const int64_t rows = end - begin;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    for (int64_t t = t0; t < rows * per; t += stride) {
        const int64_t k = t / per;
        const int u = (int)(t - k * per);
        const int64_t r = (int64_t)__ldg(order + begin + k);
        if (r < row_lo || r >= row_hi) continue;
        float* o = out + (r - row_lo) * ldo;
        if (vec) {
            reinterpret_cast<float4*>(o)[u] = make_float4(0.f, 0.f, 0.f, 0.f);
        } else {  // APPNP: an empty row keeps only the teleport term; GCN: the bias
            const float* hb = blend ? blend + (r - row_lo) * ldb : nullptr;
            o[u] = (hb ? fmaf(blend_b, hb[u], 0.0f) : 0.0f) + (col_bias ? __ldg(col_bias + u) : 0.0f);
        }
    }
    if (!arg) return;
    // args: pairs of int64 (16-byte stores) when the row is 16-byte aligned, else single values
    const bool pairs = (ncols % 2 == 0) && (lda % 2 == 0) && !(reinterpret_cast<uintptr_t>(arg) & 15);
    const int pa = pairs ? ncols / 2 : ncols;
    for (int64_t t = t0; t < rows * pa; t += stride) {
        const int64_t k = t / pa;
        const int u = (int)(t - k * pa);
        const int64_t r = (int64_t)__ldg(order + begin + k);
        if (r < row_lo || r >= row_hi) continue;
        int64_t* ap = arg + (r - row_lo) * lda;
        if (pairs) reinterpret_cast<longlong2*>(ap)[u] = make_longlong2(E, E);
        else ap[u] = E;
    }
}

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

// The empty rows of a plan (tail of row_order from empty_begin), after the gather kernel.  (Filling
// them on a side stream concurrently with the gather measured no gain for R-MAT sum, 10.68 vs
// 10.71 ms, and a loss for max, 15.5 vs 13.5 ms: the 7.7 GB of value + arg stores compete with the
// gather for DRAM; gpurun_out/r2x.)
pyg_status_t fill_empty(const SegArgs& a, int reduce, const pyg_plan* plan, int F, cudaStream_t s) {
    const int64_t n_empty = plan->n_empty;
    if (n_empty <= 0) return PYG_OK;
    const int vec_ok = (F % 4 == 0) && (a.ldo % 4 == 0) && ((reinterpret_cast<uintptr_t>(a.out) & 15) == 0);
    const int64_t units = n_empty * (int64_t)F;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(units, 256 * 4), 148 * 8));
    tma::empty_rows_kernel<<<blocks, 256, 0, s>>>(
        plan->row_order, plan->empty_begin, plan->empty_begin + n_empty, plan->row_offset,
        plan->row_offset + plan->n_rows, F, a.out, a.ldo, reduce == PYG_MAX ? a.arg : nullptr, a.lda, a.E_sentinel,
        vec_ok, a.blend, a.ldb, a.blend_b, reduce == PYG_MAX ? nullptr : a.col_bias);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

// Whether the TMA path applies: unblocked propagate plan with tasks, 16-byte rows, F in [64, 1024].
bool tma_eligible(const SegArgs& a, const pyg_plan* plan) {
    const int mode = knobs().seg_tma;  // PYG_SEG_TMA unset: auto, 0: off, 1: whenever possible (tests)
    if (mode == 0 || (a.flags & PYG_NO_TMA) || !plan || !plan->parts.empty() || plan->n_tasks <= 0 ||
        !plan->task_pos || !plan->pos_row)
        return false;
    if (!a.gidx || a.gdeg || a.accum || a.deg_total) return false;
    if (a.hw && a.hC % 4) return false;  // a float4 chunk must stay inside one head
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

    // ring budget per warp: 4 KB (R-MAT F=128 -> S = 2 stages of 2 KB) measured best (sum 10.6 ms
    // vs 12.9 ms at 8 KB and 22 ms at 12 KB): more resident warps beat deeper rings
    const int budget = knobs().tma_warp_kb * 1024;
    int warps = knobs().tma_warps;
    if (warps != 2 && warps != 4 && warps != 8) warps = 8;
    int S = std::max(2, std::min(8, budget / stage_bytes));
    if (S == 5) S = 4;
    if (S == 7) S = 6;
    const int head = 128 + (int)align_up((size_t)kMetaBytes * 8, 128);
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
    t.task_item = plan->task_item;
    t.n_tasks = part ? plan->n_tasks : plan->n_light_tasks;
    t.next = counter;
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
    t.row_lo = plan->row_offset;
    t.row_hi = plan->row_offset + plan->n_rows;
    t.E_sentinel = a.E_sentinel;
    t.row_scale = a.row_scale;
    t.col_bias = a.col_bias;
    t.hw = a.hw;
    t.hH = a.hH;
    t.hC = a.hC;
    t.blend = a.blend;
    t.ldb = a.ldb;
    t.blend_a = a.blend_a;
    t.blend_b = a.blend_b;
    t.warp_bytes = warp_bytes;
    t.data_off = head;

    const int64_t want = cdiv(t.n_tasks, warps);
    const bool extras = a.row_scale || a.blend || a.col_bias;
    if (extras && reduce != PYG_SUM) return fail(PYG_ERR_UNSUPPORTED, "internal: TMA epilogue extras need SUM");
    if (extras && a.hw) return fail(PYG_ERR_UNSUPPORTED, "internal: TMA epilogue extras with head weights");
    const int mode = extras ? kRedSumEpi : (reduce == PYG_MAX && a.w) ? kRedMaxW : reduce;
    switch (mode) {
        case kRedMaxW: PYG_TRY(launch_nch<kRedMaxW>(nch, S, want, warps * 32, smem, s, tm, t)); break;
        case kRedSumEpi: PYG_TRY(launch_nch<kRedSumEpi>(nch, S, want, warps * 32, smem, s, tm, t)); break;
        case kRedHeadW: PYG_TRY(launch_nch<kRedHeadW>(nch, S, want, warps * 32, smem, s, tm, t)); break;
        case PYG_SUM: PYG_TRY(launch_nch<PYG_SUM>(nch, S, want, warps * 32, smem, s, tm, t)); break;
        case PYG_MEAN: PYG_TRY(launch_nch<PYG_MEAN>(nch, S, want, warps * 32, smem, s, tm, t)); break;
        default: PYG_TRY(launch_nch<PYG_MAX>(nch, S, want, warps * 32, smem, s, tm, t)); break;
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return fill_empty(a, reduce, plan, F, s);  // zero the empty rows of this plan
}

}  // namespace pyg
