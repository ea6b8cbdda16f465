// segment.cu -- host side of the CSR segment-reduce (kernel in segment_kernel.cuh):
// launch geometry (vector width, lanes per row, chunks per lane, column tiles), the
// split-row (hub) path with its fp64 combine, and source-blocked multi-pass plans.
#include <cstdlib>

#include "segment_kernel.cuh"

namespace pyg {

namespace seg {
extern template pyg_status_t launch<1>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
extern template pyg_status_t launch<2>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
extern template pyg_status_t launch<4>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
extern template pyg_status_t launch<8>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
}  // namespace seg

bool tma_eligible(const SegArgs& a, const pyg_plan* plan);
bool bulk_eligible(const SegArgs& a, const pyg_plan* plan, int reduce);
pyg_status_t segment_bulk(const SegArgs& a, int reduce, unsigned long long* counter, int ovk, cudaStream_t s);
pyg_status_t segment_tma(const SegArgs& a, int reduce, const pyg_plan* plan, unsigned long long* counter,
                         float* part, int32_t* part_arg, int64_t ldp, cudaStream_t s);

namespace {

// fp64 combine of the chunk partials of each split row (deterministic order).
template <int RED>
__global__ void combine_kernel(SegArgs a, seg::HeavyArgs h) {
    const int64_t hr = h.h_lo + blockIdx.x;
    const int64_t r = (int64_t)h.heavy_rows[hr] - h.row_offset;
    const int64_t i0 = h.item_ptr[hr] - h.item_lo, i1 = h.item_ptr[hr + 1] - h.item_lo;
    const int64_t deg = a.deg_total ? (int64_t)a.deg_total[r] : a.rowptr[r + 1] - a.rowptr[r];
    const int64_t ldp = h.ldp;
    for (int col = blockIdx.y * blockDim.x + threadIdx.x; col < a.ncols; col += gridDim.y * blockDim.x) {
        if (RED == PYG_MAX) {
            float best = 0.0f;
            int b = -1;
            for (int64_t it = i0; it < i1; ++it) {
                const int pb = h.part_arg[it * ldp + col];
                const float pv = h.part[it * ldp + col];
                if (pb >= 0 && (b < 0 || pv > best)) { best = pv; b = pb; }
            }
            float* o = a.out + r * a.ldo + col;
            int64_t* ap = a.arg + r * a.lda + col;
            if (!a.accum && a.finalize) {
                *o = b >= 0 ? best : 0.0f;
                *ap = b >= 0 ? (int64_t)b : a.E_sentinel;
            } else {  // multi-pass: packed keys in the arg buffer (see seg_kernel)
                unsigned long long* kp = reinterpret_cast<unsigned long long*>(ap);
                const unsigned long long nk = b >= 0 ? max_key(best, (uint32_t)b) : 0ull;
                const unsigned long long k = a.accum ? (*kp > nk ? *kp : nk) : nk;
                if (a.finalize) {
                    *o = k ? ord2f((uint32_t)(k >> 32)) : 0.0f;
                    *ap = k ? (int64_t)(0xffffffffu - (uint32_t)(k & 0xffffffffu)) : a.E_sentinel;
                } else {
                    *kp = k;
                }
            }
        } else {
            double s = 0.0;
            for (int64_t it = i0; it < i1; ++it) s += (double)h.part[it * ldp + col];
            if (a.accum) s += (double)a.out[r * a.ldo + col];
            if (RED == PYG_MEAN && a.finalize) s = deg > 0 ? s / (double)deg : 0.0;
            if (a.row_scale && a.finalize) s *= (double)a.row_scale[r];
            if (a.blend && a.finalize)
                s = (double)a.blend_a * s + (double)a.blend_b * (double)a.blend[r * a.ldb + col];
            if (a.col_bias && a.finalize) s += (double)a.col_bias[col];
            a.out[r * a.ldo + col] = (float)s;
        }
    }
}

bool aligned(const void* p, int bytes) { return (reinterpret_cast<uintptr_t>(p) % bytes) == 0; }

constexpr int kNch[] = {1, 2, 3, 4, 5, 6, 8, 12, 16};

struct Geometry {
    int V, lpr, nch, tiles;
    double util;  // useful fraction of the lane x chunk slots
};

Geometry geometry(int64_t ncols, int V) {
    Geometry g{V, 4, 1, 1, 0.0};
    const int64_t nvec = cdiv(ncols, V);
    if (nvec <= 32) {
        while (g.lpr < nvec) g.lpr <<= 1;
    } else {
        g.lpr = 32;
        int64_t need = cdiv(nvec, 32);
        g.tiles = (int)cdiv(need, 16);
        need = cdiv(nvec, 32 * (int64_t)g.tiles);
        g.nch = 16;
        for (int c : kNch) if (c >= need) { g.nch = c; break; }
    }
    g.util = (double)nvec / ((double)g.lpr * g.nch * g.tiles);
    return g;
}

bool v_ok(const SegArgs& a, int V) {
    if (a.hw && a.hC % V) return false;  // per-head weights: a vector chunk must stay inside one head
    const bool cols_ok = (a.ncols % V == 0) ||
                         (a.allow_pad_read && V >= 4 && a.ldx >= (int64_t)align_up(a.ncols, V));
    return cols_ok && a.ldx % V == 0 && aligned(a.X, 4 * V);
}

// widest vector whose lane utilisation is not worse than the next narrower one
Geometry choose(const SegArgs& a) {
    static const int forced = [] {
        const char* e = getenv("PYG_SEG_VEC");
        return e ? atoi(e) : 0;
    }();
    if (forced == 1 || forced == 2 || forced == 4 || forced == 8)
        if (v_ok(a, forced)) return geometry(a.ncols, forced);
    Geometry best = geometry(a.ncols, 1);
    for (int V : {2, 4, 8}) {
        if (!v_ok(a, V)) continue;
        Geometry g = geometry(a.ncols, V);
        // 256-bit loads only when they fill clearly more lanes: at equal utilisation V = 4 won
        // (GCN aggregation at F = 512 on 9 L2-resident passes: 13.0 ms with V = 4, NCH = 4 vs 20.8 ms
        // with V = 8, NCH = 2, whose SASS keeps the loaded rows in local memory; gpurun_out/r2h)
        // Rows of <= 64 floats are the exception: 8 lanes x 256 bits per row keep twice the rows per warp
        // in flight (point clouds F = 64: 0.072 -> 0.048 ms per step; F = 128 / 500 measured slower with
        // V = 8, 3.72 -> 4.77 / 0.064 -> 0.074 ms; gpurun_out/r3r)
        const bool narrow8 = V == 8 && a.ncols <= 64 && g.util >= best.util - 1e-9;
        if (V == 8 ? (g.util > best.util * 1.05 || narrow8)
                   : (g.util >= best.util - 1e-9 || (V <= 4 && g.util >= 0.75)))
            best = g;
    }
    // Few rows with narrow features (e.g. 10,000 rows x 16 columns): one group of LPR lanes per row
    // leaves most of the GPU idle (4 lanes per row at V = 4 -> 40k threads).  Narrow the vector
    // while that raises the thread count toward ~148 SMs x 1,024 threads (a row's positions stay
    // sequential; more lanes per row split its columns finer).
    const int64_t rows = a.row_order ? a.order_len : a.n_rows;
    const int64_t want = 148LL * 1024;
    while (best.V > 1 && rows * best.lpr * best.tiles < want) {
        const int V2 = best.V / 2;
        if (!v_ok(a, V2)) break;
        const Geometry g = geometry(a.ncols, V2);
        if (g.lpr * g.tiles <= best.lpr * best.tiles) break;  // no more lanes per row to gain
        best = g;
    }
    return best;
}

pyg_status_t launch(const SegArgs& a, int reduce, const Geometry& g, int mode, const seg::HeavyArgs& h, int ovk,
                    cudaStream_t s) {
    switch (g.V) {
        case 8: return seg::launch<8>(a, reduce, g.nch, g.lpr, g.tiles, mode, h, ovk, s);
        case 4: return seg::launch<4>(a, reduce, g.nch, g.lpr, g.tiles, mode, h, ovk, s);
        case 2: return seg::launch<2>(a, reduce, g.nch, g.lpr, g.tiles, mode, h, ovk, s);
        default: return seg::launch<1>(a, reduce, g.nch, g.lpr, g.tiles, mode, h, ovk, s);
    }
}

pyg_status_t segment_reduce_one(const SegArgs& a0, int reduce, const pyg_plan* plan, void* ws, size_t ws_bytes,
                                cudaStream_t s) {
    SegArgs a = a0;
    if (a.n_rows <= 0 || a.ncols <= 0) return PYG_OK;
    // MAX keeps 16-bit argmax positions per segment on the LDG kernel: segments come from plans,
    // whose rows above kHeavyThreshold are split
    if ((reduce == PYG_MAX) && (!plan || plan->heavy_threshold > 0xfffe))
        return fail(PYG_ERR_UNSUPPORTED, "internal: MAX segment-reduce needs a plan with split rows");
    if (plan && plan->row_order) {
        a.row_order = plan->row_order;
        a.order_len = plan->order_len;
        a.order_offset = plan->row_offset;
    }
    const Geometry g = choose(a);
    const int sv = g.V >= 4 ? 4 : g.V;  // store width
    const int ovk = (a.ldo % sv == 0) && aligned(a.out, 4 * sv);
    const bool split = plan && (plan->item_hi > plan->item_lo);
    if (a.heavy_threshold <= 0 || !split) a.heavy_threshold = INT64_MAX;

    seg::HeavyArgs h;
    Carver cv(ws, ws_bytes);
    unsigned long long* counter = cv.take<unsigned long long>(1);  // TMA dynamic task counter
    const bool extras = a.row_scale || a.blend || a.col_bias;
    if (extras && reduce != PYG_SUM) return fail(PYG_ERR_UNSUPPORTED, "internal: epilogue extras need SUM");
    // LDG / combine instantiation (weighted max has its own: the plain MAX one skips the multiply)
    const int red_k = extras ? kRedSumEpi : (reduce == PYG_MAX && a.w) ? kRedMaxW : reduce;
    const bool tma = ws && cv.ok() && tma_eligible(a, plan);
    // hub chunks through the TMA pipeline too (as partial tasks after the light tasks), unless
    // PYG_TMA_HUBS=0 keeps them on the LDG chunk kernel
    const bool tma_hubs = tma && split && knobs().tma_hubs != 0;
    // wide rows without split hubs (source-blocked passes): the row-staged bulk-copy kernel
    const bool bulk = !tma && ws && cv.ok() && bulk_eligible(a, plan, reduce);
    // light rows: TMA gather4 pipeline, the bulk-copy kernel or the LDG kernel
    if (tma && !tma_hubs) {
        PYG_TRY(segment_tma(a, reduce, plan, counter, nullptr, nullptr, 0, s));
    } else if (bulk) {
        const int ovk4 = (a.ldo % 4 == 0) && aligned(a.out, 16);
        PYG_TRY(segment_bulk(a, extras ? kRedSumEpi : (reduce == PYG_MAX && a.w) ? kRedMaxW : reduce, counter, ovk4, s));
    } else if (!tma) {
        PYG_TRY(launch(a, red_k, g, 0, h, ovk, s));
    }
    if (!split) return PYG_OK;

    // split hub rows: chunk partials, then the fp64 combine
    h.heavy_rows = plan->heavy_rows;
    h.item_ptr = plan->heavy_item_ptr;
    h.h_lo = plan->h_lo;
    h.h_hi = plan->h_hi;
    h.item_lo = plan->item_lo;
    h.n_items = plan->item_hi - plan->item_lo;
    h.row_offset = plan->row_offset;
    h.chunk = plan->chunk;
    h.ldp = (int64_t)align_up((size_t)a.ncols, 4);
    h.part = cv.take<float>((size_t)h.n_items * h.ldp);
    h.part_arg = reduce == PYG_MAX ? cv.take<int32_t>((size_t)h.n_items * h.ldp) : nullptr;
    if (!ws || !cv.ok())
        return fail(PYG_ERR_NO_MEMORY, "workspace too small for %lld split-row chunks (need %zu bytes)",
                    (long long)h.n_items, segment_ws_bytes(plan, a.ncols, reduce));
    if (tma_hubs) PYG_TRY(segment_tma(a, reduce, plan, counter, h.part, h.part_arg, h.ldp, s));
    else PYG_TRY(launch(a, red_k, g, 1, h, ovk, s));  // hub chunks on the LDG kernel (mode 1)
    // one CTA per split row, threads over columns (one warp for narrow rows)
    const int ct = (int)std::min<int64_t>(256, align_up((size_t)a.ncols, 32));
    dim3 grid((unsigned)(h.h_hi - h.h_lo), (unsigned)cdiv(a.ncols, ct));
    switch (red_k) {
        case PYG_SUM: combine_kernel<PYG_SUM><<<grid, ct, 0, s>>>(a, h); break;
        case kRedSumEpi: combine_kernel<kRedSumEpi><<<grid, ct, 0, s>>>(a, h); break;
        case PYG_MEAN: combine_kernel<PYG_MEAN><<<grid, ct, 0, s>>>(a, h); break;
        case kRedHeadW: combine_kernel<kRedHeadW><<<grid, ct, 0, s>>>(a, h); break;
        default: combine_kernel<PYG_MAX><<<grid, ct, 0, s>>>(a, h); break;
    }
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace

size_t segment_ws_bytes(const pyg_plan* plan, int64_t ncols, int reduce) {
    if (!plan) return 0;
    if (!plan->parts.empty()) {
        size_t b = 0;
        for (const auto& p : plan->parts) b = std::max(b, segment_ws_bytes(&p, ncols, reduce));
        return b;
    }
    size_t b = 256;  // TMA task counter
    const int64_t items = plan->item_hi - plan->item_lo;
    if (items <= 0) return b;
    const size_t ldp = align_up((size_t)ncols, 4);
    b += align_up((size_t)items * ldp * sizeof(float), 256);
    if (reduce == PYG_MAX) b += align_up((size_t)items * ldp * sizeof(int32_t), 256);
    return b;
}

// Source-blocked plans: one pass per block of source rows (sized so the block of X stays
// L2-resident), accumulating into `out` in block order (deterministic); the last pass applies
// the mean division with the total in-degree.
pyg_status_t segment_reduce(const SegArgs& a0, int reduce, const pyg_plan* plan, void* ws, size_t ws_bytes,
                            cudaStream_t s) {
    if (!plan || plan->parts.empty()) return segment_reduce_one(a0, reduce, plan, ws, ws_bytes, s);
    // a pass view (pyg_plan_passes) holds a consecutive range of the root's source blocks: the first
    // block of the root writes, later ones accumulate, the root's last one finalizes
    const size_t nb = plan->parts.size();
    const int64_t total = plan->n_passes > 0 ? plan->n_passes : (int64_t)nb;
    for (size_t b = 0; b < nb; ++b) {
        SegArgs a = a0;
        const pyg_plan& p = plan->parts[b];
        const int64_t gb = plan->pass_base + (int64_t)b;
        a.rowptr = p.rowptr;
        a.accum = gb > 0;
        a.finalize = (gb + 1 == total);
        a.deg_total = plan->deg;
        a.heavy_threshold = p.heavy_threshold;
        PYG_TRY(segment_reduce_one(a, reduce, &p, ws, ws_bytes, s));
    }
    return PYG_OK;
}

}  // namespace pyg
