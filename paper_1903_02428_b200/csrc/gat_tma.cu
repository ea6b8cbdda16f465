// gat_tma.cu -- GAT backward on the TMA gather4 pipeline (NEXT-1: GAT; "our own optimized
// sparse softmax kernels"; semantics S:421-429).  One streaming pass over the forward plan
// computes, per edge k = (j -> i) and head h,
//
//     d_alpha[k][h] = g_i . z_j |_h                                   (the SDDMM)
//     dlogit[k][h]  = alpha[k][h] (d_alpha[k][h] - t_i[h]) leaky_relu'(s_src[j][h] + s_dst[i][h])
//     grad_s_dst[i][h] = sum over i's in-edges of dlogit[k][h]
//
// with t_i[h] = sum_{k in seg(i)} alpha[k][h] d_alpha[k][h] = g_i . (sum_k alpha[k][h] z_j)|_h =
// g_i . out_i|_h taken from the FORWARD OUTPUT (gat_t_kernel), so the softmax backward needs no
// second pass over the row (the two-pass kernels in attention.cu need d_alpha of every position
// before any dlogit).
//
// Pipeline (same task / ring structure as seg_tma_kernel, segment_tma.cuh): per warp a ring of S
// stages, each holding 4 positions; lane 0 issues per stage
//   * one gather4 per column box of the 4 z_j rows (the dominant bytes),
//   * one gather4 of the 4 alpha rows (by edge id) and one of the 4 s_src rows (by source),
//   * for every slot that STARTS a row (target differs from the previous position of the stream):
//     bulk copies of g_i (F floats), t_i (H floats, parked in grad_s_dst by gat_t_kernel) and
//     s_dst[i] (H floats),
// all completing on the stage's mbarrier.  The consumer keeps g_i's float4 chunks in registers for
// the row, dots them with each slot's z_j chunks, reduces each head over its lanes (butterfly), and
// then 32 lanes = 4 slots x 8 heads finish the stage: dlogit (one 32-byte store per slot at H = 8),
// and the per-row head sums in position order (fp32; hub-row chunks write partials that
// gat_combine_kernel adds in fp64 in chunk order -- deterministic, reading Q12).
#include "segment_tma.cuh"

namespace pyg {
#ifndef PYG_GAT_STCS
#define PYG_GAT_STCS 1
#endif

namespace gat {

using tma::bar_expect;
using tma::bar_init;
using tma::bar_wait;
using tma::gather4;
using tma::lds128;
using tma::lds128f;
using tma::sts32;

__device__ __forceinline__ void bulk_copy(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ float lds32f(uint32_t addr) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr));
    return v;
}
__device__ __forceinline__ void sts32f(uint32_t addr, float v) {
    asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}

// predicated shared-memory loads: the destination keeps its value when p is false (no branch, so
// the shuffles around them need no divergence handling)
__device__ __forceinline__ void lds128f_if(bool p, float4& v, uint32_t addr) {
    asm volatile(
        "{\n .reg .pred q;\n setp.ne.u32 q, %5, 0;\n @q ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];\n}\n"
        : "+f"(v.x), "+f"(v.y), "+f"(v.z), "+f"(v.w)
        : "r"(addr), "r"((unsigned)p));
}
__device__ __forceinline__ void lds32f_if(bool p, float& v, uint32_t addr) {
    asm volatile("{\n .reg .pred q;\n setp.ne.u32 q, %2, 0;\n @q ld.shared.f32 %0, [%1];\n}\n"
                 : "+f"(v)
                 : "r"(addr), "r"((unsigned)p));
}

__device__ __forceinline__ int sel4(const int4& v, int i) { return i == 0 ? v.x : i == 1 ? v.y : i == 2 ? v.z : v.w; }

constexpr int kMeta = 64;  // per stage: int keys[4] | int rows[4] | int eids[4] | int cols[4]

struct BwdArgs {
    const int64_t* rowptr;   // ROOT rowptr
    const int32_t* pos_row;  // ROOT row of each position
    const int64_t* task_pos;
    const int32_t* task_item;
    int64_t n_tasks;
    unsigned long long* next;
    int64_t E_root;
    const int32_t* gidx;     // source j per position
    const int32_t* eid;      // edge id per position (null: identity)
    float* gsd;              // grad_s_dst [n x H]: t_i on entry, the row sums on exit
    float* dlogit;           // [E x H] packed, by edge id
    float* part;             // hub chunk partials [items x H]
    int64_t item_lo;
    int64_t row_lo, row_hi;  // this plan's root rows
    int F, H, C, box_w, nb;
    float slope;
    int warp_bytes, data_off;
    int zbytes, off_g, off_a, off_s, off_t, off_d, stage_bytes;
};

// The chunk visiting order of head h (C = 4 CPH columns = CPH float4 chunks): j-th chunk visited is
// (j + rot(h)) mod CPH.  rot spreads the 8 heads of a staged row over distinct 16-byte bank groups
// (a row's heads are CPH * 16 bytes apart), so the 8 lanes reading one row are conflict-free.  The
// SDDMM (gat_bwd_tma_kernel) and t_i (gat_t_row_head_kernel) both add the chunk dots sequentially in
// this order, each chunk as x0 y0 then fma of y, z, w: t_i of a row whose output equals one source
// row bitwise equals that edge's d_alpha bitwise.
template <int CPH>
__device__ __forceinline__ int head_rot(int h) { return CPH >= 8 ? h % CPH : h / (8 / CPH); }

template <int CPH>
__device__ __forceinline__ float head_dot(uint32_t zb, uint32_t gb, int rot) {
    float acc = 0.0f;
#pragma unroll
    for (int j = 0; j < CPH; ++j) {
        const uint32_t off = 16u * (uint32_t)((j + rot) % CPH);
        const float4 x = lds128f(gb + off);
        const float4 y = lds128f(zb + off);
        float q = x.x * y.x;
        q = fmaf(x.y, y.y, q);
        q = fmaf(x.z, y.z, q);
        q = fmaf(x.w, y.w, q);
        acc = j == 0 ? q : acc + q;
    }
    return acc;
}

// One pass per stage of 4 positions: lane (i, h) = (lane / 8, lane % 8) owns slot i, head h.  Lane 0
// gathers (TMA gather4, all completing on the stage's mbarrier): the 4 z_j rows and the 4 g_i rows
// (by target), and the 4 rows of alpha (by edge id), s_src (by source), t and s_dst (by target).
// Each lane then needs no shuffles for its d_alpha and dlogit; the per-row head sums are a 4-step
// segmented scan over the slots.
template <int CPH, int NB, int S>
__global__ void __launch_bounds__(256, 2) gat_bwd_tma_kernel(const __grid_constant__ CUtensorMap tz,
                                                             const __grid_constant__ CUtensorMap tg,
                                                             const __grid_constant__ CUtensorMap ta,
                                                             const __grid_constant__ CUtensorMap ts,
                                                             const __grid_constant__ CUtensorMap tt,
                                                             const __grid_constant__ CUtensorMap td, BwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t region = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(warp * a.warp_bytes);
    const uint32_t bar0 = region;
    const uint32_t meta0 = region + 128;
    const uint32_t data0 = region + (uint32_t)a.data_off;
    const int H = a.H;
    const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
    const uint32_t row_bytes = (uint32_t)(4 * a.box_w);

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    const int my_i = lane >> 3, my_h = lane & 7;
    const bool hv = my_h < H;
    // this lane's head inside a staged row: column my_h * C lives in box (my_h * C) / box_w
    const int hc0 = hv ? my_h * a.C : 0;
    const uint32_t hoff = (uint32_t)(4 * ((hc0 / a.box_w) * 4 * a.box_w + hc0 % a.box_w)) + (uint32_t)my_i * row_bytes;
    const int rot = head_rot<CPH>(my_h);
    const int64_t plo = __ldg(a.rowptr + a.row_lo), phi = __ldg(a.rowptr + a.row_hi);

    // ---------------- producer (warp-uniform) ----------------
    int64_t pp = 0, pe = 0, iwb = 0, nwb = -1, task = 0;
    bool done = false;
    int wg = 0, wr = 0, we = 0, ng = 0, nr = 0, ne = 0;
    int citem = -1;
    auto load_window = [&](int64_t base, int& gg, int& rr, int& ee) {
        const int64_t p = base + lane;
        gg = 0; rr = -1; ee = 0;
        if (p < a.E_root) {
            gg = __ldg(a.gidx + p);
            rr = __ldg(a.pos_row + p);
            ee = a.eid ? __ldg(a.eid + p) : (int)p;
        }
    };
    auto set_window = [&](int64_t base) {
        if (base == nwb) {
            wg = ng; wr = nr; we = ne;
        } else {
            load_window(base, wg, wr, we);
        }
        iwb = base;
        nwb = base + 32;
        load_window(nwb, ng, nr, ne);
    };
    auto next_task = [&]() -> bool {
        for (;;) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(a.next, 1ull);
            task = (int64_t)__shfl_sync(0xffffffffu, t, 0);
            if (task >= a.n_tasks) return false;
            const int64_t t0 = max(__ldg(a.task_pos + 2 * task), plo);
            const int64_t t1 = min(__ldg(a.task_pos + 2 * task + 1), phi);
            const int it = a.task_item ? __ldg(a.task_item + task) : -1;
            if (t0 < t1) {
                pp = t0;
                pe = t1;
                citem = it;
                return true;
            }
        }
    };
    if (next_task()) set_window(pp); else done = true;

    auto fill = [&](int s) {
        const uint32_t m = meta0 + (uint32_t)(s * kMeta) + 4u * (uint32_t)lane;
        if (done) {
            if (lane < 4) sts32(m, -1);
            return;
        }
        if (pp - iwb >= 32) set_window(pp);
        const int j = (int)(pp - iwb);
        const int cnt = (int)min((int64_t)4, pe - pp);
        const int src = j + (lane & 3);
        const int gj = __shfl_sync(0xffffffffu, wg, src);
        const int row = __shfl_sync(0xffffffffu, wr, src);
        const int e = __shfl_sync(0xffffffffu, we, src);
        if (lane < 4) {
            sts32(m, lane < cnt ? (citem >= 0 ? -(citem + 2) : row) : -1);
            sts32(m + 16, row);
            sts32(m + 32, e);
            sts32(m + 48, gj);
        }
        __syncwarp();
        if (lane == 0) {  // the stage's slots back from shared memory (missing slots repeat slot 0)
            const uint32_t ms = meta0 + (uint32_t)(s * kMeta);
            const int4 r4 = lds128(ms + 16), e4 = lds128(ms + 32), g4 = lds128(ms + 48);
            const int lo = (int)a.row_lo;
            const int r0 = r4.x - lo, r1 = (cnt > 1 ? r4.y : r4.x) - lo, r2 = (cnt > 2 ? r4.z : r4.x) - lo,
                      r3 = (cnt > 3 ? r4.w : r4.x) - lo;
            const int gs1 = cnt > 1 ? g4.y : g4.x, gs2 = cnt > 2 ? g4.z : g4.x, gs3 = cnt > 3 ? g4.w : g4.x;
            const int es1 = cnt > 1 ? e4.y : e4.x, es2 = cnt > 2 ? e4.z : e4.x, es3 = cnt > 3 ? e4.w : e4.x;
            const uint32_t bar = bar0 + 8 * s;
            const uint32_t st = data0 + (uint32_t)s * stage_bytes;
            bar_expect(bar, 2u * (uint32_t)a.zbytes + 64u * (uint32_t)H);
#pragma unroll
            for (int b = 0; b < NB; ++b) {
                gather4(st + (uint32_t)b * 4u * row_bytes, &tz, b * a.box_w, g4.x, gs1, gs2, gs3, bar);
                gather4(st + (uint32_t)a.off_g + (uint32_t)b * 4u * row_bytes, &tg, b * a.box_w, r0, r1, r2, r3, bar);
            }
            gather4(st + (uint32_t)a.off_a, &ta, 0, e4.x, es1, es2, es3, bar);
            gather4(st + (uint32_t)a.off_s, &ts, 0, g4.x, gs1, gs2, gs3, bar);
            gather4(st + (uint32_t)a.off_t, &tt, 0, r0, r1, r2, r3, bar);
            gather4(st + (uint32_t)a.off_d, &td, 0, r0, r1, r2, r3, bar);
        }
        pp += cnt;
        if (pp >= pe) {
            if (next_task()) {
                if (pp != iwb + 32 && (pp < iwb || pp - iwb >= 32 || ((pp - iwb) & 3))) set_window(pp);
            } else {
                done = true;
            }
        }
    };

    // ---------------- consumer ----------------
    int gkey = -1;            // key of the row whose head sums are being accumulated
    float* gdst = nullptr;    // where they go (grad_s_dst row, or a hub chunk's partial)
    float gs = 0.0f;          // lanes < H: running head sum of dlogit

#pragma unroll 1
    for (int s = 0; s < S; ++s) fill(s);
    __syncwarp();
    uint32_t phase = 0;
#pragma unroll 1
    for (int s = 0;; s = (s + 1 == S) ? 0 : s + 1) {
        const uint32_t m = meta0 + (uint32_t)(s * kMeta);
        const int4 keys = lds128(m);
        const int c = (keys.x != -1) + (keys.y != -1) + (keys.z != -1) + (keys.w != -1);
        if (c == 0) break;
        const int4 rows = lds128(m + 16);
        const int4 eids = lds128(m + 32);
        bar_wait(bar0 + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
        const uint32_t st = data0 + (uint32_t)s * stage_bytes;
        // (slot my_i, head my_h): d_alpha, then dlogit
        const bool mine = my_i < c && hv;
        float dl = 0.0f;
        if (mine) {
            const float d = head_dot<CPH>(st + hoff, st + (uint32_t)a.off_g + hoff, rot);
            const uint32_t q = 4u * (uint32_t)(my_i * H + my_h);
            const float al = lds32f(st + (uint32_t)a.off_a + q);
            const float ss = lds32f(st + (uint32_t)a.off_s + q);
            const float t = lds32f(st + (uint32_t)a.off_t + q);
            const float sd = lds32f(st + (uint32_t)a.off_d + q);
            dl = al * (d - t);
            if (!(ss + sd > 0.0f)) dl *= a.slope;
            const int e = my_i == 0 ? eids.x : my_i == 1 ? eids.y : my_i == 2 ? eids.z : eids.w;
            a.dlogit[(int64_t)e * H + my_h] = dl;
        }
        // head sums per row, in position order (lanes < H hold head `lane`): the four slot values first
        // (shuffles outside any branch), then the rare row changes store through a pointer kept per row
        const int kk[4] = {keys.x, keys.y, keys.z, keys.w};
        const int rr[4] = {rows.x, rows.y, rows.z, rows.w};
        float vs[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) vs[i] = __shfl_sync(0xffffffffu, dl, i * 8 + my_h);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i < c && kk[i] != gkey) {
                if (gdst && lane < H) gdst[lane] = gs;
                gkey = kk[i];
                gdst = kk[i] < -1 ? a.part + ((int64_t)(-kk[i] - 2) - a.item_lo) * H
                                  : a.gsd + ((int64_t)rr[i] - a.row_lo) * H;
                gs = 0.0f;
            }
            gs = i < c ? gs + vs[i] : gs;
        }
        __syncwarp();  // every lane is done with stage s before it is refilled
        fill(s);
    }
    if (gdst && lane < H) gdst[lane] = gs;
}

// t_i[h] = g_i . out_i |_h (0 for rows without in-edges), written into grad_s_dst (the backward
// kernel reads it per slot, then overwrites the row with its head sums).  A thread per (row, head),
// the chunks in head_dot's order (rotation, product order, sequential sum), so a row whose forward
// output equals one source row bitwise (one in-edge, alpha = 1) gets t_i equal to that edge's
// d_alpha bitwise; every thread keeps 2 CPH vector loads in flight.
template <int CPH>
__global__ void gat_t_row_head_kernel(const float* __restrict__ g, int64_t ldg, const float* __restrict__ out,
                                      int64_t ldo, const int64_t* __restrict__ rowptr, int64_t n, int H, float* gsd,
                                      const float* __restrict__ rs, float* gsc) {
    const int64_t total = n * H;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t r = t / H;
        const int h = (int)(t - r * H);
        float v = 0.0f;
        if (__ldg(rowptr + r + 1) > __ldg(rowptr + r)) {
            const float4* gr = reinterpret_cast<const float4*>(g + r * ldg) + h * CPH;
            const float4* orr = reinterpret_cast<const float4*>(out + r * ldo) + h * CPH;
            const int rot = head_rot<CPH>(h);
            // factored alpha: this head's grad_out / row sum for the alpha-weighted grad_z
            const float inv = gsc ? 1.0f / __ldg(rs + t) : 0.0f;
            float4* gs = gsc ? reinterpret_cast<float4*>(gsc + r * (int64_t)H * 4 * CPH) + h * CPH : nullptr;
#pragma unroll
            for (int j = 0; j < CPH; ++j) {
                const int k = (j + rot) % CPH;
                float4 x = __ldg(gr + k);
                const float4 y = __ldg(orr + k);
                if (gs) {  // factored alpha: t and the SDDMM both use g / row_sum (see gat_bwd_tma)
                    x = make_float4(x.x * inv, x.y * inv, x.z * inv, x.w * inv);
                    gs[k] = x;
                }
                float q = x.x * y.x;
                q = fmaf(x.y, y.y, q);
                q = fmaf(x.z, y.z, q);
                q = fmaf(x.w, y.w, q);
                v = j == 0 ? q : v + q;
            }
        }
        gsd[t] = v;
    }
}

// grad_s_dst of a split hub row = its chunk partials added in fp64 in chunk order
__global__ void gat_combine_kernel(const int32_t* heavy_rows, const int64_t* item_ptr, int64_t h_lo, int64_t h_hi,
                                   int64_t item_lo, int64_t row_offset, const float* part, int H, float* gsd) {
    const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t hr = h_lo + t / H;
    const int h = (int)(t % H);
    if (hr >= h_hi) return;
    double s = 0.0;
    for (int64_t it = item_ptr[hr]; it < item_ptr[hr + 1]; ++it) s += (double)part[(it - item_lo) * H + h];
    gsd[((int64_t)heavy_rows[hr] - row_offset) * H + h] = (float)s;
}

template <int CPH, int NB>
pyg_status_t launch(int S, int64_t want, int warps, int smem, cudaStream_t s, const CUtensorMap (&tm)[6],
                    const BwdArgs& a) {
    void (*k)(const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap, const CUtensorMap,
              const CUtensorMap, BwdArgs) =
        S >= 3 ? gat_bwd_tma_kernel<CPH, NB, 3> : gat_bwd_tma_kernel<CPH, NB, 2>;
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int kSmemPerSm = std::min(227, std::max(32, knobs().gat_sm_kb)) * 1024;
    int dev = 0, sms = 148, per_sm = 1;
    PYG_CUDA(cudaGetDevice(&dev));
    PYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int cap = std::max(1, kSmemPerSm / (smem + 1024));
    const int carve = std::min(100, (int)cdiv((int64_t)cap * (smem + 1024) * 100, 228 * 1024));
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    PYG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * warps, smem));
    per_sm = std::min(per_sm, cap);
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1))));
    k<<<grid, 32 * warps, smem, s>>>(tm[0], tm[1], tm[2], tm[3], tm[4], tm[5], a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

bool encode_rows(CUtensorMap* tm, const float* base, int64_t cols, int64_t rows, int64_t ld, int box_w) {
    cuuint64_t gdim[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t gstr[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {(cuuint32_t)box_w, 1};
    cuuint32_t es[2] = {1, 1};
    return tma::encode_fn()(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), gdim, gstr, box, es,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

bool al16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }


// ============================================================================================
// Forward: softmax + alpha-weighted aggregation in ONE streaming pass.
//
// Softmax is shift-invariant: alpha[k][h] = exp(l_k - c_i) / sum_{k' in seg(i)} exp(l_k' - c_i) for
// ANY per-row shift c_i.  The usual c_i = max_k l_k needs a pass over the row before the first
// weight.  Because leaky_relu is monotone, c_i[h] = leaky_relu(S_h + s_dst[i][h]) with S_h = max_j
// s_src[j][h] (one tiny reduction over s_src) bounds every logit of row i from above (in fp32 too:
// rounding is monotone), so every weight p = exp(l - c_i) lies in (0, 1] -- no overflow -- and the
// row is aggregated as out_i = (sum p z_j) / (sum p) in the same pass that gathers z_j.  The
// weights p are stored by edge id and divided by the row sum afterwards (gat_alpha_norm_kernel).
// If a row's sum underflows (its logits all sit ~80 below the global bound -- far outside GAT's
// range), the row is listed and recomputed exactly with its own max (gat_fwd_fix_kernel).
// ============================================================================================

struct FwdArgs {
    const int64_t* rowptr;   // ROOT rowptr
    const int32_t* pos_row;
    const int64_t* task_pos;
    const int32_t* task_item;
    int64_t n_tasks;
    unsigned long long* next;
    int64_t E_root;
    const int32_t* gidx;
    const int32_t* eid;
    const float* s_dst;      // [n x H]
    const unsigned* smax;    // [H] ordered-int max of s_src per head
    float* alpha;            // [E x H]: the weights p on exit (normalised later)
    float* out;
    int64_t ldo;
    float* rs;               // [n x H] row sums of p
    float* part;             // hub chunk partial sums of p z [items x ldp]
    float* part_s;           // hub chunk partial sums of p [items x H]
    int64_t ldp, item_lo;
    int* bad;                // [0]: count, [1..]: local rows whose sum underflowed
    int64_t row_lo, row_hi;
    int F, H, C, box_w, nb;
    float slope;
    int warp_bytes, data_off;
    int zbytes, off_s, off_d, stage_bytes;
};

constexpr float kTinySum = 1e-30f;  // a row sum below this is recomputed with the row's own max

template <int NCH, int S>
__global__ void __launch_bounds__(256, 1) gat_fwd_tma_kernel(const __grid_constant__ CUtensorMap tz,
                                                             const __grid_constant__ CUtensorMap ts,
                                                             const __grid_constant__ CUtensorMap td, FwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t region = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(warp * a.warp_bytes);
    const uint32_t bar0 = region;
    const uint32_t meta0 = region + 128;
    const uint32_t scr = meta0 + (uint32_t)(S * kMeta);  // 4 slots x 8 heads of p (128 B)
    const uint32_t data0 = region + (uint32_t)a.data_off;
    const int H = a.H, F = a.F;
    const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
    const uint32_t row_bytes = (uint32_t)(4 * a.box_w);
    const float slope = a.slope;

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    uint32_t coff[NCH];
    int hch[NCH];
    bool cval[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int c = 4 * (lane + 32 * ch);
        const int b = c / a.box_w, cc = c - b * a.box_w;
        cval[ch] = c < F;
        coff[ch] = cval[ch] ? (uint32_t)(4 * (b * 4 * a.box_w + cc)) : 0u;
        hch[ch] = cval[ch] ? c / a.C : 0;
    }
    const float smx = (lane & 7) < H ? ord2f(__ldg(a.smax + (lane & 7))) : 0.0f;  // the max s_src of lane's head
    const int64_t plo = __ldg(a.rowptr + a.row_lo), phi = __ldg(a.rowptr + a.row_hi);

    // ---------------- producer (as gat_bwd_tma_kernel: z rows, s_src rows, s_dst of new rows) -----
    int64_t pp = 0, pe = 0, iwb = 0, nwb = -1, task = 0;
    bool done = false;
    int wg = 0, wr = 0, we = 0, ng = 0, nr = 0, ne = 0;
    int citem = -1;
    auto load_window = [&](int64_t base, int& gg, int& rr, int& ee) {
        const int64_t p = base + lane;
        gg = 0; rr = -1; ee = 0;
        if (p < a.E_root) {
            gg = __ldg(a.gidx + p);
            rr = __ldg(a.pos_row + p);
            ee = a.eid ? __ldg(a.eid + p) : (int)p;
        }
    };
    auto set_window = [&](int64_t base) {
        if (base == nwb) {
            wg = ng; wr = nr; we = ne;
        } else {
            load_window(base, wg, wr, we);
        }
        iwb = base;
        nwb = base + 32;
        load_window(nwb, ng, nr, ne);
    };
    auto next_task = [&]() -> bool {
        for (;;) {
            unsigned long long t = 0;
            if (lane == 0) t = atomicAdd(a.next, 1ull);
            task = (int64_t)__shfl_sync(0xffffffffu, t, 0);
            if (task >= a.n_tasks) return false;
            const int64_t t0 = max(__ldg(a.task_pos + 2 * task), plo);
            const int64_t t1 = min(__ldg(a.task_pos + 2 * task + 1), phi);
            const int it = a.task_item ? __ldg(a.task_item + task) : -1;
            if (t0 < t1) {
                pp = t0;
                pe = t1;
                citem = it;
                return true;
            }
        }
    };
    if (next_task()) set_window(pp); else done = true;

    auto fill = [&](int s) {
        const uint32_t m = meta0 + (uint32_t)(s * kMeta) + 4u * (uint32_t)lane;
        if (done) {
            if (lane < 4) sts32(m, -1);
            return;
        }
        if (pp - iwb >= 32) set_window(pp);
        const int j = (int)(pp - iwb);
        const int cnt = (int)min((int64_t)4, pe - pp);
        const int src = j + (lane & 3);
        const int gj = __shfl_sync(0xffffffffu, wg, src);
        const int row = __shfl_sync(0xffffffffu, wr, src);
        const int e = __shfl_sync(0xffffffffu, we, src);
        if (lane < 4) {
            sts32(m, lane < cnt ? (citem >= 0 ? -(citem + 2) : row) : -1);
            sts32(m + 16, row);
            sts32(m + 32, e);
            sts32(m + 48, gj);
        }
        __syncwarp();
        if (lane == 0) {  // z_j and s_src rows by source, s_dst rows by target (missing slots repeat slot 0)
            const uint32_t ms = meta0 + (uint32_t)(s * kMeta);
            const int4 r4 = lds128(ms + 16), g4 = lds128(ms + 48);
            const int gs1 = cnt > 1 ? g4.y : g4.x, gs2 = cnt > 2 ? g4.z : g4.x, gs3 = cnt > 3 ? g4.w : g4.x;
            const int lo = (int)a.row_lo;
            const int r0 = r4.x - lo, r1 = (cnt > 1 ? r4.y : r4.x) - lo, r2 = (cnt > 2 ? r4.z : r4.x) - lo,
                      r3 = (cnt > 3 ? r4.w : r4.x) - lo;
            const uint32_t bar = bar0 + 8 * s;
            const uint32_t st = data0 + (uint32_t)s * stage_bytes;
            bar_expect(bar, (uint32_t)a.zbytes + 32u * (uint32_t)H);
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (b < a.nb) gather4(st + (uint32_t)b * 4u * row_bytes, &tz, b * a.box_w, g4.x, gs1, gs2, gs3, bar);
            gather4(st + (uint32_t)a.off_s, &ts, 0, g4.x, gs1, gs2, gs3, bar);
            gather4(st + (uint32_t)a.off_d, &td, 0, r0, r1, r2, r3, bar);
        }
        pp += cnt;
        if (pp >= pe) {
            if (next_task()) {
                if (pp != iwb + 32 && (pp < iwb || pp - iwb >= 32 || ((pp - iwb) & 3))) set_window(pp);
            } else {
                done = true;
            }
        }
    };

    // ---------------- consumer ----------------
    int arow = -1, agrow = 0;         // key / root row being aggregated
    float acc[NCH][4];
    float ssum[NCH];                  // running sum of p of each chunk's head (replicated per lane)
    const int my_i = lane >> 3, my_h = lane & 7;
    const int CLh = a.C >= 128 ? 32 : a.C / 4;
    const bool leader = (lane % CLh) == 0;  // writes its chunk's head sum
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        ssum[ch] = 0.0f;
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[ch][q] = 0.0f;
    }
    auto flush = [&]() {  // no warp-synchronous operations: called under a (uniform) branch
        if (arow < -1) {  // hub chunk: raw partials for gat_fwd_combine_kernel
            const int64_t it = (int64_t)(-arow - 2) - a.item_lo;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
                if (cval[ch]) {
                    *reinterpret_cast<float4*>(a.part + it * a.ldp + 4 * (lane + 32 * ch)) =
                        make_float4(acc[ch][0], acc[ch][1], acc[ch][2], acc[ch][3]);
                    if (leader) a.part_s[it * H + hch[ch]] = ssum[ch];
                }
            return;
        }
        const int64_t r = (int64_t)agrow - a.row_lo;
        bool tiny = false;
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
            if (cval[ch]) {
                const float sh = ssum[ch];
                const float inv = 1.0f / sh;  // one IEEE division per chunk (a division per element spilled
                                              // the registers around its slow-path calls)
                *reinterpret_cast<float4*>(a.out + r * a.ldo + 4 * (lane + 32 * ch)) =
                    make_float4(acc[ch][0] * inv, acc[ch][1] * inv, acc[ch][2] * inv, acc[ch][3] * inv);
                if (leader) a.rs[r * H + hch[ch]] = sh;
                tiny |= !(sh >= kTinySum);
            }
        // a row whose sum underflowed in any head is listed once (flush runs warp-uniformly)
        if (__ballot_sync(0xffffffffu, tiny) && lane == 0) a.bad[1 + atomicAdd(a.bad, 1)] = (int)r;
    };

#pragma unroll 1
    for (int s = 0; s < S; ++s) fill(s);
    __syncwarp();
    uint32_t phase = 0;
#pragma unroll 1
    for (int s = 0;; s = (s + 1 == S) ? 0 : s + 1) {
        const uint32_t m = meta0 + (uint32_t)(s * kMeta);
        const int4 keys = lds128(m);
        const int c = (keys.x != -1) + (keys.y != -1) + (keys.z != -1) + (keys.w != -1);
        if (c == 0) break;
        const int4 rows = lds128(m + 16);
        const int4 eids = lds128(m + 32);
        bar_wait(bar0 + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
        const uint32_t st = data0 + (uint32_t)s * stage_bytes;
        const int kk[4] = {keys.x, keys.y, keys.z, keys.w};
        // the weight of (slot my_i, head my_h), from its staged s_src and s_dst: one exp per lane per stage
        const bool mine = my_i < c && my_h < H;
        float ss = 0.0f, sme = 0.0f;
        lds32f_if(mine, ss, st + (uint32_t)a.off_s + 4u * (uint32_t)(my_i * H + my_h));
        lds32f_if(mine, sme, st + (uint32_t)a.off_d + 4u * (uint32_t)(my_i * H + my_h));
        const float pre = ss + sme, cpre = smx + sme;
        const float l = pre > 0.0f ? pre : slope * pre;
        const float cs = cpre > 0.0f ? cpre : slope * cpre;  // the row's shift c_i (>= every logit)
        const float p = mine ? expf(l - cs) : 0.0f;
        const int e = my_i == 0 ? eids.x : my_i == 1 ? eids.y : my_i == 2 ? eids.z : eids.w;
#if PYG_GAT_STCS
        if (mine) __stcs(a.alpha + (int64_t)e * H + my_h, p);  // streamed past L2 (z rows of hubs stay)
#else
        if (mine) a.alpha[(int64_t)e * H + my_h] = p;
#endif
        sts32f(scr + 4u * (uint32_t)lane, p);
        __syncwarp();
        // (3) aggregation in position order (unrolled: a rolled loop with one flush path measured slower,
        // 22.8 vs 21.4 ms on R-MAT, gpurun_out/r2y)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i >= c) break;
            const int ki = kk[i];
            if (ki != arow) {
                if (arow != -1) flush();
                arow = ki;
                agrow = sel4(rows, i);
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch) {
                    ssum[ch] = 0.0f;
#pragma unroll
                    for (int q = 0; q < 4; ++q) acc[ch][q] = 0.0f;
                }
            }
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const float w = lds32f(scr + 4u * (uint32_t)(i * 8 + hch[ch]));
                float4 zv = make_float4(0.f, 0.f, 0.f, 0.f);
                lds128f_if(cval[ch], zv, st + coff[ch] + (uint32_t)i * row_bytes);
                acc[ch][0] = fmaf(w, zv.x, acc[ch][0]);
                acc[ch][1] = fmaf(w, zv.y, acc[ch][1]);
                acc[ch][2] = fmaf(w, zv.z, acc[ch][2]);
                acc[ch][3] = fmaf(w, zv.w, acc[ch][3]);
                ssum[ch] += w;
            }
        }
        __syncwarp();
        fill(s);
    }
    if (arow != -1) flush();
}

__global__ void gat_smax_kernel(const float* __restrict__ s_src, int64_t total, int H, unsigned* smax) {
    // stride is a multiple of 32, so each thread always reads the same head (tid % H)
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    float m = -INFINITY;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) m = fmaxf(m, __ldg(s_src + i));
    for (int o = 16; o >= H; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if ((threadIdx.x & 31) < H) atomicMax(smax + (threadIdx.x & 31), f2ord(m));
}

// a split hub row: out = (sum of chunk partials of p z) / (sum of chunk partials of p), fp64 in chunk order
__global__ void gat_fwd_combine_kernel(const int32_t* heavy_rows, const int64_t* item_ptr, int64_t h_lo,
                                       int64_t item_lo, int64_t row_offset, const float* part, int64_t ldp,
                                       const float* part_s, int H, int C, int F, float* out, int64_t ldo, float* rs,
                                       int* bad) {
    const int64_t hr = h_lo + blockIdx.x;
    const int64_t r = (int64_t)heavy_rows[hr] - row_offset;
    const int64_t i0 = item_ptr[hr] - item_lo, i1 = item_ptr[hr + 1] - item_lo;
    __shared__ double sh[8];
    __shared__ int tiny;
    if (threadIdx.x == 0) tiny = 0;
    __syncthreads();
    if (threadIdx.x < H) {
        double t = 0.0;
        for (int64_t it = i0; it < i1; ++it) t += (double)part_s[it * H + threadIdx.x];
        sh[threadIdx.x] = t;
        rs[r * H + threadIdx.x] = (float)t;
        if (!(t >= (double)kTinySum)) tiny = 1;
    }
    __syncthreads();
    for (int c = threadIdx.x; c < F; c += blockDim.x) {
        double t = 0.0;
        for (int64_t it = i0; it < i1; ++it) t += (double)part[it * ldp + c];
        out[r * ldo + c] = (float)(t / sh[c / C]);
    }
    if (threadIdx.x == 0 && tiny) bad[1 + atomicAdd(bad, 1)] = (int)r;
}

// alpha[k][h] = p[k][h] / rs[row(k)][h] over this plan's positions (thread per (position, head))
__global__ void gat_alpha_norm_kernel(const int32_t* __restrict__ pos_row, const int32_t* __restrict__ eid,
                                      const int64_t* __restrict__ rowptr, int64_t n, int64_t row_lo, int H,
                                      const float* __restrict__ rs, float* alpha) {
    const int64_t plo = rowptr[0], phi = rowptr[n];  // this plan's positions (slices: a sub-range)
    const int64_t total = (phi - plo) * H;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t p = plo + t / H;
        const int h = (int)(t % H);
        const int64_t k = eid ? (int64_t)__ldg(eid + p) : p;
        const int64_t r = (int64_t)__ldg(pos_row + p) - row_lo;
        alpha[k * H + h] = alpha[k * H + h] / __ldg(rs + r * H + h);
    }
}

// rows without in-edges: out = 0 (the plan's empty-row list)
__global__ void gat_empty_rows_kernel(const int32_t* __restrict__ order, int64_t begin, int64_t end, int64_t row_lo,
                                      int64_t row_hi, int F, float* out, int64_t ldo) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t k = begin + (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); k < end; k += warps) {
        const int64_t r = (int64_t)order[k];
        if (r < row_lo || r >= row_hi) continue;
        for (int c = lane; c < F; c += 32) out[(r - row_lo) * ldo + c] = 0.0f;
    }
}

// the listed rows (sum underflow), exactly: the row's own max, then exp / sum, then the
// alpha-weighted sum (warp per row; a fallback far outside GAT's logit range, kept simple)
__global__ void gat_fwd_fix_kernel(const int* __restrict__ bad, const int64_t* __restrict__ rowptr,
                                   const int32_t* __restrict__ col, const int32_t* __restrict__ eid,
                                   const float* __restrict__ z, int64_t ldz, const float* __restrict__ s_src,
                                   const float* __restrict__ s_dst, int H, int C, int F, float slope, float* alpha,
                                   float* out, int64_t ldo, float* row_sums) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int count = bad[0];
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count; w += warps) {
        const int64_t r = bad[1 + w];
        const int64_t b = rowptr[r], e = rowptr[r + 1];
        for (int h = 0; h < H; ++h) {
            const float sd = s_dst[r * H + h];
            float m = -INFINITY;
            for (int64_t p = b + lane; p < e; p += 32) {
                const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                m = fmaxf(m, pre > 0.0f ? pre : slope * pre);
            }
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            float sum = 0.0f;
            for (int64_t p = b + lane; p < e; p += 32) {
                const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                sum += expf((pre > 0.0f ? pre : slope * pre) - m);
            }
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            for (int64_t p = b + lane; p < e; p += 32) {
                const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                const int64_t k = eid ? (int64_t)eid[p] : p;
                alpha[k * H + h] = expf((pre > 0.0f ? pre : slope * pre) - m) / sum;
            }
            if (row_sums && lane == 0) row_sums[r * H + h] = 1.0f;  // this row's alpha is normalised
        }
        __syncwarp();
        for (int c = lane; c < F; c += 32) {
            float acc = 0.0f;
            for (int64_t p = b; p < e; ++p) {
                const int64_t k = eid ? (int64_t)eid[p] : p;
                acc = fmaf(alpha[k * H + c / C], z[(int64_t)col[p] * ldz + c], acc);
            }
            out[r * ldo + c] = acc;
        }
    }
}

template <int NCH>
pyg_status_t launch_fwd(int S, int64_t want, int warps, int smem, int sm_kb, cudaStream_t s, const CUtensorMap& tz,
                        const CUtensorMap& tsrc, const CUtensorMap& tdst, const FwdArgs& a) {
    void (*k)(const CUtensorMap, const CUtensorMap, const CUtensorMap, FwdArgs) =
        S >= 3 ? gat_fwd_tma_kernel<NCH, 3> : gat_fwd_tma_kernel<NCH, 2>;
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const int kSmemPerSm = std::min(227, std::max(32, sm_kb)) * 1024;
    int dev = 0, sms = 148, per_sm = 1;
    PYG_CUDA(cudaGetDevice(&dev));
    PYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    const int cap = std::max(1, kSmemPerSm / (smem + 1024));
    const int carve = std::min(100, (int)cdiv((int64_t)cap * (smem + 1024) * 100, 228 * 1024));
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    PYG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k, 32 * warps, smem));
    per_sm = std::min(per_sm, cap);
    const dim3 grid((unsigned)std::max<int64_t>(1, std::min<int64_t>(want, (int64_t)sms * std::max(per_sm, 1))));
    k<<<grid, 32 * warps, smem, s>>>(tz, tsrc, tdst, a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace gat

size_t gat_bwd_tma_ws_bytes(const pyg_plan* plan, int64_t H) {
    if (!plan) return 0;
    return 256 + align_up((size_t)std::max<int64_t>(0, plan->item_hi - plan->item_lo) * (size_t)H * 4, 256);
}

bool gat_bwd_tma_eligible(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t ldz, const float* g,
                          int64_t ldg, const float* out, int64_t ldo, const float* alpha, const float* s_src,
                          const float* s_dst, const float* gsd) {
    using namespace gat;
    const int mode = knobs().seg_tma;
    if (mode == 0 || !out || !plan || !plan->parts.empty() || plan->n_tasks <= 0 || !plan->task_pos || !plan->pos_row)
        return false;
    if (!(H == 4 || H == 8) || F % 4 || F > 1024 || F < 16) return false;
    const bool pow2 = C > 0 && (C & (C - 1)) == 0;
    if (!(pow2 && C >= 4 && C <= 128)) return false;  // a head = 1..32 float4 chunks of one staged row
    if (mode != 1 && plan->n_light_tasks < 1024) return false;
    if (!al16(z) || ldz % 4 || !al16(g) || ldg % 4 || !al16(out) || ldo % 4) return false;
    if (!al16(alpha) || !al16(s_src) || !al16(s_dst) || !al16(gsd)) return false;
    return tma::encode_fn() != nullptr;
}

pyg_status_t gat_bwd_tma(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                         const float* g, int64_t ldg, const float* out, int64_t ldo, const float* alpha,
                         const float* row_sums, const float* s_src, const float* s_dst, float slope, float* dlogit,
                         float* gsd, float* gsc, void* ws, size_t ws_bytes, cudaStream_t s) {
    using namespace gat;
    const int64_t n = plan->n_rows;
    Carver cv(ws, ws_bytes);
    unsigned long long* counter = cv.take<unsigned long long>(1);
    const int64_t items = plan->item_hi - plan->item_lo;
    float* part = cv.take<float>((size_t)std::max<int64_t>(items, 0) * H);
    if (!ws || !cv.ok()) return fail(PYG_ERR_NO_MEMORY, "gat_backward: workspace too small (pyg_gat_backward_workspace_size)");
    PYG_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    // t_i = g_i . out_i per head, parked in grad_s_dst (0 for rows without in-edges)
    {
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n * H, 256), 148 * 16));
        switch (C / 4) {
            case 1: gat_t_row_head_kernel<1><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
            case 2: gat_t_row_head_kernel<2><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
            case 4: gat_t_row_head_kernel<4><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
            case 8: gat_t_row_head_kernel<8><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
            case 16: gat_t_row_head_kernel<16><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
            default: gat_t_row_head_kernel<32><<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, H, gsd, row_sums, gsc); break;
        }
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    const int nb = (F + 255) / 256;
    const int box_w = (int)align_up((size_t)((F + nb - 1) / nb), 8);
    BwdArgs a;
    a.rowptr = plan->rowptr - plan->row_offset;
    a.pos_row = plan->pos_row;
    a.task_pos = plan->task_pos;
    a.task_item = plan->task_item;
    a.n_tasks = items > 0 ? plan->n_tasks : plan->n_light_tasks;
    a.next = counter;
    a.E_root = plan->E;
    a.gidx = plan->col;
    a.eid = plan->perm_identity ? nullptr : plan->perm;
    a.gsd = gsd;
    a.dlogit = dlogit;
    a.part = part;
    a.item_lo = plan->item_lo;
    a.row_lo = plan->row_offset;
    a.row_hi = plan->row_offset + n;
    a.F = F; a.H = H; a.C = C; a.box_w = box_w; a.nb = nb;
    a.slope = slope;
    // stage: z boxes | g boxes | alpha rows | s_src rows | t rows | s_dst rows (TMA destinations 128 B aligned)
    a.zbytes = 16 * nb * box_w;
    a.off_g = (int)align_up((size_t)a.zbytes, 128);
    a.off_a = a.off_g + (int)align_up((size_t)a.zbytes, 128);
    a.off_s = a.off_a + (int)align_up((size_t)16 * H, 128);
    a.off_t = a.off_s + (int)align_up((size_t)16 * H, 128);
    a.off_d = a.off_t + (int)align_up((size_t)16 * H, 128);
    // factored alpha (alpha = p / rs_i): with g' = g_i / rs_i (written by the t kernel, also grad_z's
    // input), d' = g' . z_j = d / rs_i and t' = g' . out_i = t / rs_i, so p (d' - t') = alpha (d - t):
    // the SDDMM gathers g' and needs no row-sum gather or division
    a.stage_bytes = (int)align_up((size_t)(a.off_d + 16 * H), 128);
    const int S = std::max(2, std::min(3, (knobs().gat_warp_kb * 1024) / a.stage_bytes));
    a.data_off = (int)align_up((size_t)(128 + S * kMeta), 128);
    a.warp_bytes = (int)align_up((size_t)(a.data_off + S * a.stage_bytes), 128);
    // 8 warps per CTA while two CTAs still fit an SM (F = 128: 8 x 9.9 KB); wide rows take fewer
    int warps = knobs().gat_warps == 4 || knobs().gat_warps == 2 ? knobs().gat_warps : 8;
    while (warps > 1 && warps * a.warp_bytes > 112 * 1024) warps >>= 1;
    const int smem = warps * a.warp_bytes;
    if (smem > 227 * 1024) return fail(PYG_ERR_UNSUPPORTED, "gat_backward: stage ring does not fit shared memory");

    CUtensorMap tm[6];
    if (row_sums && !gsc) return fail(PYG_ERR_INVALID_ARGUMENT, "internal: factored alpha without g' scratch");
    if (!encode_rows(&tm[0], z, F, n_src, ldz, box_w) ||
        !(row_sums ? encode_rows(&tm[1], gsc, F, n, F, box_w) : encode_rows(&tm[1], g, F, n, ldg, box_w)) ||
        !encode_rows(&tm[2], alpha, H, plan->E, H, H) || !encode_rows(&tm[3], s_src, H, n_src, H, H) ||
        !encode_rows(&tm[4], gsd, H, n, H, H) || !encode_rows(&tm[5], s_dst, H, n, H, H))
        return fail(PYG_ERR_CUDA, "gat_backward: cuTensorMapEncodeTiled failed");
    const int64_t want = cdiv(a.n_tasks, warps);
    // C = 4 CPH <= 128: F <= 1024 -> NB = 1 (F <= 256), 2 (<= 512) or 4 column boxes
    auto go = [&](auto nbc) -> pyg_status_t {
        constexpr int NBc = decltype(nbc)::value;
        switch (C / 4) {
            case 1: return launch<1, NBc>(S, want, warps, smem, s, tm, a);
            case 2: return launch<2, NBc>(S, want, warps, smem, s, tm, a);
            case 4: return launch<4, NBc>(S, want, warps, smem, s, tm, a);
            case 8: return launch<8, NBc>(S, want, warps, smem, s, tm, a);
            case 16: return launch<16, NBc>(S, want, warps, smem, s, tm, a);
            default: return launch<32, NBc>(S, want, warps, smem, s, tm, a);
        }
    };
    if (nb == 1) PYG_TRY(go(std::integral_constant<int, 1>()));
    else if (nb == 2) PYG_TRY(go(std::integral_constant<int, 2>()));
    else PYG_TRY(go(std::integral_constant<int, 4>()));
    if (items > 0) {
        const int64_t nt = (plan->h_hi - plan->h_lo) * H;
        gat_combine_kernel<<<(unsigned)cdiv(nt, 256), 256, 0, s>>>(plan->heavy_rows, plan->heavy_item_ptr, plan->h_lo,
                                                                   plan->h_hi, plan->item_lo, plan->row_offset, part,
                                                                   H, gsd);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    return PYG_OK;
}


// ---- helpers ----

namespace gat {
__global__ void scale_rows_kernel(const float* __restrict__ g, int64_t ldg, int64_t n, int H, int C,
                                  const float* __restrict__ rs, float* gsc) {
    const int64_t F = (int64_t)H * C, total = n * F;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
        const int64_t r = t / F, c = t - r * F;
        gsc[t] = g[r * ldg + c] / rs[r * H + c / C];
    }
}
__global__ void fill_kernel(float* p, int64_t n, float v) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n; t += stride) p[t] = v;
}
}  // namespace gat

pyg_status_t gat_scale_rows(const float* g, int64_t ldg, int64_t n, int H, int C, const float* row_sums, float* gsc,
                            cudaStream_t s) {
    const int64_t total = n * H * C;
    if (total <= 0) return PYG_OK;
    gat::scale_rows_kernel<<<(unsigned)std::min<int64_t>(cdiv(total, 256), 148 * 16), 256, 0, s>>>(g, ldg, n, H, C,
                                                                                                   row_sums, gsc);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t fill_const(float* p, int64_t n, float v, cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    gat::fill_kernel<<<(unsigned)std::min<int64_t>(cdiv(n, 256), 148 * 16), 256, 0, s>>>(p, n, v);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

// ---- forward host side ----

size_t gat_fwd_tma_ws_bytes(const pyg_plan* plan, int64_t H, int64_t F) {
    if (!plan) return 0;
    const size_t items = (size_t)std::max<int64_t>(0, plan->item_hi - plan->item_lo);
    const size_t ldp = align_up((size_t)F, 4);
    return 256 + 256 + align_up((size_t)plan->n_rows * H * 4, 256) + align_up(items * ldp * 4, 256) +
           align_up(items * H * 4, 256) + align_up(((size_t)plan->n_rows + 1) * 4, 256);
}

bool gat_fwd_tma_eligible(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t ldz, float* out,
                          int64_t ldo, const float* alpha, const float* s_src, const float* s_dst) {
    using namespace gat;
    const int mode = knobs().seg_tma;
    if (mode == 0 || knobs().gat_fused == 0 || !plan || !plan->parts.empty() || plan->n_tasks <= 0 ||
        !plan->task_pos || !plan->pos_row)
        return false;
    if (plan->n_empty > 0 && !plan->row_order) return false;
    // C % 4: a float4 chunk of z must stay inside one head (its weight is the head's alpha); C = 75
    // (Reddit's 600 = 8 x 75) straddles heads and takes the two-pass kernels
    if (!(H == 4 || H == 8) || F % 4 || F > 1024 || F < 16 || C <= 0 || C % 4) return false;
    if (mode != 1 && plan->n_light_tasks < 1024) return false;
    if (!al16(z) || ldz % 4 || !al16(out) || ldo % 4) return false;
    if (!al16(alpha) || !al16(s_src) || !al16(s_dst)) return false;
    return tma::encode_fn() != nullptr;
}

pyg_status_t gat_fwd_tma(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                         const float* s_src, const float* s_dst, float slope, float* out, int64_t ldo, float* alpha,
                         float* row_sums, void* ws, size_t ws_bytes, cudaStream_t s) {
    using namespace gat;
    const int64_t n = plan->n_rows;
    const int64_t items = plan->item_hi - plan->item_lo;
    const int64_t ldp = (int64_t)align_up((size_t)F, 4);
    Carver cv(ws, ws_bytes);
    unsigned long long* counter = cv.take<unsigned long long>(1);
    unsigned* smax = cv.take<unsigned>(8);
    float* rs = cv.take<float>((size_t)n * H);
    float* part = cv.take<float>((size_t)std::max<int64_t>(items, 0) * ldp);
    float* part_s = cv.take<float>((size_t)std::max<int64_t>(items, 0) * H);
    int* bad = cv.take<int>((size_t)n + 1);
    if (row_sums) rs = row_sums;  // factored alpha: the caller keeps the row sums, alpha stays p
    if (!ws || !cv.ok()) return fail(PYG_ERR_NO_MEMORY, "gat_propagate: workspace too small (pyg_gat_propagate_workspace_size)");
    PYG_CUDA(cudaMemsetAsync(counter, 0, 256 + 256, s));  // counter and smax (adjacent carves)
    PYG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    {
        const int64_t total = n_src * H;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 4));
        gat_smax_kernel<<<blocks, 256, 0, s>>>(s_src, total, H, smax);
        PYG_LAUNCHED();
    }
    const int nb = (F + 255) / 256;
    const int box_w = (int)align_up((size_t)((F + nb - 1) / nb), 8);
    const int nch = (int)cdiv(nb * box_w, 128);
    FwdArgs a;
    a.rowptr = plan->rowptr - plan->row_offset;
    a.pos_row = plan->pos_row;
    a.task_pos = plan->task_pos;
    a.task_item = plan->task_item;
    a.n_tasks = items > 0 ? plan->n_tasks : plan->n_light_tasks;
    a.next = counter;
    a.E_root = plan->E;
    a.gidx = plan->col;
    a.eid = plan->perm_identity ? nullptr : plan->perm;
    a.s_dst = s_dst;
    a.smax = smax;
    a.alpha = alpha;
    a.out = out;
    a.ldo = ldo;
    a.rs = rs;
    a.part = part;
    a.part_s = part_s;
    a.ldp = ldp;
    a.item_lo = plan->item_lo;
    a.bad = bad;
    a.row_lo = plan->row_offset;
    a.row_hi = plan->row_offset + n;
    a.F = F; a.H = H; a.C = C; a.box_w = box_w; a.nb = nb;
    a.slope = slope;
    a.zbytes = 16 * nb * box_w;
    a.off_s = (int)align_up((size_t)a.zbytes, 128);
    a.off_d = a.off_s + (int)align_up((size_t)16 * H, 128);
    a.stage_bytes = (int)align_up((size_t)(a.off_d + 16 * H), 128);
    const int S = std::max(2, std::min(3, (knobs().gat_fwd_warp_kb * 1024) / a.stage_bytes));
    a.data_off = (int)align_up((size_t)(128 + S * kMeta + 128), 128);
    a.warp_bytes = (int)align_up((size_t)(a.data_off + S * a.stage_bytes), 128);
    int warps = knobs().gat_warps == 4 || knobs().gat_warps == 2 ? knobs().gat_warps : 8;
    while (warps > 1 && warps * a.warp_bytes > 112 * 1024) warps >>= 1;
    const int smem = warps * a.warp_bytes;
    if (smem > 227 * 1024) return fail(PYG_ERR_UNSUPPORTED, "gat_propagate: stage ring does not fit shared memory");
    CUtensorMap tz, tsrc;
    CUtensorMap tdst;
    if (!encode_rows(&tz, z, F, n_src, ldz, box_w) || !encode_rows(&tsrc, s_src, H, n_src, H, H) ||
        !encode_rows(&tdst, s_dst, H, n, H, H))
        return fail(PYG_ERR_CUDA, "gat_propagate: cuTensorMapEncodeTiled failed");
    const int64_t want = cdiv(a.n_tasks, warps);
    const int sm_kb = knobs().gat_fwd_sm_kb;
    switch (nch) {
        case 1: PYG_TRY(launch_fwd<1>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
        case 2: PYG_TRY(launch_fwd<2>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
        case 3: PYG_TRY(launch_fwd<3>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
        case 4: PYG_TRY(launch_fwd<4>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
        case 5: case 6: PYG_TRY(launch_fwd<6>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
        default: PYG_TRY(launch_fwd<8>(S, want, warps, smem, sm_kb, s, tz, tsrc, tdst, a)); break;
    }
    if (items > 0) {
        gat_fwd_combine_kernel<<<(unsigned)(plan->h_hi - plan->h_lo), 128, 0, s>>>(
            plan->heavy_rows, plan->heavy_item_ptr, plan->h_lo, plan->item_lo, plan->row_offset, part, ldp, part_s, H,
            C, F, out, ldo, rs, bad);
        PYG_LAUNCHED();
    }
    if (plan->n_empty > 0) {
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(plan->n_empty, 8), 148 * 16));
        gat_empty_rows_kernel<<<blocks, 256, 0, s>>>(plan->row_order, plan->empty_begin,
                                                     plan->empty_begin + plan->n_empty, plan->row_offset,
                                                     plan->row_offset + n, F, out, ldo);
        PYG_LAUNCHED();
    }
    if (!row_sums) {
        const int64_t total_max = plan->E * H;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total_max, 256), 148 * 16));
        gat_alpha_norm_kernel<<<blocks, 256, 0, s>>>(plan->pos_row, a.eid, plan->rowptr, n, plan->row_offset, H, rs,
                                                     alpha);
        PYG_LAUNCHED();
    }
    gat_fwd_fix_kernel<<<148, 256, 0, s>>>(bad, plan->rowptr, plan->col, a.eid, z, ldz, s_src, s_dst, H, C, F, slope,
                                           alpha, out, ldo, row_sums);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}


// ============================================================================================
// Forward on a SOURCE-BLOCKED plan (one pass per L2-resident block of z rows, like the segment-reduce
// passes): the fixed per-row shift of the one-pass forward (reading A9) makes the softmax additive
// across passes -- each pass adds sum p z_j into out and sum p into the row sums; the last pass
// divides.  A warp per row of the pass, the lanes over float4 column chunks; every lane forms the
// weight of its chunk's head (s_src[j] load, exp) per position.
// ============================================================================================
namespace gat {

struct BlockArgs {
    const int64_t* rowptr;  // this pass's virtual rows (n + 1)
    int64_t n;
    const int32_t* col;
    const int32_t* eid;
    const float* z;
    int64_t ldz;
    const float* s_src;
    const float* s_dst;
    const unsigned* smax;
    const int32_t* deg;     // total in-degree per row (blocked plans)
    float* out;
    int64_t ldo;
    float* rs;              // [n x H] running row sums
    float* alpha;           // [E x H]: p by edge id
    int* bad;
    int H, C, F;
    float slope;
    int accum, finalize;
};

// A warp per row of the pass; positions in groups of 4: lane (i, h) = (lane / 8, lane % 8) forms the
// weight of position i, head h (one s_src load and one exp per lane per group), the column lanes
// gather the 4 z_j rows (loads in flight together) and take each weight by a shuffle.
template <int NCH>
__global__ void __launch_bounds__(256, NCH >= 3 ? 2 : 3) gat_fwd_block_kernel(BlockArgs a) {
    const int lane = threadIdx.x & 31;
    const int my_i = lane >> 3, my_h = lane & 7;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int H = a.H;
    const bool hv = my_h < H;
    int hch[NCH];
    bool cval[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) {
        const int c = 4 * (lane + 32 * ch);
        cval[ch] = c < a.F;
        hch[ch] = cval[ch] ? c / a.C : 0;
    }
    const float smax_h = hv ? ord2f(__ldg(a.smax + my_h)) : 0.0f;
    for (int64_t r = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); r < a.n; r += nw) {
        const int64_t beg = a.rowptr[r], end = a.rowptr[r + 1];
        // this lane's head: s_dst and the row's shift (>= every logit of the row, reading A9)
        const float sd = hv ? __ldg(a.s_dst + r * H + my_h) : 0.0f;
        const float cpre = smax_h + sd;
        const float cs = cpre > 0.0f ? cpre : a.slope * cpre;
        float ps = 0.0f, acc[NCH][4];
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
            for (int q = 0; q < 4; ++q) acc[ch][q] = 0.0f;
        for (int64_t base = beg; base < end; base += 32) {
            const int cnt = (int)min((int64_t)32, end - base);
            int jl = 0, el = 0;
            if (lane < cnt) {
                jl = __ldg(a.col + base + lane);
                el = a.eid ? __ldg(a.eid + base + lane) : (int)(base + lane);
            }
            for (int t0 = 0; t0 < cnt; t0 += 4) {
                int js[4];
#pragma unroll
                for (int u = 0; u < 4; ++u) js[u] = __shfl_sync(0xffffffffu, jl, (t0 + u) & 31);
                // z rows in flight per lane: all 4 positions for rows of <= 2 chunks, 2 or 1 at a time for wider
                // rows (a wide row's 4 x NCH float4 capped the kernel at 1-2 CTAs per SM: NCH = 6 took 182
                // registers)
                constexpr int UH = NCH <= 2 ? 4 : (NCH <= 4 ? 2 : 1);
                float4 zv[UH][NCH];
                auto load_z = [&](int u0) {
#pragma unroll
                    for (int u = 0; u < UH; ++u)
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch)
                            zv[u][ch] = (cval[ch] && t0 + u0 + u < cnt)
                                            ? __ldg(reinterpret_cast<const float4*>(a.z + (int64_t)js[u0 + u] * a.ldz) +
                                                    lane + 32 * ch)
                                            : make_float4(0.f, 0.f, 0.f, 0.f);
                };
                load_z(0);
                // weight of (position t0 + my_i, head my_h)
                const int jm = __shfl_sync(0xffffffffu, jl, (t0 + my_i) & 31);
                const int em = __shfl_sync(0xffffffffu, el, (t0 + my_i) & 31);
                float p = 0.0f;
                if (hv && t0 + my_i < cnt) {
                    const float pre = __ldg(a.s_src + (int64_t)jm * H + my_h) + sd;
                    const float l = pre > 0.0f ? pre : a.slope * pre;
                    p = expf(l - cs);
#if PYG_GAT_STCS
                    __stcs(a.alpha + (int64_t)em * H + my_h, p);  // streamed: keeps the L2-resident z block
#else
                    a.alpha[(int64_t)em * H + my_h] = p;
#endif
                }
                ps += p;
#pragma unroll
                for (int u0 = 0; u0 < 4; u0 += UH) {
                    if (u0 > 0) load_z(u0);
#pragma unroll
                    for (int u = 0; u < UH; ++u)
#pragma unroll
                        for (int ch = 0; ch < NCH; ++ch) {
                            const float w = __shfl_sync(0xffffffffu, p, (u0 + u) * 8 + hch[ch]);
                            acc[ch][0] = fmaf(w, zv[u][ch].x, acc[ch][0]);
                            acc[ch][1] = fmaf(w, zv[u][ch].y, acc[ch][1]);
                            acc[ch][2] = fmaf(w, zv[u][ch].z, acc[ch][2]);
                            acc[ch][3] = fmaf(w, zv[u][ch].w, acc[ch][3]);
                        }
                }
            }
        }
        // the row's per-head sum over its position groups (lanes h, h + 8, h + 16, h + 24)
        ps += __shfl_xor_sync(0xffffffffu, ps, 8);
        ps += __shfl_xor_sync(0xffffffffu, ps, 16);
        float tot = ps;
        if (a.accum && hv && lane < 8) tot += a.rs[r * H + my_h];
        if (hv && lane < 8) a.rs[r * H + my_h] = tot;
        // a row whose sum underflowed in any head is listed once (the list holds at most n rows)
        const bool tiny = a.finalize && hv && lane < 8 && !(tot >= kTinySum) && __ldg(a.deg + r) > 0;
        if (__ballot_sync(0xffffffffu, tiny) && lane == 0) a.bad[1 + atomicAdd(a.bad, 1)] = (int)r;
        // epilogue: add the earlier passes, divide in the last
#pragma unroll
        for (int ch = 0; ch < NCH; ++ch) {
            const float th = __shfl_sync(0xffffffffu, tot, hch[ch]);
            if (!cval[ch]) continue;
            float4* o = reinterpret_cast<float4*>(a.out + r * a.ldo) + lane + 32 * ch;
            if (a.accum) {
                const float4 prev = *o;
                acc[ch][0] += prev.x; acc[ch][1] += prev.y; acc[ch][2] += prev.z; acc[ch][3] += prev.w;
            }
            if (a.finalize) {
                const float inv = th > 0.0f ? 1.0f / th : 0.0f;
                *o = make_float4(acc[ch][0] * inv, acc[ch][1] * inv, acc[ch][2] * inv, acc[ch][3] * inv);
            } else {
                *o = make_float4(acc[ch][0], acc[ch][1], acc[ch][2], acc[ch][3]);
            }
        }
    }
}

// alpha[k] /= rs[row] over one pass's rows (non-factored calls on blocked plans): warp per row
__global__ void gat_alpha_norm_rows_kernel(const int64_t* __restrict__ rowptr, int64_t n, const int32_t* __restrict__ eid,
                                           int H, const float* __restrict__ rs, float* alpha) {
    const int lane = threadIdx.x & 31;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t r = (((int64_t)blockIdx.x * blockDim.x) >> 5) + (threadIdx.x >> 5); r < n; r += nw) {
        const int64_t beg = rowptr[r], end = rowptr[r + 1];
        for (int64_t u = beg * H + lane; u < end * H; u += 32) {
            const int64_t p = u / H;
            const int h = (int)(u - p * H);
            const int64_t k = eid ? (int64_t)eid[p] : p;
            alpha[k * H + h] = alpha[k * H + h] / rs[r * H + h];
        }
    }
}

constexpr int kMaxParts = 64;
struct PartPtrs {
    const int64_t* rp[kMaxParts];
    int n;
};

// the listed rows of a blocked plan, exactly (as gat_fwd_fix_kernel, positions spread over the passes)
__global__ void gat_fwd_fix_blocked_kernel(const int* __restrict__ bad, PartPtrs parts, const int32_t* __restrict__ col,
                                           const int32_t* __restrict__ eid, const float* __restrict__ z, int64_t ldz,
                                           const float* __restrict__ s_src, const float* __restrict__ s_dst, int H,
                                           int C, int F, float slope, float* alpha, float* out, int64_t ldo,
                                           float* row_sums) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    const int count = bad[0];
    for (int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < count; w += warps) {
        const int64_t r = bad[1 + w];
        for (int h = 0; h < H; ++h) {
            const float sd = s_dst[r * H + h];
            float m = -INFINITY, sum = 0.0f;
            for (int b = 0; b < parts.n; ++b)
                for (int64_t p = parts.rp[b][r] + lane; p < parts.rp[b][r + 1]; p += 32) {
                    const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                    m = fmaxf(m, pre > 0.0f ? pre : slope * pre);
                }
            for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
            for (int b = 0; b < parts.n; ++b)
                for (int64_t p = parts.rp[b][r] + lane; p < parts.rp[b][r + 1]; p += 32) {
                    const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                    sum += expf((pre > 0.0f ? pre : slope * pre) - m);
                }
            for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
            for (int b = 0; b < parts.n; ++b)
                for (int64_t p = parts.rp[b][r] + lane; p < parts.rp[b][r + 1]; p += 32) {
                    const float pre = s_src[(int64_t)col[p] * H + h] + sd;
                    const int64_t k = eid ? (int64_t)eid[p] : p;
                    alpha[k * H + h] = expf((pre > 0.0f ? pre : slope * pre) - m) / sum;
                }
            if (row_sums && lane == 0) row_sums[r * H + h] = 1.0f;
        }
        __syncwarp();
        for (int c = lane; c < F; c += 32) {
            float acc = 0.0f;
            for (int b = 0; b < parts.n; ++b)
                for (int64_t p = parts.rp[b][r]; p < parts.rp[b][r + 1]; ++p) {
                    const int64_t k = eid ? (int64_t)eid[p] : p;
                    acc = fmaf(alpha[k * H + c / C], z[(int64_t)col[p] * ldz + c], acc);
                }
            out[r * ldo + c] = acc;
        }
    }
}

}  // namespace gat

size_t gat_fwd_blocked_ws_bytes(const pyg_plan* plan, int64_t H) {
    if (!plan) return 0;
    return 256 + 256 + align_up((size_t)plan->n_rows * H * 4, 256) + align_up(((size_t)plan->n_rows + 1) * 4, 256);
}

pyg_status_t gat_fwd_blocked(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                             const float* s_src, const float* s_dst, float slope, float* out, int64_t ldo, float* alpha,
                             float* row_sums, void* ws, size_t ws_bytes, cudaStream_t s) {
    using namespace gat;
    const int64_t n = plan->n_rows;
    const size_t np = plan->parts.size();
    if (np > (size_t)kMaxParts) return fail(PYG_ERR_UNSUPPORTED, "gat_propagate: at most %d source blocks", kMaxParts);
    if (C % 4 || F > 1024 || (reinterpret_cast<uintptr_t>(z) & 15) || ldz % 4 || (reinterpret_cast<uintptr_t>(out) & 15) ||
        ldo % 4 || !plan->deg)
        return fail(PYG_ERR_UNSUPPORTED, "gat_propagate on a source-blocked plan: C %% 4 == 0 (a float4 chunk inside one "
                                         "head), H*C <= 1024, 16-byte rows");
    Carver cv(ws, ws_bytes);
    cv.take<unsigned long long>(1);
    unsigned* smax = cv.take<unsigned>(8);
    float* rs = cv.take<float>((size_t)n * H);
    int* bad = cv.take<int>((size_t)n + 1);
    if (!ws || !cv.ok()) return fail(PYG_ERR_NO_MEMORY, "gat_propagate: workspace too small (pyg_gat_propagate_workspace_size)");
    if (row_sums) rs = row_sums;
    PYG_CUDA(cudaMemsetAsync(smax, 0, 8 * sizeof(unsigned), s));
    PYG_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
    {
        const int64_t total = n_src * H;
        const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 4));
        gat_smax_kernel<<<blocks, 256, 0, s>>>(s_src, total, H, smax);
        PYG_LAUNCHED();
    }
    BlockArgs a;
    a.n = n;
    a.col = plan->col;
    a.eid = plan->perm_identity ? nullptr : plan->perm;
    a.z = z; a.ldz = ldz; a.s_src = s_src; a.s_dst = s_dst; a.smax = smax; a.deg = plan->deg;
    a.out = out; a.ldo = ldo; a.rs = rs; a.alpha = alpha; a.bad = bad;
    a.H = H; a.C = C; a.F = F; a.slope = slope;
    const int nch = (int)cdiv(F, 128);
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8), 148 * 8));
    const int64_t total_passes = plan->n_passes > 0 ? plan->n_passes : (int64_t)np;
    for (size_t b = 0; b < np; ++b) {
        const int64_t gb = plan->pass_base + (int64_t)b;
        a.rowptr = plan->parts[b].rowptr;
        a.accum = gb > 0;
        a.finalize = gb + 1 == total_passes;
        switch (nch) {
            case 1: gat_fwd_block_kernel<1><<<blocks, 256, 0, s>>>(a); break;
            case 2: gat_fwd_block_kernel<2><<<blocks, 256, 0, s>>>(a); break;
            case 3: gat_fwd_block_kernel<3><<<blocks, 256, 0, s>>>(a); break;
            case 4: gat_fwd_block_kernel<4><<<blocks, 256, 0, s>>>(a); break;
            case 5: case 6: gat_fwd_block_kernel<6><<<blocks, 256, 0, s>>>(a); break;
            default: gat_fwd_block_kernel<8><<<blocks, 256, 0, s>>>(a); break;
        }
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    if (!row_sums)
        for (size_t b = 0; b < np; ++b) {
            gat_alpha_norm_rows_kernel<<<blocks, 256, 0, s>>>(plan->parts[b].rowptr, n, a.eid, H, rs, alpha);
            PYG_LAUNCHED();
        }
    PartPtrs pp;
    pp.n = (int)np;
    for (size_t b = 0; b < np; ++b) pp.rp[b] = plan->parts[b].rowptr;
    gat_fwd_fix_blocked_kernel<<<148, 256, 0, s>>>(bad, pp, plan->col, a.eid, z, ldz, s_src, s_dst, H, C, F, slope,
                                                   alpha, out, ldo, row_sums);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
