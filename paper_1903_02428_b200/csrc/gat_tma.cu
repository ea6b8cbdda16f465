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

constexpr int kMeta = 48;  // per stage: int keys[4] | int rows[4] | int eids[4]

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
    const float* g;          // grad_out [n x F] stride ldg (rows 16-byte aligned)
    int64_t ldg;
    const float* s_dst;      // [n x H] packed
    float* gsd;              // grad_s_dst [n x H]: t_i on entry, the row sums on exit
    float* dlogit;           // [E x H] packed, by edge id
    float* part;             // hub chunk partials [items x H]
    int64_t item_lo;
    int64_t row_lo, row_hi;  // this plan's root rows
    int F, H, C, box_w, nb;
    float slope;
    int warp_bytes, data_off;
    int zbytes, off_a, off_s, off_g, off_t, off_d, stage_bytes;
};

template <int NCH, int S>
__global__ void __launch_bounds__(256) gat_bwd_tma_kernel(const __grid_constant__ CUtensorMap tz,
                                                          const __grid_constant__ CUtensorMap ta,
                                                          const __grid_constant__ CUtensorMap ts, BwdArgs a) {
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int warp = threadIdx.x >> 5;
    const uint32_t region = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)(warp * a.warp_bytes);
    const uint32_t bar0 = region;                     // S barriers
    const uint32_t meta0 = region + 128;              // S x kMeta
    const uint32_t scr = meta0 + (uint32_t)(S * kMeta);  // 4 slots x 8 heads of d_alpha (128 B)
    const uint32_t data0 = region + (uint32_t)a.data_off;
    const int H = a.H, F = a.F;
    const uint32_t stage_bytes = (uint32_t)a.stage_bytes;
    const uint32_t row_bytes = (uint32_t)(4 * a.box_w);

    if (lane == 0) {
#pragma unroll
        for (int s = 0; s < S; ++s) bar_init(bar0 + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();

    // lane chunk layout: float4 chunk (lane + 32 ch) = columns 4 (lane + 32 ch) .. + 3
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
    const int CL = a.C >= 128 ? 32 : a.C / 4;  // lanes sharing a head inside one chunk row
    const bool leader = (lane % CL) == 0;
    const int64_t plo = __ldg(a.rowptr + a.row_lo), phi = __ldg(a.rowptr + a.row_hi);

    // ---------------- producer state (warp-uniform) ----------------
    int64_t pp = 0, pe = 0, iwb = 0, nwb = -1, task = 0;
    bool done = false;
    int wg = 0, wr = 0, we = 0, ng = 0, nr = 0, ne = 0;
    int citem = -1;
    int pkey = -1;  // key of the last position issued (row starts are detected against it)

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
        const int key = citem >= 0 ? -(citem + 2) : row;
        int prev = __shfl_up_sync(0xffffffffu, key, 1);
        if (lane == 0) prev = pkey;
        const unsigned newm = __ballot_sync(0xffffffffu, lane < cnt && key != prev) & 0xFu;
        pkey = __shfl_sync(0xffffffffu, key, cnt - 1);
        if (lane < 4) {
            sts32(m, lane < cnt ? key : -1);
            sts32(m + 16, row);
            sts32(m + 32, e);
        }
        int gs4[4], es4[4], rs4[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const int sl = cnt > i ? i : 0;
            gs4[i] = __shfl_sync(0xffffffffu, gj, sl);
            es4[i] = __shfl_sync(0xffffffffu, e, sl);
            rs4[i] = __shfl_sync(0xffffffffu, row, sl);
        }
        if (lane == 0) {
            const uint32_t bar = bar0 + 8 * s;
            const uint32_t st = data0 + (uint32_t)s * stage_bytes;
            const uint32_t nnew = (uint32_t)__popc(newm);
            bar_expect(bar, (uint32_t)a.zbytes + 32u * (uint32_t)H + nnew * (uint32_t)(4 * F + 8 * H));
#pragma unroll
            for (int b = 0; b < 4; ++b)
                if (b < a.nb)
                    gather4(st + (uint32_t)b * 4u * row_bytes, &tz, b * a.box_w, gs4[0], gs4[1], gs4[2], gs4[3], bar);
            gather4(st + (uint32_t)a.off_a, &ta, 0, es4[0], es4[1], es4[2], es4[3], bar);
            gather4(st + (uint32_t)a.off_s, &ts, 0, gs4[0], gs4[1], gs4[2], gs4[3], bar);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                if (!((newm >> i) & 1u)) continue;
                const int64_t lr = (int64_t)rs4[i] - a.row_lo;
                bulk_copy(st + (uint32_t)a.off_g + (uint32_t)(i * 4 * F), a.g + lr * a.ldg, (uint32_t)(4 * F), bar);
                bulk_copy(st + (uint32_t)a.off_t + (uint32_t)(i * 4 * H), a.gsd + lr * H, (uint32_t)(4 * H), bar);
                bulk_copy(st + (uint32_t)a.off_d + (uint32_t)(i * 4 * H), a.s_dst + lr * H, (uint32_t)(4 * H), bar);
            }
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
    float4 gv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) gv[ch] = make_float4(0.f, 0.f, 0.f, 0.f);
    float treg = 0.0f, sdreg = 0.0f;  // lanes < H: t_i[h], s_dst[i][h] of the current row
    int crow = -1;                    // key of the row whose g_i is in gv
    int gkey = -1, grow = 0;          // key / root row of the head sums being accumulated
    float gs = 0.0f;                  // lanes < H: running head sum of dlogit
    const int my_i = lane >> 3, my_h = lane & 7;

    auto flush = [&]() {
        if (lane < H) {
            if (gkey < -1) a.part[((int64_t)(-gkey - 2) - a.item_lo) * H + lane] = gs;
            else a.gsd[((int64_t)grow - a.row_lo) * H + lane] = gs;
        }
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
        sts32f(scr + 4u * (uint32_t)lane, 0.0f);
        bar_wait(bar0 + 8 * s, (phase >> s) & 1u);
        phase ^= 1u << s;
        __syncwarp();
        const uint32_t st = data0 + (uint32_t)s * stage_bytes;
        const int kk[4] = {keys.x, keys.y, keys.z, keys.w};
        float tme = 0.0f, sme = 0.0f;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i >= c) break;
            if (kk[i] != crow) {  // a row starts at slot i: its g_i / t_i / s_dst[i] are in this stage
                crow = kk[i];
                const uint32_t gb = st + (uint32_t)a.off_g + (uint32_t)(i * 4 * F) + 16u * (uint32_t)lane;
#pragma unroll
                for (int ch = 0; ch < NCH; ++ch)
                    gv[ch] = cval[ch] ? lds128f(gb + 512u * (uint32_t)ch) : make_float4(0.f, 0.f, 0.f, 0.f);
                if (lane < H) {
                    treg = lds32f(st + (uint32_t)a.off_t + (uint32_t)(i * 4 * H) + 4u * (uint32_t)lane);
                    sdreg = lds32f(st + (uint32_t)a.off_d + (uint32_t)(i * 4 * H) + 4u * (uint32_t)lane);
                }
            }
            const float tv = __shfl_sync(0xffffffffu, treg, my_h);
            const float sv = __shfl_sync(0xffffffffu, sdreg, my_h);
            if (my_i == i) { tme = tv; sme = sv; }
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const float4 zv = cval[ch] ? lds128f(st + coff[ch] + (uint32_t)i * row_bytes)
                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                float d = gv[ch].x * zv.x;
                d = fmaf(gv[ch].y, zv.y, d);
                d = fmaf(gv[ch].z, zv.z, d);
                d = fmaf(gv[ch].w, zv.w, d);
                for (int o = 1; o < CL; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (leader && cval[ch]) {
                    const uint32_t q = scr + 4u * (uint32_t)(i * 8 + hch[ch]);
                    sts32f(q, lds32f(q) + d);
                }
            }
        }
        __syncwarp();
        // 32 lanes = 4 slots x 8 heads: dlogit of (slot my_i, head my_h)
        float dl = 0.0f;
        if (my_i < c && my_h < H) {
            const float d = lds32f(scr + 4u * (uint32_t)lane);
            const float al = lds32f(st + (uint32_t)a.off_a + 4u * (uint32_t)(my_i * H + my_h));
            const float ss = lds32f(st + (uint32_t)a.off_s + 4u * (uint32_t)(my_i * H + my_h));
            const int e = my_i == 0 ? eids.x : my_i == 1 ? eids.y : my_i == 2 ? eids.z : eids.w;
            dl = al * (d - tme);
            if (!(ss + sme > 0.0f)) dl *= a.slope;
            a.dlogit[(int64_t)e * H + my_h] = dl;
        }
        // head sums per row, in position order
        const int rr[4] = {rows.x, rows.y, rows.z, rows.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            if (i >= c) break;
            const float v = __shfl_sync(0xffffffffu, dl, i * 8 + my_h);
            if (kk[i] != gkey) {
                if (gkey != -1) flush();
                gkey = kk[i];
                grow = rr[i];
                gs = 0.0f;
            }
            gs += v;
        }
        __syncwarp();  // every lane is done with stage s (data, scratch) before it is refilled
        fill(s);
    }
    if (gkey != -1) flush();
}

// t_i[h] = g_i . out_i |_h (0 for rows without in-edges), written into grad_s_dst.  Same lane
// layout, product order and reduction tree as the SDDMM in gat_bwd_tma_kernel, so a row whose
// forward output equals one source row bitwise (a single in-edge: alpha = 1) gets t_i equal to its
// d_alpha bitwise and dlogit exactly 0.  A warp takes RU rows per step (their loads in flight
// together).
template <int NCH, int RU>
__global__ void gat_t_kernel(const float* __restrict__ g, int64_t ldg, const float* __restrict__ out, int64_t ldo,
                             const int64_t* __restrict__ rowptr, int64_t n, int F, int H, int C, float* gsd) {
    const int lane = threadIdx.x & 31;
    const int CL = C >= 128 ? 32 : C / 4;
    const bool leader = (lane % CL) == 0;
    const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
    for (int64_t r0 = ((int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * RU; r0 < n; r0 += warps * RU) {
        // rowptr[r0 .. r0 + RU] in lanes 0..RU
        const int64_t rp = (lane <= RU && r0 + lane <= n) ? rowptr[r0 + lane] : 0;
        float4 x[RU][NCH], y[RU][NCH];
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int64_t r = r0 + u;
            const bool ok = r < n;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const bool cv = ok && 4 * (lane + 32 * ch) < F;
                x[u][ch] = cv ? __ldg(reinterpret_cast<const float4*>(g + r * ldg) + lane + 32 * ch) : make_float4(0.f, 0.f, 0.f, 0.f);
                y[u][ch] = cv ? __ldg(reinterpret_cast<const float4*>(out + r * ldo) + lane + 32 * ch) : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
#pragma unroll
        for (int u = 0; u < RU; ++u) {
            const int64_t r = r0 + u;
            const int64_t b = __shfl_sync(0xffffffffu, rp, u), e = __shfl_sync(0xffffffffu, rp, u + 1);
            if (r >= n) break;
            float acc[8];
#pragma unroll
            for (int h = 0; h < 8; ++h) acc[h] = 0.0f;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                const int c = 4 * (lane + 32 * ch);
                float d = x[u][ch].x * y[u][ch].x;
                d = fmaf(x[u][ch].y, y[u][ch].y, d);
                d = fmaf(x[u][ch].z, y[u][ch].z, d);
                d = fmaf(x[u][ch].w, y[u][ch].w, d);
                for (int o = 1; o < CL; o <<= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
                if (leader && c < F) {
                    const int hh = c / C;
#pragma unroll
                    for (int h = 0; h < 8; ++h)
                        if (h == hh) acc[h] += d;
                }
            }
#pragma unroll
            for (int h = 0; h < 8; ++h) {
                if (h >= H) break;
                const int owner = C >= 128 ? 0 : (h * (C / 4)) % 32;  // the leader lane of head h's chunk
                if (lane == owner) gsd[r * H + h] = e > b ? acc[h] : 0.0f;
            }
        }
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

template <int NCH>
pyg_status_t launch(int S, int64_t want, int warps, int smem, cudaStream_t s, const CUtensorMap& tz,
                    const CUtensorMap& ta, const CUtensorMap& tsrc, const BwdArgs& a) {
    void (*k)(const CUtensorMap, const CUtensorMap, const CUtensorMap, BwdArgs) =
        S >= 4 ? gat_bwd_tma_kernel<NCH, 4> : S == 3 ? gat_bwd_tma_kernel<NCH, 3> : gat_bwd_tma_kernel<NCH, 2>;
    PYG_CUDA(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    // as seg_tma, keep part of the SM's unified array as L1 for the index windows (two 77 KB CTAs
    // at F = 128 leave ~100 KB)
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
    k<<<grid, 32 * warps, smem, s>>>(tz, ta, tsrc, a);
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
    if (!((pow2 && C >= 4 && C <= 128) || C % 128 == 0)) return false;
    if (mode != 1 && plan->n_light_tasks < 1024) return false;
    if (!al16(z) || ldz % 4 || !al16(g) || ldg % 4 || !al16(out) || ldo % 4) return false;
    if (!al16(alpha) || !al16(s_src) || !al16(s_dst) || !al16(gsd)) return false;
    return tma::encode_fn() != nullptr;
}

pyg_status_t gat_bwd_tma(const pyg_plan* plan, int H, int C, int F, const float* z, int64_t n_src, int64_t ldz,
                         const float* g, int64_t ldg, const float* out, int64_t ldo, const float* alpha,
                         const float* s_src, const float* s_dst, float slope, float* dlogit, float* gsd, void* ws,
                         size_t ws_bytes, cudaStream_t s) {
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
        const int nch_t = (int)cdiv(F, 128);
        auto go = [&](auto k, int ru) {
            const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 8 * ru), 148 * 8));
            k<<<blocks, 256, 0, s>>>(g, ldg, out, ldo, plan->rowptr, n, F, H, C, gsd);
        };
        if (nch_t == 1) go(gat_t_kernel<1, 4>, 4);
        else if (nch_t == 2) go(gat_t_kernel<2, 2>, 2);
        else if (nch_t <= 4) go(gat_t_kernel<4, 1>, 1);
        else go(gat_t_kernel<8, 1>, 1);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
    }
    const int nb = (F + 255) / 256;
    const int box_w = (int)align_up((size_t)((F + nb - 1) / nb), 8);
    const int nch = (int)cdiv(nb * box_w, 128);
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
    a.g = g;
    a.ldg = ldg;
    a.s_dst = s_dst;
    a.gsd = gsd;
    a.dlogit = dlogit;
    a.part = part;
    a.item_lo = plan->item_lo;
    a.row_lo = plan->row_offset;
    a.row_hi = plan->row_offset + n;
    a.F = F; a.H = H; a.C = C; a.box_w = box_w; a.nb = nb;
    a.slope = slope;
    // stage: z boxes | alpha rows | s_src rows | g rows | t rows | s_dst rows (TMA destinations 128 B aligned)
    a.zbytes = 16 * nb * box_w;
    a.off_a = (int)align_up((size_t)a.zbytes, 128);
    a.off_s = a.off_a + (int)align_up((size_t)16 * H, 128);
    a.off_g = a.off_s + (int)align_up((size_t)16 * H, 128);
    a.off_t = a.off_g + 16 * F;
    a.off_d = a.off_t + 16 * H;
    a.stage_bytes = (int)align_up((size_t)(a.off_d + 16 * H), 128);
    const int S = std::max(2, std::min(4, (knobs().gat_warp_kb * 1024) / a.stage_bytes));
    a.data_off = (int)align_up((size_t)(128 + S * kMeta + 128), 128);
    a.warp_bytes = (int)align_up((size_t)(a.data_off + S * a.stage_bytes), 128);
    // 8 warps per CTA while two CTAs still fit an SM (F = 128: 8 x 9.6 KB); wide rows take fewer
    int warps = 8;
    while (warps > 1 && warps * a.warp_bytes > 112 * 1024) warps >>= 1;
    const int smem = warps * a.warp_bytes;
    if (smem > 227 * 1024) return fail(PYG_ERR_UNSUPPORTED, "gat_backward: stage ring does not fit shared memory");

    CUtensorMap tz, ta, tsrc;
    if (!encode_rows(&tz, z, F, n_src, ldz, box_w) || !encode_rows(&ta, alpha, H, plan->E, H, H) ||
        !encode_rows(&tsrc, s_src, H, n_src, H, H))
        return fail(PYG_ERR_CUDA, "gat_backward: cuTensorMapEncodeTiled failed");
    const int64_t want = cdiv(a.n_tasks, warps);
    switch (nch) {
        case 1: PYG_TRY(launch<1>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
        case 2: PYG_TRY(launch<2>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
        case 3: PYG_TRY(launch<3>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
        case 4: PYG_TRY(launch<4>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
        case 5: case 6: PYG_TRY(launch<6>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
        default: PYG_TRY(launch<8>(S, want, warps, smem, s, tz, ta, tsrc, a)); break;
    }
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

}  // namespace pyg
