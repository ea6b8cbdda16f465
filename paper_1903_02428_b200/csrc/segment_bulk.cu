// segment_bulk.cu -- the row-staged CSR segment-reduce for wide rows (sm_100a bulk copies): the same
// reduction as seg_kernel (gather of x_j, phi, BOX of Eq. (1)) with the in-flight rows held
// in SHARED memory instead of registers.
//
// Why: on a source-blocked plan every pass gathers from an L2-resident block of X, so the kernel is
// bound by how many gathered bytes each SM keeps in flight against the L2 latency.  seg_kernel keeps
// them in registers; the MAX instantiation (value + edge id per element) then fits only one edge per
// lane in flight at 3 CTAs per SM (Reddit max: 2.2 ms per pass vs 1.4 for sum).  Here one elected
// lane of each warp streams the rows of its positions with `cp.async.bulk.shared::cta.global`
// (SASS UBLKCP) into a ring of S row-sized stages completed on mbarriers; the 32 lanes read their
// float4 chunks of a landed row from shared memory (conflict-free: lane l reads bytes 16 l ..) and
// reduce in registers.  Registers hold only the accumulators (and argmax ids), so the ring depth,
// not the register file, sets the memory-level parallelism.
//
// Work: tasks of consecutive rows (contiguous position ranges of the CSR) pulled from a global
// counter; rows are closed in order (deterministic, same per-row summation order as seg_kernel, so
// results are bitwise equal to it); the row epilogue (mean divide, GCN / APPNP extras, multi-pass
// accumulate, MAX packed keys) is seg_kernel's row_epilogue.  Eligible: plans (or source-blocked
// parts) without split hub rows and without a light-row order, 256 <= F <= 1024, 16-byte aligned
// rows whose padded width may be read.
#include "segment_kernel.cuh"

namespace pyg {
namespace bulk {

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
        " BULK_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra BULK_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
// one contiguous row, global -> shared, completion counted on `bar`
__device__ __forceinline__ void copy_row(uint32_t dst, const void* src, uint32_t bytes, uint32_t bar) {
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                 "l"(src), "r"(bytes), "r"(bar)
                 : "memory");
}
__device__ __forceinline__ float4 lds128f(uint32_t addr) {
    float4 v;
    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(addr));
    return v;
}

struct Ring {
    int S;               // stages per warp
    uint32_t stride;     // bytes per stage (multiple of 128)
    uint32_t copy;       // bytes per copied row (multiple of 16)
    uint32_t warp_bytes; // 128 (barriers) + S * stride
    int rows_per_task;
    unsigned long long* next;
};

template <int NCH, int RED>
__global__ void __launch_bounds__(256) seg_bulk_kernel(SegArgs a, Ring g, int out_vec_ok) {
    constexpr bool IS_MAX = RED == PYG_MAX || RED == kRedMaxW;
    extern __shared__ __align__(128) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const uint32_t region = (uint32_t)__cvta_generic_to_shared(smem) + (uint32_t)((threadIdx.x >> 5) * g.warp_bytes);
    const uint32_t data0 = region + 128;
    if (lane == 0) {
        for (int s = 0; s < g.S; ++s) bar_init(region + 8 * s);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
    bool cv[NCH];
#pragma unroll
    for (int ch = 0; ch < NCH; ++ch) cv[ch] = 4 * (lane + 32 * ch) < a.ncols;
    const char* X = reinterpret_cast<const char*>(a.X);
    const uint64_t row_bytes = (uint64_t)a.ldx * 4;
    const bool need_e = IS_MAX || a.w != nullptr;
    uint32_t cnt = 0;  // positions consumed by this warp (ring slot = cnt % S, phase = cnt / S)

    for (;;) {
        int64_t task = 0;
        if (lane == 0) task = (int64_t)atomicAdd(g.next, 1ull);
        task = __shfl_sync(0xffffffffu, task, 0);
        const int64_t r0 = task * g.rows_per_task;
        if (r0 >= a.n_rows) break;
        const int64_t r1 = min(a.n_rows, r0 + (int64_t)g.rows_per_task);
        // the task's row pointers, one per lane (rows_per_task + 1 <= 32), read coalesced once
        const int64_t rp = (r0 + lane <= r1) ? __ldg(a.rowptr + r0 + lane) : 0;
        const int64_t pb = __shfl_sync(0xffffffffu, rp, 0);
        const int64_t pe = __shfl_sync(0xffffffffu, rp, (int)(r1 - r0));
        const int64_t n = pe - pb;
        // index windows (coalesced, one per 32 positions): A = [wb, wb + 32), B = the next 32
        int gA = 0, eA = 0, gB = 0, eB = 0;
        float sA = 1.0f, sB = 1.0f;
        auto load = [&](int64_t base, int& gg, int& ee, float& ss) {
            const int64_t p = base + lane;
            gg = 0; ee = 0; ss = 1.0f;
            if (p < pe) {
                gg = __ldg(a.gidx + p);
                if (need_e) {
                    ee = a.eid ? __ldg(a.eid + p) : (int)p;
                    if (a.w) ss = __ldg(a.w + ee);
                }
            }
        };
        int64_t wb = pb;
        load(wb, gA, eA, sA);
        load(wb + 32, gB, eB, sB);
        // the source row of window position j (j < 64), all lanes
        auto gsrc = [&](int j) -> int {
            const int a0 = __shfl_sync(0xffffffffu, gA, j & 31);
            const int b0 = __shfl_sync(0xffffffffu, gB, j & 31);
            return j < 32 ? a0 : b0;
        };
        // prologue: the first S positions of the task in flight
        for (int k = 0; k < g.S && k < n; ++k) {
            const int gq = gsrc(k);
            if (lane == 0) {
                const uint32_t slot = (cnt + k) % g.S;
                const uint32_t bar = region + 8 * slot;
                bar_expect(bar, g.copy);
                copy_row(data0 + slot * g.stride, X + (uint64_t)(uint32_t)gq * row_bytes, g.copy, bar);
            }
        }
        int64_t row = r0, rbeg = pb, rend = __shfl_sync(0xffffffffu, rp, 1);
        float acc[NCH][4];
        int bi[NCH][4];
        auto reset = [&]() {
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch)
#pragma unroll
                for (int q = 0; q < 4; ++q) { acc[ch][q] = IS_MAX ? -INFINITY : 0.0f; bi[ch][q] = -1; }
        };
        reset();
        for (int64_t k = 0; k < n; ++k) {
            const int64_t p = pb + k;
            if (p - wb >= 32) {
                wb += 32;
                gA = gB; eA = eB; sA = sB;
                load(wb + 32, gB, eB, sB);
            }
            while (rend <= p) {  // rows ending here (incl. empty rows) are complete
                seg::row_epilogue<4, NCH, RED, 32>(a, row, rend - rbeg, lane, 0, acc, bi, out_vec_ok);
                reset();
                ++row;
                rbeg = rend;
                rend = __shfl_sync(0xffffffffu, rp, (int)(row - r0 + 1));
            }
            const int jj = (int)(p - wb);
            int e = 0;
            float sc = 1.0f;
            if (need_e) {
                e = __shfl_sync(0xffffffffu, eA, jj);
                if (a.w) sc = __shfl_sync(0xffffffffu, sA, jj);
            }
            const uint32_t slot = cnt % g.S;
            bar_wait(region + 8 * slot, (cnt / g.S) & 1u);
            const uint32_t base = data0 + slot * g.stride + 16u * lane;
#pragma unroll
            for (int ch = 0; ch < NCH; ++ch) {
                if (!cv[ch]) continue;
                const float4 v4 = lds128f(base + 512u * ch);
                const float v[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    if (IS_MAX) {
                        const float m = RED == kRedMaxW ? __fmul_rn(sc, v[q]) : v[q];
                        if (m > acc[ch][q]) { acc[ch][q] = m; bi[ch][q] = e; }
                    } else {
                        acc[ch][q] = a.w ? fmaf(sc, v[q], acc[ch][q]) : acc[ch][q] + v[q];
                    }
                }
            }
            __syncwarp();  // every lane has read the stage: refill it with position p + S
            if (k + g.S < n) {
                const int gq = gsrc(jj + g.S);
                if (lane == 0) {
                    const uint32_t bar = region + 8 * slot;
                    bar_expect(bar, g.copy);
                    copy_row(data0 + slot * g.stride, X + (uint64_t)(uint32_t)gq * row_bytes, g.copy, bar);
                }
            }
            ++cnt;
        }
        while (row < r1) {  // the last row with positions and trailing empty rows
            seg::row_epilogue<4, NCH, RED, 32>(a, row, rend - rbeg, lane, 0, acc, bi, out_vec_ok);
            reset();
            ++row;
            if (row < r1) {
                rbeg = rend;
                rend = __shfl_sync(0xffffffffu, rp, (int)(row - r0 + 1));
            }
        }
    }
}

template <int RED>
pyg_status_t launch_red(const SegArgs& a, int nch, const Ring& g, int smem, int ovk, cudaStream_t s) {
    auto pick = [&](auto kern) -> pyg_status_t {
        // opt in to > 48 KB of dynamic shared memory on every launch (a cached "done once" flag went
        // stale inside the GPU test suite: the launch then failed with cudaErrorInvalidValue)
        PYG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        int dev = 0, sms = 0, per_sm = 0;
        PYG_CUDA(cudaGetDevice(&dev));
        PYG_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
        PYG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, 256, smem));
        const int64_t tasks = cdiv(a.n_rows, g.rows_per_task);
        const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((int64_t)sms * std::max(per_sm, 1), cdiv(tasks, 8)));
        kern<<<grid, 256, smem, s>>>(a, g, ovk);
        PYG_LAUNCHED();
        PYG_CUDA(cudaGetLastError());
        return PYG_OK;
    };
    switch (nch) {
        case 2: return pick(seg_bulk_kernel<2, RED>);
        case 3: return pick(seg_bulk_kernel<3, RED>);
        case 4: return pick(seg_bulk_kernel<4, RED>);
        case 5: return pick(seg_bulk_kernel<5, RED>);
        case 6: return pick(seg_bulk_kernel<6, RED>);
        case 7: return pick(seg_bulk_kernel<7, RED>);
        default: return pick(seg_bulk_kernel<8, RED>);
    }
}

}  // namespace bulk

bool bulk_eligible(const SegArgs& a, const pyg_plan* plan, int reduce) {
    // opt-in only (PYG_SEG_BULK=1): on Reddit's source-blocked MAX passes it measured 3.15 ms per pass
    // against 2.52 ms for seg_kernel (gpurun_out/r2k launch lists), so auto mode does not pick it
    const int mode = knobs().seg_bulk;
    (void)reduce;
    if (mode != 1 || (a.flags & PYG_NO_TMA) || !plan) return false;
    if (plan->item_hi > plan->item_lo || a.row_order || !a.gidx || a.gdeg || a.hw) return false;
    if (a.ncols < 256 || a.ncols > 1024) return false;
    if ((reinterpret_cast<uintptr_t>(a.X) & 15) || (a.ldx % 4)) return false;
    if (a.ncols % 4 && !(a.allow_pad_read && a.ldx >= (int64_t)align_up(a.ncols, 4))) return false;
    return true;
}

pyg_status_t segment_bulk(const SegArgs& a, int reduce, unsigned long long* counter, int ovk, cudaStream_t s) {
    if (!counter) return fail(PYG_ERR_NO_MEMORY, "bulk path needs workspace (see pyg_workspace_size)");
    PYG_CUDA(cudaMemsetAsync(counter, 0, sizeof(unsigned long long), s));
    bulk::Ring g;
    g.copy = (uint32_t)align_up((size_t)a.ncols * 4, 16);
    g.stride = (uint32_t)align_up(g.copy, 128);
    g.S = std::max(2, std::min(8, (knobs().bulk_warp_kb * 1024 - 128) / (int)g.stride));
    g.warp_bytes = 128 + g.S * g.stride;
    g.rows_per_task = 16;
    g.next = counter;
    const int smem = 8 * (int)g.warp_bytes;
    const int nch = (int)cdiv(cdiv(a.ncols, 4), 32);
    switch (reduce) {
        case PYG_SUM: return bulk::launch_red<PYG_SUM>(a, nch, g, smem, ovk, s);
        case PYG_MEAN: return bulk::launch_red<PYG_MEAN>(a, nch, g, smem, ovk, s);
        case kRedSumEpi: return bulk::launch_red<kRedSumEpi>(a, nch, g, smem, ovk, s);
        case kRedMaxW: return bulk::launch_red<kRedMaxW>(a, nch, g, smem, ovk, s);
        default: return bulk::launch_red<PYG_MAX>(a, nch, g, smem, ovk, s);
    }
}

}  // namespace pyg
