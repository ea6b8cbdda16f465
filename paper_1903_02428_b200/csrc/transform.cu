// transform.cu -- NEXT-2: the dense feature transform Y = X W^T of GCN / SGC /
// APPNP layers on the 5th-generation tensor cores -- the one place of the path that is
// a dense contraction (north_star: "Tensor cores are used only for the dense feature transform").
//
// tcgen05 (sm_100a) TF32 GEMM, fp32 in / fp32 accumulate / fp32 out:
//   * one CTA per 128-row tile of X (UMMA M = 128), the whole output width in one UMMA N
//     (N = F_out rounded up to 16, <= 256); 4 warps;
//   * warp 0 / one lane: TMA producer -- X tile [128 x 32] and W tile [N x 32] (K-major, 128-byte
//     rows, SWIZZLE_128B) per stage into an S-stage shared-memory ring guarded by full/empty
//     mbarriers (out-of-range rows / columns / K are zero-filled by the TMA unit);
//   * warp 1 / one lane: MMA issuer -- 4 x tcgen05.mma.cta_group::1.kind::tf32 (UMMA K = 8) per
//     stage into a TMEM accumulator (128 lanes x N fp32 columns), tcgen05.commit -> empty[s];
//     a final commit signals the epilogue;
//   * epilogue, all 4 warps: tcgen05.ld.32x32b (warp w reads TMEM lanes 32w..32w+31 = its 32
//     rows), optional per-row scale (e.g. GCN's D^-1/2, fusing the normalisation into the
//     transform) and bias, fp32 stores.
// TF32 keeps 10 mantissa bits of each operand: |Y - XW^T| <= ~2^-9 sum_k |x_k w_k| + fp32
// accumulation (reading A7).
#include <cuda.h>

#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace pyg {
namespace xform {

constexpr int kBM = 128;       // UMMA M
constexpr int kBK = 32;        // fp32 elements per 128-byte swizzle row
constexpr int kUmmaK = 8;      // TF32 UMMA K
constexpr int kThreads = 128;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint32_t bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n"
        " .reg .pred p;\n"
        " XF_WAIT_%=:\n"
        " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        " @!p bra XF_WAIT_%=;\n"
        "}\n" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void tma_load_2d(uint32_t dst, const CUtensorMap* map, int c0, int c1, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
            dst),
        "l"(map), "r"(c0), "r"(c1), "r"(bar)
        : "memory");
}

// K-major operand, SWIZZLE_128B: rows of 128 bytes, 8-row atoms 1024 bytes apart (SBO), LBO unused
// (encoded 1), version 1 (sm_100), layout type 2 (SWIZZLE_128B); K steps inside the atom advance the
// start address by 32 bytes.
__device__ __forceinline__ uint64_t smem_desc(uint32_t addr) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;                 // leading byte offset (16 B units)
    d |= (uint64_t)(1024 >> 4) << 32;       // stride byte offset
    d |= (uint64_t)1 << 46;                 // version
    d |= (uint64_t)2 << 61;                 // SWIZZLE_128B
    return d;
}

// instruction descriptor: D fp32, A/B TF32, both K-major, N >> 3, M >> 4
__host__ __device__ constexpr uint32_t instr_desc(int N) {
    return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

struct Args {
    int64_t M, K;
    int N;            // output columns (F_out)
    int UN;           // UMMA N (multiple of 16)
    int tmem_cols;    // power of two >= UN
    int stages;
    int kb;           // K blocks
    float* Y;
    int64_t ldy;
    const float* bias;       // [N] or null
    const float* row_scale;  // [M] or null
    // GAT attention projections fused into the epilogue: s_src[m][h] = sum_{c in head h} y[m][c] a_src[c]
    const float* att_src;    // [N] or null
    const float* att_dst;    // [N] or null
    float* s_src;            // [M x heads] packed
    float* s_dst;
    int heads, hc;           // heads and channels per head (N = heads * hc)
};

__global__ void __launch_bounds__(kThreads) tf32_gemm_kernel(const __grid_constant__ CUtensorMap map_x,
                                                                 const __grid_constant__ CUtensorMap map_w, Args a) {
    extern __shared__ __align__(1024) unsigned char smem_raw[];
    // 1024-byte aligned stage buffers (SWIZZLE_128B atoms must start on 1024-byte boundaries)
    const uint32_t base = (smem_u32(smem_raw) + 1023u) & ~1023u;
    unsigned char* gbase = smem_raw + (base - smem_u32(smem_raw));
    const uint32_t a_bytes = kBM * kBK * 4;            // 16 KB
    const uint32_t b_bytes = (uint32_t)a.UN * kBK * 4; // <= 32 KB
    const uint32_t stage_bytes = a_bytes + b_bytes;
    const uint32_t bars = base + (uint32_t)a.stages * stage_bytes;  // full[S], empty[S], done
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(gbase + (size_t)a.stages * stage_bytes + 8 * (2 * a.stages + 1));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t m0 = (int64_t)blockIdx.x * kBM;
    const int n0 = blockIdx.y * a.UN;            // this CTA's output-column tile (N > 256: several)
    const int nl = min(a.UN, a.N - n0);

    if (threadIdx.x == 0) {
        for (int s = 0; s < a.stages; ++s) {
            mbar_init(bars + 8 * s, 1);
            mbar_init(bars + 8 * (a.stages + s), 1);
        }
        mbar_init(bars + 8 * (2 * a.stages), 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
    }
    if (warp == 0) {  // TMEM accumulator: 128 lanes x tmem_cols fp32 columns
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                     "r"(a.tmem_cols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const uint32_t tmem = *tmem_slot;

    if (warp == 0 && lane == 0) {
        // ---- TMA producer ----
        for (int kb = 0; kb < a.kb; ++kb) {
            const int s = kb % a.stages;
            if (kb >= a.stages) mbar_wait(bars + 8 * (a.stages + s), ((kb / a.stages) - 1) & 1);
            const uint32_t sa = base + (uint32_t)s * stage_bytes;
            mbar_expect_tx(bars + 8 * s, stage_bytes);
            tma_load_2d(sa, &map_x, kb * kBK, (int)m0, bars + 8 * s);
            tma_load_2d(sa + a_bytes, &map_w, kb * kBK, n0, bars + 8 * s);
        }
    } else if (warp == 1 && lane == 0) {
        // ---- MMA issuer ----
        const uint32_t idesc = instr_desc(a.UN);
        for (int kb = 0; kb < a.kb; ++kb) {
            const int s = kb % a.stages;
            mbar_wait(bars + 8 * s, (kb / a.stages) & 1);
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint32_t sa = base + (uint32_t)s * stage_bytes;
#pragma unroll
            for (int k = 0; k < kBK / kUmmaK; ++k) {
                const uint64_t da = smem_desc(sa + k * kUmmaK * 4);
                const uint64_t db = smem_desc(sa + a_bytes + k * kUmmaK * 4);
                const uint32_t acc = (kb > 0 || k > 0) ? 1u : 0u;
                asm volatile(
                    "{\n"
                    " .reg .pred p;\n"
                    " setp.ne.b32 p, %4, 0;\n"
                    " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
                    "}\n" ::"r"(tmem),
                    "l"(da), "l"(db), "r"(idesc), "r"(acc)
                    : "memory");
            }
            // frees the stage once these MMAs have read it
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             bars + 8 * (a.stages + s))
                         : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                         bars + 8 * (2 * a.stages))
                     : "memory");
    }
    __syncwarp();

    // ---- epilogue: TMEM -> registers -> (row scale, bias) -> global ----
    mbar_wait(bars + 8 * (2 * a.stages), 0);
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    const int64_t row = m0 + warp * 32 + lane;
    const float rs = (a.row_scale && row < a.M) ? __ldg(a.row_scale + row) : 1.0f;
    const bool vec = ((a.ldy & 3) == 0) && ((reinterpret_cast<uintptr_t>(a.Y) & 15) == 0);
    float ps[8], pd[8];  // per-head projections of this thread's row (heads <= 8)
#pragma unroll
    for (int h = 0; h < 8; ++h) { ps[h] = 0.0f; pd[h] = 0.0f; }
    for (int c0 = 0; c0 < nl; c0 += 16) {
        uint32_t v[16];
        const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, "
            "%14, %15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(taddr));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (row < a.M) {
            float r[16];
#pragma unroll
            for (int q = 0; q < 16; ++q)
                r[q] = __uint_as_float(v[q]) * rs + ((a.bias && c0 + q < nl) ? __ldg(a.bias + n0 + c0 + q) : 0.0f);
            if (a.att_src) {
#pragma unroll
                for (int q = 0; q < 16; ++q) {
                    if (c0 + q >= nl) break;
                    const int hh = (n0 + c0 + q) / a.hc;
                    const float vs = r[q] * __ldg(a.att_src + n0 + c0 + q), vd = r[q] * __ldg(a.att_dst + n0 + c0 + q);
#pragma unroll
                    for (int h = 0; h < 8; ++h)
                        if (h == hh) { ps[h] += vs; pd[h] += vd; }
                }
            }
            float* y = a.Y + row * a.ldy + n0 + c0;
            if (vec && c0 + 16 <= nl) {
#pragma unroll
                for (int q = 0; q < 16; q += 4) *reinterpret_cast<float4*>(y + q) = make_float4(r[q], r[q + 1], r[q + 2], r[q + 3]);
            } else {
#pragma unroll
                for (int q = 0; q < 16; ++q)
                    if (c0 + q < nl) y[q] = r[q];
            }
        }
    }
    if (a.att_src && row < a.M) {
        for (int h = 0; h < a.heads; ++h) {
            a.s_src[row * a.heads + h] = ps[h];
            a.s_dst[row * a.heads + h] = pd[h];
        }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(a.tmem_cols));
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

}  // namespace xform

namespace {
// dinv[i] = deg_i^-1/2 with deg_i = the row length of the plan (in-degree incl. self-loops, Q7),
// computed in fp64 and rounded once; 0 for empty rows
// (source-blocked plans: deg = the total in-degree the plan keeps per row)
__global__ void deg_rsqrt_kernel(const int64_t* __restrict__ rowptr, const int32_t* __restrict__ deg, int64_t n,
                                 float* dinv) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t d = deg ? (int64_t)deg[i] : rowptr[i + 1] - rowptr[i];
        dinv[i] = d > 0 ? (float)(1.0 / sqrt((double)d)) : 0.0f;
    }
}
}  // namespace

pyg_status_t gcn_dinv(const int64_t* rowptr, const int32_t* deg, int64_t n, float* dinv, cudaStream_t s) {
    if (n <= 0) return PYG_OK;
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16));
    deg_rsqrt_kernel<<<blocks, 256, 0, s>>>(rowptr, deg, n, dinv);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

pyg_status_t dense_transform_impl(const float* X, int64_t M, int64_t K, int64_t ldx, const float* W, int64_t N,
                                  int64_t ldw, const float* bias, const float* row_scale, float* Y, int64_t ldy,
                                  cudaStream_t s, const float* att_src, const float* att_dst, float* s_src,
                                  float* s_dst, int heads) {
    using namespace xform;
    if (M == 0 || N == 0) return PYG_OK;
    if (!encode_fn()) return fail(PYG_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    Args a;
    a.M = M; a.K = K; a.N = (int)N;
    a.UN = (int)std::min<size_t>(256, align_up((size_t)N, 16));  // UMMA N per CTA; more columns -> grid.y
    a.tmem_cols = 32;
    while (a.tmem_cols < a.UN) a.tmem_cols <<= 1;
    a.kb = (int)cdiv(std::max<int64_t>(K, 1), kBK);
    a.Y = Y; a.ldy = ldy; a.bias = bias; a.row_scale = row_scale;
    a.att_src = att_src; a.att_dst = att_dst; a.s_src = s_src; a.s_dst = s_dst;
    a.heads = heads > 0 ? heads : 1;
    a.hc = (int)(N / a.heads);
    const int stage_bytes = kBM * kBK * 4 + a.UN * kBK * 4;
    // ~100 KB of stages per CTA so that two CTAs share an SM: one's epilogue (TMEM -> global)
    // overlaps the other's TMA / MMA main loop (measured: 1 CTA/SM with 6 stages ran at 2.7 TB/s)
    static const int budget_kb = [] {
        const char* e = getenv("PYG_XF_SMEM_KB");
        return e ? atoi(e) : 100;
    }();
    a.stages = std::max(2, std::min(8, (budget_kb * 1024) / stage_bytes));
    const int smem = a.stages * stage_bytes + 1024 + 8 * (2 * a.stages + 1) + 16;

    CUtensorMap mx, mw;
    {
        cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)M};
        cuuint64_t gstr[1] = {(cuuint64_t)ldx * 4};
        cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)kBM};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode_fn()(&mx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(X), gdim, gstr, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(PYG_ERR_CUDA, "tensor map for X failed (%d)", (int)r);
    }
    {
        cuuint64_t gdim[2] = {(cuuint64_t)K, (cuuint64_t)N};
        cuuint64_t gstr[1] = {(cuuint64_t)ldw * 4};
        cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)a.UN};
        cuuint32_t es[2] = {1, 1};
        CUresult r = encode_fn()(&mw, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(W), gdim, gstr, box, es,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(PYG_ERR_CUDA, "tensor map for W failed (%d)", (int)r);
    }
    PYG_CUDA(cudaFuncSetAttribute(tf32_gemm_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    const dim3 grid((unsigned)cdiv(M, kBM), (unsigned)cdiv(N, a.UN));
    if (att_src && grid.y > 1) return fail(PYG_ERR_UNSUPPORTED, "gat_transform: H*C <= 256");
    tf32_gemm_kernel<<<grid, kThreads, smem, s>>>(mx, mw, a);
    PYG_LAUNCHED();
    PYG_CUDA(cudaGetLastError());
    return PYG_OK;
}

}  // namespace pyg
