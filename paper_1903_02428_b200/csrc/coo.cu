// coo.cu -- atomic COO scatter: the strategy of P:270-271 ("parallelization over
// *all* elements and making use of atomic operations") rebuilt for sm_100a.
//
//   * a group of `lpr` lanes walks a contiguous run of `epg` edges in input order,
//     fusing the gather of x_j and phi;
//   * equal consecutive targets are aggregated in registers and flushed with one
//     vector red.global.add.v{2,4}.f32 (REDG.E.ADD.F32x4) per run -- for
//     target-sorted ("coalesced") input this removes almost all atomics,
//     for unsorted input it degrades to one RED per element, which is the
//     paper's scheme ("GS is always fast, nevertheless of the input being
//     coalesced");
//   * MAX uses 64-bit atomicMax on a packed key (order-preserving value bits in
//     the high word, 0xffffffff - edge id in the low word), so the result is
//     deterministic and ties go to the lowest edge id (Q4) without a second pass
//     over the edges; the keys live in the caller's arg_out buffer and are
//     decoded in place.
#include "kernels.cuh"

namespace pyg {

namespace {

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
#pragma unroll
            for (int q = 0; q < V; ++q)
                if (q < nv && bi[ch][q] >= 0) atomicMax(kp + q, max_key(acc[ch][q], (uint32_t)bi[ch][q]));
        } else {
            float* op = a.out + cur * a.ldo + col;
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

    for (int64_t base = e0; base < e1; base += lpr) {
        const int n = (int)min((int64_t)lpr, e1 - base);
        long long mi = 0, mg = 0;
        float ms = 1.0f;
        if (l < n) {
            const int64_t p = base + l;
            mi = __ldg(a.sidx + p);
            mg = a.gidx ? __ldg(a.gidx + p) : p;
            if (a.w) ms = __ldg(a.w + p);
            if (a.gdeg) ms = ms / (float)__ldg(a.gdeg + mg);
        }
        int t = 0;
        for (; t + U <= n; t += U) {
            float v[U][NCH][V];
            float sv[U];
            long long iv[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const long long g = __shfl_sync(mask, mg, t + u, lpr);
                sv[u] = __shfl_sync(mask, ms, t + u, lpr);
                iv[u] = __shfl_sync(mask, mi, t + u, lpr);
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
            for (int u = 0; u < U; ++u) consume(iv[u], (int)(base + t + u), sv[u], v[u]);
        }
        for (; t < n; ++t) {
            const long long g = __shfl_sync(mask, mg, t, lpr);
            const float sc = __shfl_sync(mask, ms, t, lpr);
            const long long i = __shfl_sync(mask, mi, t, lpr);
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
            consume(i, (int)(base + t), sc, v);
        }
    }
    if (cur >= 0) flush<V, NCH, RED>(a, cur, l, lpr, c0, cv, acc, bi, out_vec_ok);
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

__global__ void degree_kernel(const int64_t* __restrict__ sidx, int64_t E, int32_t* deg, int32_t* first) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < E; k += (int64_t)gridDim.x * blockDim.x) {
        const int64_t i = sidx[k];
        if (deg) atomicAdd(deg + i, 1);
        if (first) atomicMin(first + i, (int32_t)k);
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

}  // namespace

pyg_status_t coo_reduce(const CooArgs& a, int reduce, cudaStream_t s) {
    if (a.n_out <= 0 || a.ncols <= 0) return PYG_OK;
    // zero the accumulation target (outputs are overwritten, Q14)
    if (reduce == PYG_MAX) {
        PYG_CUDA(cudaMemset2DAsync(a.keys, a.ldk * 8, 0, (size_t)a.ncols * 8, (size_t)a.n_out, s));
    } else {
        PYG_CUDA(cudaMemset2DAsync(a.out, a.ldo * 4, 0, (size_t)a.ncols * 4, (size_t)a.n_out, s));
    }
    if (a.E <= 0) return PYG_OK;
    int V = 1;
    for (int cand : {4, 2}) {
        const bool cols_ok = (a.ncols % cand == 0) || (a.allow_pad_read && cand == 4 &&
                                                       a.ldx >= (int64_t)align_up(a.ncols, 4));
        if (cols_ok && a.ldx % cand == 0 && aligned(a.X, 4 * cand)) { V = cand; break; }
    }
    const int ovk = (reduce != PYG_MAX) && (a.ldo % V == 0) && aligned(a.out, 4 * V);
    const int64_t nvec = cdiv(a.ncols, V);
    int lpr, nch, tiles;
    if (nvec <= 32) {
        lpr = 4;
        while (lpr < nvec) lpr <<= 1;
        nch = 1;
        tiles = 1;
    } else {
        lpr = 32;
        int64_t need = cdiv(nvec, 32);
        tiles = (int)cdiv(need, 16);
        need = cdiv(nvec, 32 * (int64_t)tiles);
        nch = 16;
        for (int c : kNch) if (c >= need) { nch = c; break; }
    }
    const int epg = lpr * 8;  // 8 batches of lpr edges per group
    switch (reduce) {
        case PYG_SUM:
        case PYG_MEAN: return launch_red<PYG_SUM>(a, V, nch, lpr, tiles, epg, ovk, s);
        default: return launch_red<PYG_MAX>(a, V, nch, lpr, tiles, epg, ovk, s);
    }
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
