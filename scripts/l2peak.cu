// l2peak.cu -- measured L2 -> SM read bandwidth on this B200, the roof of the source-blocked
// segment-reduce (each pass gathers rows of an L2-resident block of X).
//
//   stream : every warp reads consecutive 512-byte pieces of an L2-resident buffer (float4),
//            the plain L2 read bandwidth;
//   gather : the gather pattern of seg_kernel on Reddit rows -- a warp reads U random rows of
//            `row_floats` floats (row stride ld) with V-float loads (lane l: chunks l, l+32, ...);
//            rows are drawn by a hash of the position from a table of `rows` rows that fits in L2
//            (no index traffic); bytes = useful row bytes.  Variants U x V are swept too.
// Each kernel sweeps the resident CTAs per SM; the best is reported.  Prints one JSON line.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2peak l2peak.cu && ./l2peak
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                                              \
    do {                                                                                   \
        cudaError_t e = (x);                                                               \
        if (e != cudaSuccess) {                                                            \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));                        \
            return 1;                                                                      \
        }                                                                                  \
    } while (0)

__global__ void stream_kernel(const float4* __restrict__ buf, int64_t n4, int64_t reps, float* sink) {
    const int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t nt = (int64_t)gridDim.x * blockDim.x;
    float s = 0.f;
    for (int64_t r = 0; r < reps; ++r)
        for (int64_t i = tid; i < n4; i += nt) {
            const float4 v = __ldg(buf + i);
            s += v.x + v.y + v.z + v.w;
        }
    if (s == 123.456f) sink[tid] = s;
}

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ void ld8(float (&r)[8], const float* p) {
    asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=f"(r[0]), "=f"(r[1]), "=f"(r[2]), "=f"(r[3]), "=f"(r[4]), "=f"(r[5]), "=f"(r[6]), "=f"(r[7])
                 : "l"(p));
}

// U rows in flight per warp, V-float vectors (V = 8: 256-bit LDG.E.ENL2.256, V = 4: LDG.E.128)
template <int U, int V>
__global__ void gather_kernel(const float* __restrict__ X, int64_t ld, int row_floats, uint32_t rows,
                              int64_t n_gathers, float* sink) {
    constexpr int NCH = (608 / V + 31) / 32;  // chunks per lane for rows up to 608 floats
    const int lane = threadIdx.x & 31;
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    const int nchunk = (row_floats + V - 1) / V;
    float acc[NCH][V] = {};
    for (int64_t k0 = w * U; k0 < n_gathers; k0 += nw * U) {
        float v[U][NCH][V];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint32_t r = hash32((uint32_t)(k0 + u) * 2654435761u + 12345u) % rows;
            const float* row = X + (int64_t)r * ld;
#pragma unroll
            for (int c = 0; c < NCH; ++c) {
                if (lane + 32 * c < nchunk) {
                    if constexpr (V == 8) ld8(v[u][c], row + 8 * (lane + 32 * c));
                    else {
                        const float4 t = __ldg(reinterpret_cast<const float4*>(row) + lane + 32 * c);
                        v[u][c][0] = t.x; v[u][c][1] = t.y; v[u][c][2] = t.z; v[u][c][3] = t.w;
                    }
                }
            }
        }
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
            for (int c = 0; c < NCH; ++c)
                if (lane + 32 * c < nchunk)
#pragma unroll
                    for (int q = 0; q < V; ++q) acc[c][q] += v[u][c][q];
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int q = 0; q < V; ++q) s += acc[c][q];
    if (s == 123.456f) sink[w] = s;
}

typedef void (*gather_fn)(const float*, int64_t, int, uint32_t, int64_t, float*);

int main() {
    int dev = 0, sms = 0, l2 = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    CK(cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    // table = 0.4 x L2 (the source block size pyg_plan_suggest_col_block targets)
    const int ld = 608, row_floats = 602;
    const uint32_t rows = (uint32_t)((0.4 * l2) / (ld * 4.0));
    const size_t bytes = (size_t)rows * ld * 4;
    float *X = nullptr, *sink = nullptr;
    CK(cudaMalloc(&X, bytes));
    CK(cudaMalloc(&sink, (size_t)sms * 2048 * 4 * 8));
    CK(cudaMemset(X, 0, bytes));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    double best_stream = 0, best_gather = 0;
    int best_stream_b = 0, best_gather_b = 0;
    const char* best_variant = "";
    const int64_t n4 = (int64_t)(bytes / 16);
    const int64_t reps = 200;
    const int64_t n_gathers = 40LL * 1000 * 1000;
    for (int b = 1; b <= 8; ++b) {
        const int grid = sms * b;
        for (int it = 0; it < 2; ++it) {  // first run warms L2
            CK(cudaEventRecord(e0));
            stream_kernel<<<grid, 256>>>(reinterpret_cast<const float4*>(X), n4, reps, sink);
            CK(cudaEventRecord(e1));
            CK(cudaEventSynchronize(e1));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            const double gbs = (double)bytes * reps / (ms * 1e-3) / 1e9;
            if (it && gbs > best_stream) { best_stream = gbs; best_stream_b = b; }
        }
        const gather_fn fns[] = {gather_kernel<1, 8>, gather_kernel<2, 8>, gather_kernel<1, 4>, gather_kernel<2, 4>,
                                 gather_kernel<4, 4>};
        const char* names[] = {"U1V8", "U2V8", "U1V4", "U2V4", "U4V4"};
        for (int f = 0; f < 5; ++f)
            for (int it = 0; it < 2; ++it) {
                CK(cudaEventRecord(e0));
                fns[f]<<<grid, 256>>>(X, ld, row_floats, rows, n_gathers, sink);
                CK(cudaEventRecord(e1));
                CK(cudaEventSynchronize(e1));
                float ms = 0;
                CK(cudaEventElapsedTime(&ms, e0, e1));
                const double gbs = (double)n_gathers * row_floats * 4 / (ms * 1e-3) / 1e9;
                if (it && gbs > best_gather) { best_gather = gbs; best_gather_b = b; best_variant = names[f]; }
            }
    }
    CK(cudaGetLastError());
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d, \"table_bytes\": %zu, \"row_bytes\": %d, "
           "\"l2_stream_gbs\": %.1f, \"l2_stream_ctas_per_sm\": %d, \"l2_row_gather_gbs\": %.1f, "
           "\"l2_row_gather_ctas_per_sm\": %d, \"l2_row_gather_variant\": \"%s\", \"n_gathers\": %lld}\n",
           prop.name, sms, l2, bytes, row_floats * 4, best_stream, best_stream_b, best_gather, best_gather_b,
           best_variant, (long long)n_gathers);
    return 0;
}
