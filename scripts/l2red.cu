// l2red.cu -- measured L2 atomic-reduction throughput on this B200: the roof of the atomic COO
// strategy once its column tiles keep the accumulation target in L2 (coo.cu l2_tile_cols; Reddit:
// 19 tiles of 32 columns, a 30 MB out slice + a 30 MB X slice per tile).
//
//   red        : groups of W/4 lanes issue red.global.add.v4.f32 (REDG.E.ADD.F32x4) into random
//                W-float rows of an L2-resident table (rows hashed from the position, no index
//                traffic); payload = W * 4 bytes per row;
//   gather_red : the COO kernel's per-edge pattern -- load a random W-float row of table A
//                (LDG.128 per lane) and red.global.add it into a random row of table B;
//   gather_red_ld608 : gather_red on 32-float slices of 608-float rows (a column tile of Reddit's
//                X / out: the same bytes over 19x the address range -- TLB reach);
//   bulk_red   : one lane per warp issues cp.reduce.async.bulk.global.shared::cta.add.f32 of a
//                W-float smem row into a random row (the TMA bulk-reduce engine instead of REDs).
// Tables: 233k rows (Reddit's N) x W floats.  Best over 1..8 CTAs of 256 threads per SM.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o l2red l2red.cu && ./l2red
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#define CK(x)                                                               \
    do {                                                                    \
        cudaError_t e = (x);                                                \
        if (e != cudaSuccess) {                                             \
            fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(e));         \
            return 1;                                                       \
        }                                                                   \
    } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
    x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
    return x;
}

__device__ __forceinline__ void red4(float* p, float a, float b, float c, float d) {
    asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a), "f"(b), "f"(c), "f"(d) : "memory");
}

template <int W>
__global__ void red_kernel(float* T, uint32_t rows, int64_t n, float v) {
    constexpr int L = W / 4;  // lanes per row
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / L;
    const int l = threadIdx.x % L;
    for (int64_t k = g; k < n; k += ng) {
        const uint32_t r = hash32((uint32_t)k * 2654435761u + 777u) % rows;
        red4(T + (int64_t)r * W + 4 * l, v, v, v, v);
    }
}

template <int W>
__global__ void gather_red_kernel(const float* __restrict__ A, float* B, uint32_t rows, int64_t n) {
    constexpr int L = W / 4;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / L;
    const int l = threadIdx.x % L;
    for (int64_t k = g; k < n; k += ng) {
        const uint32_t s = hash32((uint32_t)k * 2246822519u + 99u) % rows;
        const uint32_t r = hash32((uint32_t)k * 2654435761u + 777u) % rows;
        const float4 x = __ldg(reinterpret_cast<const float4*>(A + (int64_t)s * W) + l);
        red4(B + (int64_t)r * W + 4 * l, x.x, x.y, x.z, x.w);
    }
}

// the same pattern on W-float slices of rows `ld` floats apart (the atomic kernel's column tile of a
// wide row-major X / out: same bytes, spread over ld / W times the address range)
template <int W>
__global__ void gather_red_strided_kernel(const float* __restrict__ A, float* B, uint32_t rows, int64_t ld, int64_t n) {
    constexpr int L = W / 4;
    const int64_t g = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / L;
    const int64_t ng = ((int64_t)gridDim.x * blockDim.x) / L;
    const int l = threadIdx.x % L;
    for (int64_t k = g; k < n; k += ng) {
        const uint32_t s = hash32((uint32_t)k * 2246822519u + 99u) % rows;
        const uint32_t r = hash32((uint32_t)k * 2654435761u + 777u) % rows;
        const float4 x = __ldg(reinterpret_cast<const float4*>(A + (int64_t)s * ld) + l);
        red4(B + (int64_t)r * ld + 4 * l, x.x, x.y, x.z, x.w);
    }
}

template <int W>
__global__ void bulk_red_kernel(float* T, uint32_t rows, int64_t n) {
    __shared__ __align__(128) float buf[8][W];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int i = lane; i < W; i += 32) buf[warp][i] = 1.0f;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncwarp();
    const int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    if (lane == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(&buf[warp][0]);
        int inflight = 0;
        for (int64_t k = w; k < n; k += nw) {
            const uint32_t r = hash32((uint32_t)k * 2654435761u + 777u) % rows;
            asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;"
                         ::"l"(T + (int64_t)r * W), "r"(sa), "n"(W * 4) : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            if (++inflight == 16) {
                asm volatile("cp.async.bulk.wait_group.read 8;" ::: "memory");
                inflight = 8;
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
}

typedef void (*red_fn)(float*, uint32_t, int64_t, float);
typedef void (*gred_fn)(const float*, float*, uint32_t, int64_t);
typedef void (*bred_fn)(float*, uint32_t, int64_t);

template <typename F>
static double best_rate(int sms, F launch, double bytes_per_call, int* best_b) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double best = 0;
    for (int b = 1; b <= 8; ++b)
        for (int it = 0; it < 2; ++it) {
            cudaEventRecord(e0);
            launch(sms * b);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            const double gbs = bytes_per_call / (ms * 1e-3) / 1e9;
            if (it && gbs > best) { best = gbs; *best_b = b; }
        }
    return best;
}

int main() {
    int dev = 0, sms = 0;
    CK(cudaGetDevice(&dev));
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, dev));
    const uint32_t rows = 232965;
    const int64_t n = 40LL * 1000 * 1000;
    float *A = nullptr, *B = nullptr;
    CK(cudaMalloc(&A, (size_t)rows * 64 * 4));
    CK(cudaMalloc(&B, (size_t)rows * 64 * 4));
    CK(cudaMemset(A, 0, (size_t)rows * 64 * 4));
    CK(cudaMemset(B, 0, (size_t)rows * 64 * 4));
    printf("{\"gpu\": \"%s\", \"sms\": %d, \"rows\": %u, \"n\": %lld", prop.name, sms, rows, (long long)n);
    int bb = 0;
    double r;
    r = best_rate(sms, [&](int g) { red_kernel<32><<<g, 256>>>(B, rows, n, 1.0f); }, (double)n * 128, &bb);
    printf(", \"red_w32_gbs\": %.1f, \"red_w32_ctas\": %d", r, bb);
    r = best_rate(sms, [&](int g) { red_kernel<16><<<g, 256>>>(B, rows, n, 1.0f); }, (double)n * 64, &bb);
    printf(", \"red_w16_gbs\": %.1f, \"red_w16_ctas\": %d", r, bb);
    r = best_rate(sms, [&](int g) { red_kernel<64><<<g, 256>>>(B, rows, n, 1.0f); }, (double)n * 256, &bb);
    printf(", \"red_w64_gbs\": %.1f, \"red_w64_ctas\": %d", r, bb);
    r = best_rate(sms, [&](int g) { gather_red_kernel<32><<<g, 256>>>(A, B, rows, n); }, (double)n * 128, &bb);
    printf(", \"gather_red_w32_gbs\": %.1f, \"gather_red_w32_ctas\": %d", r, bb);
    {
        const int64_t ld = 608;  // Reddit's padded row: 19 column tiles of 32 floats
        float *SA = nullptr, *SB = nullptr;
        CK(cudaMalloc(&SA, (size_t)rows * ld * 4));
        CK(cudaMalloc(&SB, (size_t)rows * ld * 4));
        CK(cudaMemset(SA, 0, (size_t)rows * ld * 4));
        CK(cudaMemset(SB, 0, (size_t)rows * ld * 4));
        r = best_rate(sms, [&](int g) { gather_red_strided_kernel<32><<<g, 256>>>(SA, SB, rows, ld, n); },
                      (double)n * 128, &bb);
        printf(", \"gather_red_w32_ld608_gbs\": %.1f, \"gather_red_w32_ld608_ctas\": %d", r, bb);
        CK(cudaFree(SA));
        CK(cudaFree(SB));
    }
    r = best_rate(sms, [&](int g) { bulk_red_kernel<32><<<g, 256>>>(B, rows, n); }, (double)n * 128, &bb);
    printf(", \"bulk_red_w32_gbs\": %.1f, \"bulk_red_w32_ctas\": %d", r, bb);
    r = best_rate(sms, [&](int g) { bulk_red_kernel<64><<<g, 256>>>(B, rows, n); }, (double)n * 256, &bb);
    printf(", \"bulk_red_w64_gbs\": %.1f, \"bulk_red_w64_ctas\": %d", r, bb);
    CK(cudaGetLastError());
    printf("}\n");
    return 0;
}
