// Probe of TMA tile::gather4 semantics on sm_100a (not part of the library).
// X [N x ld] fp32; tensor map 2D {cols=ld, rows=N}, box {BOX, 1}; one gather4 of rows r0..r3 at
// column c0 -> smem; compare with direct reads.
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

constexpr int BOX = 128;

__global__ void k(const __grid_constant__ CUtensorMap tmap, const int* rows, int c0, float* out) {
    __shared__ alignas(128) float buf[4 * BOX];
    __shared__ alignas(8) uint64_t bar;
    uint32_t sbar = (uint32_t)__cvta_generic_to_shared(&bar);
    uint32_t sbuf = (uint32_t)__cvta_generic_to_shared(buf);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(sbar));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(sbar), "r"(4 * BOX * 4));
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5, %6}], [%7];"
            :: "r"(sbuf), "l"(&tmap), "r"(c0), "r"(rows[0]), "r"(rows[1]), "r"(rows[2]), "r"(rows[3]), "r"(sbar)
            : "memory");
    }
    // wait phase 0
    asm volatile(
        "{\n .reg .pred p;\n WAIT:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n @!p bra WAIT;\n}\n" :: "r"(sbar));
    for (int i = threadIdx.x; i < 4 * BOX; i += blockDim.x) out[i] = buf[i];
}

int main() {
    const int N = 1000, F = 602, ld = 608;
    std::vector<float> h((size_t)N * ld);
    for (int r = 0; r < N; ++r) for (int c = 0; c < ld; ++c) h[(size_t)r * ld + c] = r * 1000.0f + c;
    float* d; cudaMalloc(&d, h.size() * 4); cudaMemcpy(d, h.data(), h.size() * 4, cudaMemcpyHostToDevice);
    EncodeFn enc = nullptr; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&enc, cudaEnableDefault, &q);
    if (!enc) { printf("no entry point\n"); return 1; }
    CUtensorMap tm;
    cuuint64_t gdim[2] = {(cuuint64_t)ld, (cuuint64_t)N};
    cuuint64_t gstr[1] = {(cuuint64_t)ld * 4};
    cuuint32_t box[2] = {BOX, 1};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, d, gdim, gstr, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    int hr[4] = {7, 999, 3, 512};
    int* dr; cudaMalloc(&dr, 16); cudaMemcpy(dr, hr, 16, cudaMemcpyHostToDevice);
    float* dout; cudaMalloc(&dout, 4 * BOX * 4);
    for (int c0 : {0, 480, 512}) {
        cudaMemset(dout, 0, 4 * BOX * 4);
        k<<<1, 128>>>(tm, dr, c0, dout);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<float> o(4 * BOX);
        cudaMemcpy(o.data(), dout, o.size() * 4, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int i = 0; i < 4; ++i) for (int c = 0; c < BOX; ++c) {
            float want = (c0 + c < ld) ? hr[i] * 1000.0f + c0 + c : 0.0f;
            if (o[i * BOX + c] != want) { if (bad < 5) printf("  mismatch row %d col %d got %f want %f\n", i, c, o[i*BOX+c], want); ++bad; }
        }
        printf("c0=%d err=%s bad=%d  sample %f %f %f\n", c0, cudaGetErrorString(e), bad, o[0], o[BOX], o[3*BOX+BOX-1]);
    }
    return 0;
}
