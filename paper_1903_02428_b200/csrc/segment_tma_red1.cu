// segment_tma_red1.cu -- instantiation of the TMA gather4 segment-reduce kernels for PYG_MEAN
// (one translation unit per reduction so the kernel variants of each compile in parallel).
#include "segment_tma.cuh"

namespace pyg {
namespace tma {
template pyg_status_t launch_nch<PYG_MEAN>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
}  // namespace tma
}  // namespace pyg
