// segment_v1.cu -- instantiation of the segment-reduce kernels for V = 1 floats per load
// (one translation unit per vector width so the library builds in parallel).
#include "segment_kernel.cuh"

namespace pyg {
namespace seg {
template pyg_status_t launch<1>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
}  // namespace seg
}  // namespace pyg
