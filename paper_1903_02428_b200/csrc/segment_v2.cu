// segment_v2.cu -- instantiation of the segment-reduce kernels for V = 2 floats per load
// (one translation unit per vector width so the library builds in parallel).
#include "segment_kernel.cuh"

namespace pyg {
namespace seg {
template pyg_status_t launch<2>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
}  // namespace seg
}  // namespace pyg
