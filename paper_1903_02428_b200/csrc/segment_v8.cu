// segment_v8.cu -- instantiation of the segment-reduce kernels for V = 8 floats per load
// (one translation unit per vector width so the library builds in parallel).
#include "segment_kernel.cuh"

namespace pyg {
namespace seg {
template pyg_status_t launch<8>(const SegArgs&, int, int, int, int, int, const HeavyArgs&, int, cudaStream_t);
}  // namespace seg
}  // namespace pyg
