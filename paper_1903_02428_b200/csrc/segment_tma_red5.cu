// segment_tma_red5.cu -- instantiation of the TMA gather4 segment-reduce kernels for MAX of weighted
// messages (kRedMaxW); the plain PYG_MAX kernels skip the multiply and the scale loads.
#include "segment_tma.cuh"

namespace pyg {
namespace tma {
template pyg_status_t launch_nch<kRedMaxW>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
}  // namespace tma
}  // namespace pyg
