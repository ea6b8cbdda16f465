// segment_tma_red3.cu -- instantiation of the TMA gather4 segment-reduce kernels for the GAT
// alpha-weighted sum (kRedHeadW: SUM with the per-(edge, head) weight alpha[eid][c / C]).
#include "segment_tma.cuh"

namespace pyg {
namespace tma {
template pyg_status_t launch_nch<kRedHeadW>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
}  // namespace tma
}  // namespace pyg
