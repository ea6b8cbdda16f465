// segment_tma_red4.cu -- instantiation of the TMA gather4 segment-reduce kernels for SUM with the
// row-scale / blend / bias epilogue (kRedSumEpi: APPNP, the GCN layer), kept apart so the plain
// kernels keep their register count (54 vs 70 registers -> 4 vs 3 CTAs per SM).
#include "segment_tma.cuh"

namespace pyg {
namespace tma {
template pyg_status_t launch_nch<kRedSumEpi>(int, int, int64_t, int, int, cudaStream_t, const CUtensorMap&, const Args&);
}  // namespace tma
}  // namespace pyg
