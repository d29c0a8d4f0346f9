// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (24,4,0,128).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_24_4_0_128 = Shape<24,4,0,128>;
template cudaError_t launch<S_24_4_0_128>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_24_4_0_128>(size_t);
template int stage_doubles<S_24_4_0_128>();
template int is_big<S_24_4_0_128>();
}  // namespace fastk
}  // namespace ocpqp
