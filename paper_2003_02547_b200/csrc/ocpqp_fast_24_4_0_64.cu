// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (24,4,0,64).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_24_4_0_64 = Shape<24,4,0,64>;
template cudaError_t launch<S_24_4_0_64>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_24_4_0_64>(size_t);
template int stage_doubles<S_24_4_0_64>();
template int is_big<S_24_4_0_64>();
}  // namespace fastk
}  // namespace ocpqp
