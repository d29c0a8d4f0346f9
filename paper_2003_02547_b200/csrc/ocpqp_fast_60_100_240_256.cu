// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (60,100,240,256).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_60_100_240_256 = Shape<60,100,240,256>;
template cudaError_t launch<S_60_100_240_256>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_60_100_240_256>(size_t);
template int stage_doubles<S_60_100_240_256>();
template int is_big<S_60_100_240_256>();
}  // namespace fastk
}  // namespace ocpqp
