// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (60,20,0,256).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_60_20_0_256 = Shape<60,20,0,256>;
template cudaError_t launch<S_60_20_0_256>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_60_20_0_256>(size_t);
template int stage_doubles<S_60_20_0_256>();
template int is_big<S_60_20_0_256>();
}  // namespace fastk
}  // namespace ocpqp
