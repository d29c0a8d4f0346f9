// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (30,10,10,64).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_30_10_10_64 = Shape<30,10,10,64>;
template cudaError_t launch<S_30_10_10_64>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_30_10_10_64>(size_t);
template int stage_doubles<S_30_10_10_64>();
template int is_big<S_30_10_10_64>();
}  // namespace fastk
}  // namespace ocpqp
