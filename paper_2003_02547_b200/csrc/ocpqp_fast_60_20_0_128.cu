// Explicit instantiation of the shaped kernel for (NX, NU, NG, TEAM) = (60,20,0,128).
#include "ocpqp_fast.cuh"

namespace ocpqp {
namespace fastk {
using S_60_20_0_128 = Shape<60,20,0,128>;
template cudaError_t launch<S_60_20_0_128>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int occupancy<S_60_20_0_128>(size_t);
template int stage_doubles<S_60_20_0_128>();
template int is_big<S_60_20_0_128>();
}  // namespace fastk
}  // namespace ocpqp
