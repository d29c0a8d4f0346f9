// Explicit instantiation of the row kernel for (NX, NU, NG, NB, G, WPB) = (24,4,0,28,32,1).
#include "ocpqp_row.cuh"

namespace ocpqp {
namespace rowk {
using R_24_4_0_28_32_1 = RShape<24,4,0,28,32,1>;
template cudaError_t row_launch<R_24_4_0_28_32_1>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int row_occupancy<R_24_4_0_28_32_1>(size_t);
template int row_team_tile<R_24_4_0_28_32_1>();
}  // namespace rowk
}  // namespace ocpqp
