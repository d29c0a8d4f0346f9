// Explicit instantiation of the row kernel for (NX, NU, NG, NB, G, WPB) = (8,3,0,11,8,2).
#include "ocpqp_row.cuh"

namespace ocpqp {
namespace rowk {
using R_8_3_0_11_8_2 = RShape<8,3,0,11,8,2>;
template cudaError_t row_launch<R_8_3_0_11_8_2>(const KParams&, const SolveParams&, int, size_t, cudaStream_t);
template int row_occupancy<R_8_3_0_11_8_2>(size_t);
template int row_team_tile<R_8_3_0_11_8_2>();
}  // namespace rowk
}  // namespace ocpqp
