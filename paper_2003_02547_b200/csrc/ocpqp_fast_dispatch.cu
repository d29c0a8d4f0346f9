// Dispatch table of the shaped kernel instantiations (ocpqp_fast_*.cu).
#include <cuda_runtime.h>

#include "ocpqp_internal.h"

namespace ocpqp {
namespace fastk {
template <int NX_, int NU_, int NG_, int TEAM_, int SM_>
struct Shape;
template <class S>
cudaError_t launch(const KParams& p, const SolveParams& sp, int grid, size_t smem, cudaStream_t st);
template <class S>
int occupancy(size_t smem);
template <class S>
int stage_doubles();
template <class S>
int is_big();
}  // namespace fastk
namespace rowk {
template <int NX_, int NU_, int NG_, int NB_, int G_, int WPB_>
struct RShape;
template <class S>
cudaError_t row_launch(const KParams& p, const SolveParams& sp, int grid, size_t smem, cudaStream_t st);
template <class S>
int row_occupancy(size_t smem);
template <class S>
int row_team_tile();
}  // namespace rowk

#define OCPQP_ROW_SHAPES(X) \
    X(8, 3, 0, 11, 8, 1)     \
    X(8, 3, 0, 11, 8, 2)     \
    X(24, 4, 0, 28, 32, 1)   \
    X(30, 10, 10, 40, 32, 1)

#define OCPQP_RMATCH(nx_, nu_, ng_, nb_, g_, w_)                                              \
    (s.kind == 1 && s.nx == (nx_) && s.nu == (nu_) && s.ng == (ng_) && s.nb == (nb_) &&     \
     s.team == (g_) && s.wpb == (w_))

#define OCPQP_FAST_SHAPES(X) \
    X(8, 3, 0, 32, 0)           \
    X(8, 3, 0, 64, 0)           \
    X(24, 4, 0, 64, 0)          \
    X(24, 4, 0, 128, 0)         \
    X(30, 10, 10, 128, 0)       \
    X(30, 10, 10, 64, 0)        \
    X(60, 20, 0, 256, 0)        \
    X(60, 20, 0, 128, 0)        \
    X(60, 100, 240, 256, 0)


#define OCPQP_MATCH(nx_, nu_, ng_, team_, sm_) \
    (s.kind == 0 && s.nx == (nx_) && s.nu == (nu_) && s.ng == (ng_) && s.team == (team_) && s.sm == (sm_))

bool fast_supported(const FastShape& s) {
#define X(a, b, c_, t, m) if (OCPQP_MATCH(a, b, c_, t, m)) return true;
    OCPQP_FAST_SHAPES(X)
#undef X
#define X(a, b, c_, nb, g, w) if (OCPQP_RMATCH(a, b, c_, nb, g, w)) return true;
    OCPQP_ROW_SHAPES(X)
#undef X
    return false;
}

int fast_teams_per_cta(const FastShape& s) { return s.kind == 1 ? (32 / s.team) * s.wpb : 1; }

int fast_stage_smem_doubles(const FastShape& s) {
#define X(a, b, c_, t, m) if (OCPQP_MATCH(a, b, c_, t, m)) return fastk::stage_doubles<fastk::Shape<a, b, c_, t, m>>();
    OCPQP_FAST_SHAPES(X)
#undef X
#define X(a, b, c_, nb, g, w) \
    if (OCPQP_RMATCH(a, b, c_, nb, g, w)) return rowk::row_team_tile<rowk::RShape<a, b, c_, nb, g, w>>();
    OCPQP_ROW_SHAPES(X)
#undef X
    return -1;
}

cudaError_t launch_fast_solve(const FastShape& s, const KParams& p, const SolveParams& sp, int grid,
                              size_t smem, cudaStream_t stream) {
#define X(a, b, c_, t, m) \
    if (OCPQP_MATCH(a, b, c_, t, m)) return fastk::launch<fastk::Shape<a, b, c_, t, m>>(p, sp, grid, smem, stream);
    OCPQP_FAST_SHAPES(X)
#undef X
#define X(a, b, c_, nb, g, w) \
    if (OCPQP_RMATCH(a, b, c_, nb, g, w))  \
        return rowk::row_launch<rowk::RShape<a, b, c_, nb, g, w>>(p, sp, grid, smem, stream);
    OCPQP_ROW_SHAPES(X)
#undef X
    return cudaErrorNotSupported;
}

int fast_big(const FastShape& s) {
#define X(a, b, c_, t, m) if (OCPQP_MATCH(a, b, c_, t, m)) return fastk::is_big<fastk::Shape<a, b, c_, t, m>>();
    OCPQP_FAST_SHAPES(X)
#undef X
    return 0;
}

int fast_occupancy(const FastShape& s, size_t smem) {
#define X(a, b, c_, t, m) if (OCPQP_MATCH(a, b, c_, t, m)) return fastk::occupancy<fastk::Shape<a, b, c_, t, m>>(smem);
    OCPQP_FAST_SHAPES(X)
#undef X
#define X(a, b, c_, nb, g, w) \
    if (OCPQP_RMATCH(a, b, c_, nb, g, w)) return rowk::row_occupancy<rowk::RShape<a, b, c_, nb, g, w>>(smem);
    OCPQP_ROW_SHAPES(X)
#undef X
    return 0;
}

}  // namespace ocpqp
