// Internal plan / kernel-parameter structures shared by the C ABI layer and
// the sm_100a kernels.  Not part of the public ABI (include/ocpqp_b200.h).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ocpqp_b200.h"

// team kernel: factor store of P as the packed lower triangle (see Shape::PPACK)
#ifndef OCPQP_PPACK
#define OCPQP_PPACK 1
#endif

namespace ocpqp {

// Per-stage layout record, computed once per plan on the host.  The offsets
// reproduce the reference's flat layout (view.py:337-366 OcpView._build,
// view.py:108-129 ConBlock) so that kernel outputs are the reference vectors.
struct StageInfo {
    int nx, nu, nb, ng, ns;
    int nxn;      // nx[n+1] (0 at n == N)
    int nw, m, nc;
    int u_off, x_off;   // into v / y
    int pi_off;         // into pi (n < N)
    int c_off;          // into lam / t
    int s_off;          // into the flat slack vectors (sl part at nv + s_off)
    int ib_off;         // into the concatenated idxb
    int is_off;         // into the concatenated idxs
    int m_off;          // into per-row (box+general) work vectors, sum of m
    int foff[OCPQP_NUM_FIELDS];  // per-QP element offsets of each field
    // factor workspace offsets (doubles, per slot)
    int P_off, K_off, L_off;     // P[n] (nx^2), K[n] (nu*nx), L_uu[n] (nu^2)
    int pv_off, kff_off;         // pv[n] (nx), kff[n] (nu)
};

// Workspace buffers of one slot (one CTA solving one QP at a time).
enum WsBuf {
    WS_RG = 0, WS_RB, WS_RD,                 // residuals r_g (ny), r_b (ne), r_d (nc)
    WS_DVEC,                                 // d vector (nc), view.py:156-157, 184
    WS_ACT,                                  // activity as 0/1 doubles (nc)
    WS_AFF_Y, WS_AFF_PI, WS_AFF_LAM, WS_AFF_T,   // affine step
    WS_DIR_Y, WS_DIR_PI, WS_DIR_LAM, WS_DIR_T,   // combined step
    WS_GAM,                                  // raw gamma = lam/t (nc)
    WS_COEF,                                 // ge_lo + ge_up per row (sum m)
    WS_DL, WS_DU,                            // soft-slack augmented diagonals (ns_tot)
    WS_WALL,                                 // fold_rhs w_all (nc)
    WS_RTSL, WS_RTSU,                        // fold_rhs rt_sl / rt_su (ns_tot)
    WS_CROW,                                 // per-row fold coefficient (sum m)
    WS_ROWV,                                 // per-row values Jc w (sum m)
    WS_RHAT,                                 // reduced window rhs (nv)
    WS_P, WS_K, WS_L, WS_LP0,                // Riccati factor
    WS_PV, WS_KFF,                           // backward-sweep vectors
    WS_G,                                    // stage matrix G (nw_max^2)
    WS_T1,                                   // stage temp (max(nx' * nw, nx^2))
    WS_VEC,                                  // small stage vectors (4 * nw_max)
    WS_IY, WS_IPI, WS_ILAM, WS_IT,           // working iterate (shaped kernel)
    WS_RINV,                                 // 1 / L_ii of every stage factor and of L_P0
    WS_TINV,                                 // 1 / t on active slots (nc), per iteration
    // extended workspace (modes beyond speed; generic kernel only), allocated
    // on first use in a separate per-slot region (KParams::ws2)
    WS_LPS,                                  // L_P[n] per stage (nx^2, P_off layout)
    WS_HASLP,                                // per stage: 1.0 when L_P[n] is present (N+1)
    WS_MST,                                  // stage Hessian M~ (nw_max^2)
    WS_QR,                                   // QR stack ((nw_max + nx_max) * nw_max + nx_max^2)
    WS_RMD,                                  // materialised r_m of the refined direction (nc)
    WS_GF, WS_BF,                            // view.grad() (ny), view.b() (ne): absolute form
    WS_RFY, WS_RFPI, WS_RFLAM, WS_RFT,       // refinement residual
    WS_BY, WS_BPI, WS_BLAM, WS_BT,           // refinement best direction
    WS_ZT,                                   // L_P' x temporaries of the dpi pass (ne)
    WS_RHD,                                  // refinement rhs copy of r_d (nc, shaped kernel)
    WS_NUM
};
constexpr int WS_EXT0 = WS_LPS;              // first buffer of the extended workspace

struct KParams {
    // structure
    int N, B;
    int ny, ne, nc, nv, ns_tot, msum;
    int nw_max, nx_max, nu_max, m_max, nc_max, ns_max;
    const StageInfo* st;      // [N+1] device
    const int* idxb;          // concatenated, device
    const int* idxs;          // concatenated, device
    const int* var_box;       // [nv] box row (within stage) targeting variable, or -1
    const int* row_slack;     // [msum] soft slack index (within stage) of a row, or -1
    // data
    const double* f[OCPQP_NUM_FIELDS];
    long long bs[OCPQP_NUM_FIELDS];
    // workspace
    double* ws;               // slots * ws_slot doubles
    long long ws_slot;        // doubles per slot
    double* ws2;              // extended workspace: slots * ws2_slot doubles (nullptr = none)
    long long ws2_slot;
    int ws_off[WS_NUM];       // offsets within a slot
    unsigned long long smem_mask;  // bit b set: buffer b lives in shared memory
    int smem_off[WS_NUM];     // offsets within dynamic smem (doubles)
    int* counter;             // dynamic QP scheduler
    // dispatch hint (team kernel, opt-in): `order` lists the QPs by the previous solve's
    // iteration count, slowest first; its first n_first entries go to the CTAs that find
    // themselves alone on their SM (hint_ctr: [0] / [1] list cursors, [2 + smid] CTAs per SM),
    // prev_iters receives this solve's counts for the next one (nullptr = off)
    const int* order; int n_first; int* hint_ctr; int* prev_iters;
    // shaped-kernel structure (uniform stages 0..N-1, terminal stage N)
    int NB, NBN, NGN;         // box rows (n < N), box / general rows at N
    int box_ident;            // 1: every stage's idxb is 0..nb-1 (box row i bounds variable i)
    int stage_smem;           // doubles: offset of the per-stage scratch / per-team tile
    int team_stride;          // doubles of shared memory per team (row kernel)
    long long* dbg;           // optional [B, DBG_NUM] phase-cycle counters (nullptr = off)
    const double* ba;         // shaped kernels: packed [B A] per stage (NX x NW), see
    long long ba_bs;          //   launch_pack_ba; per-QP stride (0: one copy for the batch)
    long long ba_ns;          //   per-stage stride (0: the kernel's default, QP-major packing)
    int* esc_count;           // shaped kernel, balance mode: QPs left to the generic kernel
    int* esc_list;            //   (count, [B] indices); nullptr = none
    long long* esc_meta;      //   [B, 3]: iteration, flops, alpha_last bits at the escape;
                              //   the generic kernel resumes the loop there
    const int* sinv;          // shaped kernels: bit f set = field f (A..r) identical in every
                              // stage it is read at (device word, nullptr = none)
};

// phase ids of the optional clock64 instrumentation (KParams::dbg)
enum DbgPhase { DBG_RES = 0, DBG_FACTOR, DBG_SOLVE_AFF, DBG_SOLVE_DIR, DBG_STEP, DBG_TOTAL,
                DBG_ITERS, DBG_SPARE,
                // sub-phases (team kernel): factor stage parts, solve parts
                DBG_F_T1, DBG_F_G, DBG_F_CHOL, DBG_F_K, DBG_F_P, DBG_S_PRE, DBG_S_BWD, DBG_S_FWD,
                // free slots for finer diagnostics (OCPQP_XTICK, -DOCPQP_XDIAG builds)
                DBG_X0, DBG_X1, DBG_X2, DBG_X3, DBG_X4, DBG_X5, DBG_X6, DBG_X7,
                DBG_NUM = 24 };
// phase slots a kernel keeps per QP: the diagnostic slots only in -DOCPQP_XDIAG builds (the
// accumulators live in the CTA's static shared memory; the buffer stride stays DBG_NUM)
#ifdef OCPQP_XDIAG
constexpr int DBG_KEPT = DBG_NUM;
#else
constexpr int DBG_KEPT = DBG_X0;
#endif

struct SolveParams {
    OcpIpmArgC arg;
    double* y; double* pi; double* lam; double* t;
    int32_t* status; int32_t* iters; double* res; long long* flops; double* trace;
};

// launchers (ocpqp_ipm.cu)
cudaError_t launch_ipm_solve(const KParams& p, const SolveParams& sp, int grid, int threads,
                             size_t smem, cudaStream_t stream);
cudaError_t launch_newton_step(const KParams& p, double reg, const double* lam, const double* t,
                               const double* rg, const double* rb, const double* rd,
                               const double* rm, double* sy, double* spi, double* slam,
                               double* st, int* fail, int grid, int threads, cudaStream_t stream);
cudaError_t launch_residuals(const KParams& p, const double* y, const double* pi,
                             const double* lam, const double* t, double* rg, double* rb,
                             double* rd, double* rm, double* norms, int grid, int threads,
                             cudaStream_t stream);
cudaError_t launch_shift_guess(const KParams& p, const double* sy, const double* spi,
                               const double* slam, const double* st, double* gy, double* gpi,
                               double* glam, double* gt, int grid, int threads,
                               cudaStream_t stream);
int ipm_occupancy(int threads, size_t smem);
// Pack [B A] of every stage (uniform stages 0..N-1) into out: per QP N * nx * (nu + nx)
// doubles, QP stride out_bs (0 when A and B are both broadcast); trans: each
// stage stored as [B A]' (nu + nx rows of nx), the BIG shapes' layout.
cudaError_t launch_pack_ba(const double* A, long long bsA, const double* B, long long bsB, int Bn,
                           int N, int nx, int nu, double* out, long long out_bs, cudaStream_t stream,
                           int trans = 0, int stage_major = 0);
// Stage-invariance detection of the broadcast fields A..r (uniform-stage plans):
// writes the bit mask consumed by the shaped kernels to *mask.
cudaError_t launch_stage_invariant(const double* const* f, const long long* bs, int N, int nx,
                                   int nu, int* mask, cudaStream_t stream);

// Shaped (compile-time NX, NU, NG, TEAM) fused kernel, ocpqp_fast.cu.  Returns
// cudaErrorNotSupported when no instantiation matches.
// kind 0: team kernel (ocpqp_fast.cuh), one CTA of `team` threads per QP;
// kind 1: row kernel (ocpqp_row.cuh), `team` lanes per QP, `wpb` warps per CTA.
struct FastShape {
    int kind, nx, nu, ng, nb, team, wpb;
    int sm = 0;  // team kernel: factor store + sweep vectors at fixed shared-memory offsets
};
int fast_teams_per_cta(const FastShape& s);
bool fast_supported(const FastShape& s);
int fast_stage_smem_doubles(const FastShape& s);
cudaError_t launch_fast_solve(const FastShape& s, const KParams& p, const SolveParams& sp,
                              int grid, size_t smem, cudaStream_t stream);
int fast_occupancy(const FastShape& s, size_t smem);
// the shape's kernel streams stage data by TMA from a transposed [B A] pack
// and keeps no workspace buffer in shared memory (ocpqp_fast.cuh, Shape::BIG)
int fast_big(const FastShape& s);
// message of the calling thread's last error (ocpqp_last_error)
void set_last_error(const char* msg);

}  // namespace ocpqp
