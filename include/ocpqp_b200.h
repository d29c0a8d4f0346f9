/*
 * ocpqp_b200.h -- C ABI of the B200-native batched OCP-QP interior-point solver.
 *
 * This is the drop-in boundary for the reference's OCP-QP solve path
 * (/root/reference/pkg/src/mpcqp).  The reference is a pure-Python package, so
 * it has no FFI of its own; every entry point below names the Python call it
 * replaces (file:line), and INTEGRATION.md shows the ctypes stub a maintainer
 * adds to the reference to route `solve_ocp_qp` through this library.
 *
 * Conventions
 *   - plain pointers and sizes only; no torch / C++ types cross the boundary;
 *   - all arithmetic is fp64; integers are int32 (indices) / int64 (strides);
 *   - a "plan" is created once per (dims, idxb, idxs, batch) on the current
 *     CUDA device and owns the device workspace; its calls run on that device
 *     whatever the caller's current device.  A speed-mode solve never
 *     allocates; the first solve in another mode (refinement, QR, square-root,
 *     absolute form) allocates the plan's extended workspace once.  One solve
 *     per plan may be in flight: solves on one plan are ordered on their
 *     streams by the caller (use one plan per concurrent stream);
 *   - functions return 0 on success and a negative OCPQP_E_* code on misuse or
 *     CUDA error (ocpqp_last_error() gives the message).  Numerical trouble is
 *     never an error: it is a per-QP status word, as in the reference
 *     (solver.py:18-20, ipm_core.py:56-63).
 *
 * Data layout ("packed batch"): each stage-data field of the reference catalog
 * (qp_data.py:248-270 plus A, B, b of :329-336) is one fp64 array holding, per
 * QP, all stages back to back in canonical order (stage 0..N; matrices
 * row-major; dynamics fields only for stages 0..N-1).  QP i's copy starts at
 * ptr[f] + i * batch_stride[f]; batch_stride 0 broadcasts one copy to the whole
 * batch (e.g. the shared plant of the mass-spring benchmarks).  Per-stage sizes:
 *   A nx[n+1]*nx[n]   B nx[n+1]*nu[n]   b nx[n+1]      (n < N only)
 *   Q nx*nx  S nu*nx  R nu*nu  q nx  r nu
 *   lb ub nb   C ng*nx  D ng*nu  lg ug ng
 *   Zl Zu zl zu sl_lb su_lb ns   maskl masku nb+ng
 * idxb/idxs are structural and shared by the whole batch (they are part of the
 * plan).  A NULL field pointer means "all zeros" for matrices and vectors,
 * "all ones" for masks and "-inf / +inf" for lower / upper bounds, i.e. the
 * reference's zero-initialised stage (qp_data.py:221-245).
 *
 * Iterate / solution layout: exactly the reference's flat vectors
 * (view.py:3-13): y = [v | sl | su] with v = (u_0, x_0, u_1, x_1, ...),
 * pi = (pi_0 .. pi_{N-1}), lam/t per stage [lower m | upper m | slack-lower ns |
 * slack-upper ns] with m = nb + ng.  Batched as [B, ny], [B, ne], [B, nc], [B, nc].
 */
#ifndef OCPQP_B200_H
#define OCPQP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define OCPQP_ABI_VERSION 2

/* error codes */
#define OCPQP_OK 0
#define OCPQP_E_INVALID_DIM (-1)      /* maps to mpcqp InvalidDim (errors.py:18) */
#define OCPQP_E_DIMENSION (-2)        /* DimensionMismatch (errors.py:14) */
#define OCPQP_E_UNSUPPORTED (-3)      /* option outside the implemented modes */
#define OCPQP_E_CUDA (-4)             /* CUDA runtime error */
#define OCPQP_E_ARG (-5)              /* bad argument / NULL pointer */
#define OCPQP_E_CONDENSE (-6)         /* CondenseError (errors.py; condensing.py:180-185) */
#define OCPQP_E_NOT_PD (-7)           /* NotPositiveDefinite (linalg.py:110-113) */
#define OCPQP_E_RANK (-8)             /* RankDeficient (linalg.py:181-184) */

/* per-QP status words; values 0..4 mirror ipm_core.Status (ipm_core.py:56-63) */
#define OCPQP_STATUS_SUCCESS 0
#define OCPQP_STATUS_MAXITER 1
#define OCPQP_STATUS_MINSTEP 2
#define OCPQP_STATUS_NAN 3
#define OCPQP_STATUS_FAILURE 4
/* reference raises NonPositiveIterate (kkt_common.py:70-71) / SingularSlackBlock
 * (kkt_common.py:84-87) out of the solve; the library reports them per QP */
#define OCPQP_STATUS_NONPOSITIVE_ITERATE 5
#define OCPQP_STATUS_SINGULAR_SLACK 6
/* reference raises RankDeficient (linalg.py:180-184) out of the solve when the
 * QR array algorithm meets a rank-deficient stage stack outside the per-stage
 * fallback (kkt_ocp.py:174-191 with use_qr) */
#define OCPQP_STATUS_RANK_DEFICIENT 7

/* stage-data field ids (reference catalog qp_data.py:248-270, :329-336) */
enum OcpQpField {
    OCPQP_F_A = 0,
    OCPQP_F_B,
    OCPQP_F_b,
    OCPQP_F_Q,
    OCPQP_F_S,
    OCPQP_F_R,
    OCPQP_F_q,
    OCPQP_F_r,
    OCPQP_F_lb,
    OCPQP_F_ub,
    OCPQP_F_C,
    OCPQP_F_D,
    OCPQP_F_lg,
    OCPQP_F_ug,
    OCPQP_F_Zl,
    OCPQP_F_Zu,
    OCPQP_F_zl,
    OCPQP_F_zu,
    OCPQP_F_sl_lb,
    OCPQP_F_su_lb,
    OCPQP_F_maskl,
    OCPQP_F_masku,
    OCPQP_NUM_FIELDS
};

/* Stage dimensions; replaces OcpQpDim (qp_data.py:65-111) plus the structural
 * index sets idxb / idxs of every stage (qp_data.py:254, :261).  All arrays are
 * host memory; nx..ns have N+1 entries, idxb has sum(nb), idxs sum(ns). */
typedef struct OcpQpDimC {
    int32_t N;
    const int32_t* nx;
    const int32_t* nu;
    const int32_t* nb;
    const int32_t* ng;
    const int32_t* ns;
    const int32_t* idxb;
    const int32_t* idxs;
} OcpQpDimC;

/* Packed batch of QP data (see layout above). */
typedef struct OcpQpDataC {
    const double* ptr[OCPQP_NUM_FIELDS];
    int64_t batch_stride[OCPQP_NUM_FIELDS];
} OcpQpDataC;

/* IpmArg (ipm_core.py:66-128).  The leading block is what the speed-mode loop
 * reads; the trailing block (ABI version 2) selects the other modes of
 * mode_preset (ipm_core.py:131-168): square-root Riccati, QR array algorithm,
 * iterative refinement and the absolute formulation.  Unused: reg_dual (not
 * applied on the OCP backend, kkt_ocp.py:39-41) and kkt_method (dense QPs). */
typedef struct OcpIpmArgC {
    int32_t iter_max;
    int32_t pred_corr;       /* bool */
    int32_t cond_pred_corr;  /* bool */
    int32_t warm_start;      /* 0 none, 1 primal, 2 primal_dual */
    double alpha_min;
    double mu0;
    double tol_stat;
    double tol_eq;
    double tol_ineq;
    double tol_comp;
    double reg_prim;
    double lam_min;
    double t_min;
    double t0;
    double corr_ratio;
    double ftb;
    /* ABI v2: modes beyond speed */
    int32_t itref_pred_max;   /* refinement steps on the prediction */
    int32_t itref_corr_max;   /* refinement steps on the combined direction */
    int32_t use_qr_fallback;  /* bool: per-stage / whole-factor QR retry */
    int32_t use_qr_always;    /* bool: every factor by the QR array algorithm */
    int32_t riccati_variant;  /* 0 classical, 1 square_root */
    int32_t abs_form;         /* bool: absolute formulation (speed_abs) */
    int32_t comp_res_pred;    /* bool: residuals every iteration */
    int32_t mu_only_exit;     /* bool: exit test on mu only (mode speed_abs, ipm_core.py:303-304) */
    double itref_stop_ratio;
    double qr_fallback_ratio;
} OcpIpmArgC;

/* Primal-dual point, batched: y [B,ny], pi [B,ne], lam [B,nc], t [B,nc].
 * Replaces QpSolution (view.py:568-672). */
typedef struct OcpIterC {
    double* y;
    double* pi;
    double* lam;
    double* t;
} OcpIterC;

/* Per-QP outcome; replaces SolverStats (ipm_core.py:186-198) and the final
 * QpResiduals norms (view.py:675-695).  trace may be NULL; otherwise it is
 * [B, iter_max, 8] = (alpha_aff, alpha, mu, sigma, res_g, res_b, res_d, res_m)
 * per iteration, the IterRecord fields (ipm_core.py:171-184). */
typedef struct OcpStatsC {
    int32_t* status;      /* [B] OCPQP_STATUS_* */
    int32_t* iterations;  /* [B] */
    double* res;          /* [B,5] res_g, res_b, res_d, res_m, mu */
    int64_t* flops;       /* [B] nominal flops, linalg.py:41-78 counting rules */
    double* trace;        /* [B, iter_max, 8] or NULL */
} OcpStatsC;

/* Layout sizes of one QP: out[0..5] = ny, ne, nc, nv, ns_tot, n_act_max (=nc),
 * out[6 + f] = per-QP element count of field f (OCPQP_NUM_FIELDS entries).
 * Mirrors make_view / OcpView._build (view.py:337-366, :551-565). */
int ocpqp_layout(const OcpQpDimC* dim, int64_t* out, int32_t out_len);

typedef struct OcpPlan OcpPlan;

/* Create a plan for `batch` QPs of identical structure.  Validates the dims
 * like OcpQpDim.__init__ (qp_data.py:82-111) and the index sets like
 * validate() (qp_data.py:528-533). */
int ocpqp_plan_create(const OcpQpDimC* dim, int32_t batch, OcpPlan** out);
int ocpqp_plan_destroy(OcpPlan* plan);

/* Batched `solve_ocp_qp(qp, arg, guess)` (solver.py:103-105, loop
 * solver.py:180-308) over device-resident data.  `iter` holds the warm-start
 * guess on entry when arg->warm_start != 0 and the solution on exit.
 * Stream-ordered on `stream` (a cudaStream_t; NULL = legacy default stream).
 * Stage shapes whose kernel streams stage data by TMA (nx >= 48, box rows
 * only, ocpqp_plan_info) need Q, S, R, q, r, b 16-byte aligned with even batch
 * strides (cudaMalloc'd / torch buffers are); misaligned data is OCPQP_E_ARG. */
int ocpqp_solve(OcpPlan* plan, const OcpQpDataC* data, const OcpIpmArgC* arg,
                OcpIterC* iter, OcpStatsC* stats, void* stream);

/* Same as ocpqp_solve with HOST buffers: copies data in, solves and copies the
 * solution and stats out, then synchronizes `stream`.  This is the call an FFI
 * binding of the reference makes with numpy arrays.  When every result buffer
 * is page-locked (cudaHostAlloc / cudaHostRegister, e.g. torch pin_memory) and
 * no trace / warm start is requested, the kernel writes each QP's solution and
 * statistics straight into them as the QP finishes (mapped host memory), so
 * the transfer overlaps the QPs still iterating; pageable buffers go through
 * device staging and a copy after the solve. */
int ocpqp_solve_host(OcpPlan* plan, const OcpQpDataC* host_data,
                     const OcpIpmArgC* arg, OcpIterC* host_iter,
                     OcpStatsC* host_stats, void* stream);

/* Residuals of a batch of points; replaces compute_residuals / residuals
 * (view.py:698-706, :272-288).  r_* may be NULL (norms only); norms is
 * [B,5] = res_g, res_b, res_d, res_m, mu.  Device pointers. */
int ocpqp_residuals(OcpPlan* plan, const OcpQpDataC* data, const OcpIterC* point,
                    double* r_g, double* r_b, double* r_d, double* r_m,
                    double* norms, void* stream);

/* Newton step: classical riccati_factor(qp, iterate, arg) followed by
 * RiccatiFactor.solve(r_g, r_b, r_d, r_m) (kkt_ocp.py:142-201, :254-320).
 * reg is the primal regularisation (IpmArg.reg_prim).  fail_stage[B] receives
 * -1 on success or the FactorizationFailed.stage of the reference
 * (kkt_ocp.py:180-200); the step of a failed QP is left as zeros.
 * Device pointers. */
int ocpqp_newton_step(OcpPlan* plan, const OcpQpDataC* data, double reg,
                      const OcpIterC* iterate, const double* r_g,
                      const double* r_b, const double* r_d, const double* r_m,
                      OcpIterC* step, int32_t* fail_stage, void* stream);

/* Cost-to-go matrices P[n] and gains K[n] of the last classical factor of
 * ocpqp_newton_step for QP `qp` (RiccatiFactor.p_matrix / feedback_gains,
 * kkt_ocp.py:122-125, :323-330).  P_out: sum nx[n]^2, K_out: sum nu[n]*nx[n],
 * stage-major row-major, host memory. */
int ocpqp_factor_export(OcpPlan* plan, int32_t qp, double* P_out, double* K_out);

/* One-stage shift of a batch of solutions into the warm-start guesses of the
 * next closed-loop MPC solve; replaces mass_spring._shift_guess
 * (mass_spring.py:152-195): stage n takes stage n+1's x, u, pi, lam, t, the
 * last input repeats, the terminal state is rolled through the last dynamics,
 * and the stage-0 initial-state multipliers are rebuilt from the stage-0
 * stationarity gap.  Needs equal state dimensions over the horizon.  Device
 * pointers; `guess` must not alias `sol`. */
int ocpqp_shift_guess(OcpPlan* plan, const OcpQpDataC* data, const OcpIterC* sol,
                      OcpIterC* guess, void* stream);

/* Dispatch hint of the team kernel (off by default; OCPQP_DISPATCH_HINT=1 turns
 * it on at plan creation).  With it a solve hands out its QPs in the order of
 * the plan's PREVIOUS solve's iteration counts, slowest first, and the CTAs
 * that find themselves alone on their SM take the slowest ones: a QP alone on
 * an SM runs ~20 % faster per iteration, and a launch ends with its slowest
 * QP.  Meant for repeated solves of similar batches (closed-loop MPC, where
 * consecutive iteration counts correlate); the first solve after enabling
 * runs unhinted; results are identical with and without it. */
int ocpqp_plan_dispatch_hint(OcpPlan* plan, int32_t on);

/* Plan introspection: out[0..4] = threads per CTA, resident CTA slots,
 * dynamic shared memory bytes per CTA, shared-memory buffer mask, workspace
 * doubles per slot; out[5] kernel kind (0 generic, 1 team, 2 row), out[6]
 * lanes per QP, out[7] grid; out[8] (if out_len >= 9) 1 when the team kernel
 * keeps its factor store at fixed shared-memory offsets. */
int ocpqp_plan_info(const OcpPlan* plan, int64_t* out, int32_t out_len);

/* ---- dense QPs with equality constraints (reference DenseQp,
 * qp_data.py:426-500; solve_dense_qp, solver.py:98-100; kkt_dense.py:117-256) ----
 * min 1/2 v'Hv + g'v s.t. A v = b, lb <= v[idxb] <= ub, lg <= C v <= ug.
 * Dense QPs without equality rows run through ocpqp_solve as the N = 0
 * OCP-QP (see ocpqp_fc_create); these entry points handle ne > 0 with the
 * reference's two equality methods: kkt_method 0 = "schur" (Schur complement
 * A Hred^-1 A' + reg_dual I), 1 = "null_space" (Householder QR of A',
 * reduced Hessian on the null-space basis).  Speed-mode loop (predictor-
 * corrector, regularised factor retry); no soft rows. */
typedef struct OcpDensePlan OcpDensePlan;
typedef struct {
    int32_t nv, ne, nb, ng, ns;   /* ns must be 0 */
    const int32_t* idxb;          /* [nb] host, strictly increasing (NULL: 0..nb-1) */
} OcpDenseDimC;
typedef struct {
    /* device pointers, per QP: H nv*nv, g nv, A ne*nv, b ne, lb ub nb, C ng*nv,
     * lg ug ng, maskl masku nb+ng (row-major); NULL = the reference's zero-
     * initialised value (0, -inf / +inf bounds, all-one masks) */
    const double* H; const double* g; const double* A; const double* b;
    const double* lb; const double* ub; const double* C; const double* lg; const double* ug;
    const double* maskl; const double* masku;
    int64_t batch_stride[11];     /* same order; 0 broadcasts one copy */
} OcpDenseDataC;
int ocpqp_dense_plan_create(const OcpDenseDimC* dim, int32_t batch, int32_t kkt_method,
                            OcpDensePlan** out);
int ocpqp_dense_plan_destroy(OcpDensePlan* plan);
/* iter: y = v [B, nv], pi [B, ne], lam / t [B, 2 (nb + ng)] (lower rows, then
 * upper rows); stats as ocpqp_solve; reg_dual = IpmArg.reg_dual (Schur path). */
int ocpqp_dense_solve(OcpDensePlan* plan, const OcpDenseDataC* data, const OcpIpmArgC* arg,
                      double reg_dual, OcpIterC* iter, OcpStatsC* stats, void* stream);

/* ---- partial condensing (reference condensing.py:451-619) ----
 * A partial-condensing plan holds the block structure and the row routing of
 * partial_condense(qp, N1) for one (dims, idxb) structure; the arithmetic is
 * batched on the device. */
typedef struct OcpPcPlan OcpPcPlan;

/* partial_condense block structure (condensing.py:451-550). */
int ocpqp_pc_create(const OcpQpDimC* dim, int32_t N1, OcpPcPlan** out);
int ocpqp_pc_destroy(OcpPcPlan* plan);

/* Dimensions of the condensed QP; returns N2 = ceil(N / N1).  Non-NULL arrays
 * receive N2+1 entries (nx, nu, nb, ng) and the concatenated new idxb. */
int ocpqp_pc_dims(const OcpPcPlan* plan, int32_t* nx, int32_t* nu, int32_t* nb, int32_t* ng,
                  int32_t* idxb);

/* Condense a device batch of B QPs (`in`: every field present) into `out`
 * (device, every field per QP, batch stride = condensed field length).
 * Replaces partial_condense (condensing.py:451-550) for the whole batch. */
int ocpqp_pc_condense(OcpPcPlan* plan, int32_t B, const OcpQpDataC* in, OcpQpDataC* out,
                      void* stream);

/* Expand condensed solutions back to the full horizon (partial_expand,
 * condensing.py:553-619); device pointers. */
int ocpqp_pc_expand(OcpPcPlan* plan, int32_t B, const OcpQpDataC* in, const OcpIterC* short_sol,
                    OcpIterC* full_sol, void* stream);

/* ---- full condensing (reference condense / expand_solution,
 * condensing.py:160-429) ----
 * The plan of condense(qp, keep_x0): one block over stages 0..N (terminal
 * included).  keep_x0 = 0 drops x0: every component must be fixed by a
 * stage-0 box row (fix_row[j] fixes component fix_comp[j], nfix entries, as
 * _detect_fixed_x0 finds them, condensing.py:97-118), else OCPQP_E_CONDENSE.
 * The dense QP (ne = 0) is produced as a single-stage OCP-QP with N = 0,
 * nx = 0, nu = nv: R = H, r = g, D = C, idxb = dense idxb -- the IPM kernels
 * solve that form exactly like the reference's dense backend
 * (solve_dense_qp, solver.py:98-100).  ocpqp_pc_dims / _condense / _expand /
 * _destroy take this plan too (N2 = 0; expansion = expand_solution). */
int ocpqp_fc_create(const OcpQpDimC* dim, int32_t keep_x0, int32_t nfix, const int32_t* fix_row,
                    const int32_t* fix_comp, OcpPcPlan** out);

/* Cost recursion of a full-condensing plan: 0 = classical (default), 1 = the
 * square-root recursion of condense(variant="square_root") (condensing.py:
 * 134-146: U_n = qr_cholesky([chol(Q_n)'; U_{n+1} A]), P_n = U_n' U_n,
 * Y_n = (U A)' (U B) + S').  With it ocpqp_pc_condense reads one status word
 * back per call and returns OCPQP_E_NOT_PD / OCPQP_E_RANK where the reference
 * raises NotPositiveDefinite / RankDeficient. */
int ocpqp_pc_set_variant(OcpPcPlan* plan, int32_t square_root);

/* Soft rows of the condensed QP (partial or full plan): ns (N2+1 entries)
 * and the concatenated new idxs when non-NULL; returns sum(ns).  Slack data
 * (Zl Zu zl zu sl_lb su_lb) travels with its row (condensing.py:289-334). */
int ocpqp_pc_soft(const OcpPcPlan* plan, int32_t* ns, int32_t* idxs);

const char* ocpqp_pc_last_error(void);

/* fp64 peak microbenchmarks (roofline denominators): DFMA and DMMA
 * (mma.sync.m8n8k4.f64) throughput of the current device in TFLOP/s. */
int ocpqp_fp64_peak(double* dfma_tflops, double* dmma_tflops);

/* Library identity. */
int ocpqp_abi_version(void);
const char* ocpqp_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* OCPQP_B200_H */
