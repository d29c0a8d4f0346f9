// Fused batched OCP-QP interior-point solver for sm_100a (fp64).
//
// One CTA ("team") owns one QP at a time and runs the whole speed-mode
// predictor-corrector loop of the reference (solver.py:180-308) for it:
// residuals (view.py:272-288), termination (ipm_core.py:286-314), classical
// Riccati factor (kkt_ocp.py:142-201, 231-251) with the speed-mode retry ladder
// (solver.py:145-164), affine / corrector solves (kkt_ocp.py:254-320 with
// kkt_common.py:118-163), step length, centering, conditional corrector and
// update (ipm_core.py:201-272).  Different QPs run different iteration counts
// with no host involvement; CTAs pull QPs from an atomic counter (persistent
// grid, one workspace slot per CTA so the per-slot factor workspace stays hot
// in shared memory / L2 instead of streaming through HBM).
//
// Every workspace buffer is addressed through a generic pointer that the host
// places in shared memory when it fits and in the slot's global workspace
// otherwise (ocpqp_capi.cu: place_workspace).
#include <cuda_runtime.h>

#include <algorithm>
#include <math.h>
#include <stdint.h>

#include "ocpqp_internal.h"

namespace ocpqp {

// ---------------------------------------------------------------------------
// team (CTA) primitives
// ---------------------------------------------------------------------------
__device__ __forceinline__ void tsync() { __syncthreads(); }

// Deterministic team reductions: warp butterfly, then every thread combines the
// per-warp partials in the same order (so every thread holds the same value).
__device__ double team_sum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < nwarp; ++i) s += red[i];
    return s;
}

__device__ double team_max(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = red[0];
    for (int i = 1; i < nwarp; ++i) s = fmax(s, red[i]);
    return s;
}

__device__ double team_min(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(0xffffffffu, v, o));
    const int w = threadIdx.x >> 5, nwarp = blockDim.x >> 5;
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    double s = red[0];
    for (int i = 1; i < nwarp; ++i) s = fmin(s, red[i]);
    return s;
}

__device__ __forceinline__ int team_or(int v) { return __syncthreads_or(v); }

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

// max |x| with NaN propagation (np.max(np.abs(v)) semantics, view.py:291-292)
struct AbsMax {
    double m = 0.0;
    int nan = 0;
    __device__ __forceinline__ void add(double x) {
        if (isnan(x)) nan = 1;
        else m = fmax(m, fabs(x));
    }
};

__device__ double team_absmax(const AbsMax& a, double* red) {
    const int nan = team_or(a.nan);
    const double m = team_max(a.m, red);
    return nan ? qnan() : m;
}

// ---------------------------------------------------------------------------
// per-QP context
// ---------------------------------------------------------------------------
struct Ctx {
    const KParams* p;
    const StageInfo* st;
    int N;
    const double* f[OCPQP_NUM_FIELDS];  // this QP's field bases (nullptr = default)
    double* w[WS_NUM];                  // workspace buffers
    double* red;                        // reduction scratch (smem)
    int* iflag;                         // int scratch (smem)
    double n_act;                       // number of active constraint sides
};

// Absent fields point at the plan's default rows (zeros, ones for masks, -inf /
// +inf for bounds: fill_defaults in ocpqp_capi.cu), so no field pointer is null
// and `dflt` only documents the reference's zero-initialised value.
__device__ __forceinline__ double fget(const Ctx& c, int F, const StageInfo& s, int idx,
                                       double /*dflt*/) {
    return c.f[F][s.foff[F] + idx];
}
__device__ __forceinline__ const double* fptr(const Ctx& c, int F, const StageInfo& s) {
    return c.f[F] + s.foff[F];
}
// A/B of dynamics block n (n < N): A is nx' x nx, B is nx' x nu (row-major)
__device__ __forceinline__ double Aget(const Ctx& c, const StageInfo& s, int i, int j) {
    return fget(c, OCPQP_F_A, s, i * s.nx + j, 0.0);
}
__device__ __forceinline__ double Bget(const Ctx& c, const StageInfo& s, int i, int j) {
    return fget(c, OCPQP_F_B, s, i * s.nu + j, 0.0);
}
// [B A] (kkt_ocp.py:177)
__device__ __forceinline__ double BAget(const Ctx& c, const StageInfo& s, int i, int j) {
    return j < s.nu ? Bget(c, s, i, j) : Aget(c, s, i, j - s.nu);
}
// general-row matrix Jg = [D C] (view.py:113)
__device__ __forceinline__ double Jgget(const Ctx& c, const StageInfo& s, int g, int j) {
    return j < s.nu ? fget(c, OCPQP_F_D, s, g * s.nu + j, 0.0)
                    : fget(c, OCPQP_F_C, s, g * s.nx + (j - s.nu), 0.0);
}
// raw stage Hessian entry M_ij over (u, x) = [[R, S], [S', Q]]
__device__ __forceinline__ double Mraw(const Ctx& c, const StageInfo& s, int i, int j) {
    const int nu = s.nu;
    if (i < nu && j < nu) return fget(c, OCPQP_F_R, s, i * nu + j, 0.0);
    if (i < nu) return fget(c, OCPQP_F_S, s, i * s.nx + (j - nu), 0.0);
    if (j < nu) return fget(c, OCPQP_F_S, s, j * s.nx + (i - nu), 0.0);
    return fget(c, OCPQP_F_Q, s, (i - nu) * s.nx + (j - nu), 0.0);
}

// Loop over (stage, item) pairs of stages 0..NS-1 in parallel; `maxc` items
// per stage (padded).  No synchronisation: bodies must be independent.
#define FOR_STAGE_ITEMS(NS_, maxc_, n_, k_)                                              \
    for (int _i = threadIdx.x, _mc = (maxc_), _tot = (NS_) * _mc; _i < _tot;             \
         _i += blockDim.x) {                                                             \
        const int n_ = _i / _mc;                                                         \
        const int k_ = _i - n_ * _mc;
#define END_FOR_STAGE_ITEMS }

// ---------------------------------------------------------------------------
// setup: d vector and activity (view.py:108-129, 156-184)
// ---------------------------------------------------------------------------
__device__ void setup_constraints(Ctx& c) {
    const KParams& p = *c.p;
    double* dvec = c.w[WS_DVEC];
    double* act = c.w[WS_ACT];
    double cnt = 0.0;
    FOR_STAGE_ITEMS(c.N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int m = s.m;
            double d;
            bool a;
            if (k < 2 * m) {
                const bool lo = k < m;
                const int i = lo ? k : k - m;
                double bound;
                if (i < s.nb)
                    bound = fget(c, lo ? OCPQP_F_lb : OCPQP_F_ub, s, i, lo ? -INFINITY : INFINITY);
                else
                    bound = fget(c, lo ? OCPQP_F_lg : OCPQP_F_ug, s, i - s.nb,
                                 lo ? -INFINITY : INFINITY);
                const double mask = fget(c, lo ? OCPQP_F_maskl : OCPQP_F_masku, s, i, 1.0);
                a = (mask != 0.0) && isfinite(bound);
                d = lo ? bound : -bound;
            } else {
                const bool lo = k < 2 * m + s.ns;
                const int j = lo ? k - 2 * m : k - 2 * m - s.ns;
                d = fget(c, lo ? OCPQP_F_sl_lb : OCPQP_F_su_lb, s, j, 0.0);
                a = isfinite(d);
            }
            act[s.c_off + k] = a ? 1.0 : 0.0;
            dvec[s.c_off + k] = a ? d : 0.0;
            cnt += a ? 1.0 : 0.0;
        }
    END_FOR_STAGE_ITEMS
    c.n_act = team_sum(cnt, c.red);  // includes a barrier
}

// ---------------------------------------------------------------------------
// Jc w per row (ConBlock.rows_w, view.py:91-97) and Jc' coeff (rows_w_t :99-105)
// ---------------------------------------------------------------------------
__device__ void rows_values(const Ctx& c, const double* y, double* rowv) {
    const KParams& p = *c.p;
    FOR_STAGE_ITEMS(c.N + 1, p.m_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.m) {
            const double* w = y + s.u_off;
            double v;
            if (i < s.nb) {
                v = w[p.idxb[s.ib_off + i]];
            } else if (s.ng >= 32) {
                continue;   // large stages: one warp per general row, below
            } else {
                const int g = i - s.nb, nu = s.nu, nx = s.nx;
                const double* Dg = fptr(c, OCPQP_F_D, s) + g * nu;
                const double* Cg = fptr(c, OCPQP_F_C, s) + g * nx;
                v = 0.0;   // one fma chain; unrolled so that the loads of eight steps overlap
#pragma unroll 8
                for (int j = 0; j < nu; ++j) v = fma(Dg[j], w[j], v);
#pragma unroll 8
                for (int j = 0; j < nx; ++j) v = fma(Cg[j], w[nu + j], v);
            }
            rowv[s.m_off + i] = v;
        }
    END_FOR_STAGE_ITEMS
    // general rows of large stages (the condensed config-4 stage: 240 rows of
    // 160 columns): one warp per row, the lanes across the columns (coalesced
    // loads, one butterfly) instead of one thread walking a 160-term chain
    const int lane = threadIdx.x & 31, nwarp = blockDim.x >> 5;
    for (int n = 0; n <= c.N; ++n) {
        const StageInfo& s = c.st[n];
        if (s.ng < 32) continue;
        const int nu = s.nu, nx = s.nx;
        const double* w = y + s.u_off;
        const double* D = fptr(c, OCPQP_F_D, s);
        const double* C = fptr(c, OCPQP_F_C, s);
        for (int g0 = 2 * (threadIdx.x >> 5); g0 < s.ng; g0 += 2 * nwarp) {
            double v0 = 0.0, v1 = 0.0;
            const bool two = g0 + 1 < s.ng;
            for (int j = lane; j < nu; j += 32) {
                const double wj = w[j];
                v0 = fma(D[g0 * nu + j], wj, v0);
                if (two) v1 = fma(D[(g0 + 1) * nu + j], wj, v1);
            }
            for (int j = lane; j < nx; j += 32) {
                const double wj = w[nu + j];
                v0 = fma(C[g0 * nx + j], wj, v0);
                if (two) v1 = fma(C[(g0 + 1) * nx + j], wj, v1);
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                v0 += __shfl_xor_sync(0xffffffffu, v0, o);
                v1 += __shfl_xor_sync(0xffffffffu, v1, o);
            }
            if (lane == 0) {
                rowv[s.m_off + s.nb + g0] = v0;
                if (two) rowv[s.m_off + s.nb + g0 + 1] = v1;
            }
        }
    }
}

__device__ __forceinline__ double rows_t(const Ctx& c, const StageInfo& s, int j,
                                         const double* coeff /* stage rows */) {
    const int kb = c.p->var_box[s.u_off + j];
    double out = kb >= 0 ? coeff[kb] : 0.0;
    if (s.ng) {
        // column j of Jg = [D C]: stride nu (j < nu) or nx
        const bool du = j < s.nu;
        const double* col = du ? fptr(c, OCPQP_F_D, s) + j : fptr(c, OCPQP_F_C, s) + (j - s.nu);
        const int ld = du ? s.nu : s.nx;
        const double* cg = coeff + s.nb;
        double g = 0.0;
        if (s.ng >= 32) {
            // large stages: four interleaved partial sums (the chain is the cost)
            double g1 = 0.0, g2 = 0.0, g3 = 0.0;
            int r = 0;
#pragma unroll 2
            for (; r + 3 < s.ng; r += 4) {
                g = fma(col[r * ld], cg[r], g);
                g1 = fma(col[(r + 1) * ld], cg[r + 1], g1);
                g2 = fma(col[(r + 2) * ld], cg[r + 2], g2);
                g3 = fma(col[(r + 3) * ld], cg[r + 3], g3);
            }
            for (; r < s.ng; ++r) g = fma(col[r * ld], cg[r], g);
            g = (g + g1) + (g2 + g3);
        } else {
#pragma unroll 8
            for (int r = 0; r < s.ng; ++r) g = fma(col[r * ld], cg[r], g);
        }
        out += g;
    }
    return out;
}

// constraint value C y of slot k of stage s (view.py:132-142) from row values
__device__ __forceinline__ double slot_cy(const Ctx& c, const StageInfo& s, int k,
                                          const double* rowv, const double* y) {
    const KParams& p = *c.p;
    const int m = s.m;
    double cy;
    if (k < m) cy = rowv[s.m_off + k];
    else if (k < 2 * m) cy = -rowv[s.m_off + k - m];
    else cy = 0.0;
    if (s.ns) {
        if (k < 2 * m) {
            const int i = k < m ? k : k - m;
            const int j = p.row_slack[s.m_off + i];
            if (j >= 0) cy += y[p.nv + (k < m ? 0 : p.ns_tot) + s.s_off + j];
        } else {
            const bool lo = k < 2 * m + s.ns;
            const int j = lo ? k - 2 * m : k - 2 * m - s.ns;
            cy = y[p.nv + (lo ? 0 : p.ns_tot) + s.s_off + j];
        }
    }
    return cy;
}

// ---------------------------------------------------------------------------
// residuals (view.py:272-288)
// ---------------------------------------------------------------------------
struct ResNorms {
    double g, b, d, m, mu;
};

// With lamI / tI non-null: the exact KKT matrix action kkt_apply_vec
// (kkt_common.py:166-181) on the direction (y, pi, lam, t) at the iterate
// (lamI, tI) -- the same operators without g, b, d and a_m = t dlam + lam dt.
__device__ ResNorms residuals(Ctx& c, const double* y, const double* pi, const double* lam,
                              const double* t, double* r_g, double* r_b, double* r_d,
                              double* r_m /* may be null */, const double* lamI = nullptr,
                              const double* tI = nullptr) {
    const KParams& p = *c.p;
    const bool homog = lamI != nullptr;
    const int N = c.N;
    const double* act = c.w[WS_ACT];
    const double* dvec = c.w[WS_DVEC];
    double* rowv = c.w[WS_ROWV];
    double* crow = c.w[WS_CROW];
    rows_values(c, y, rowv);
    // masked lam_lo - lam_up per row (ct_lam, view.py:145-153, 197-205)
    FOR_STAGE_ITEMS(N + 1, p.m_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.m) {
            const int k = s.c_off + i;
            const double ll = act[k] != 0.0 ? lam[k] : 0.0;
            const double lu = act[k + s.m] != 0.0 ? lam[k + s.m] : 0.0;
            crow[s.m_off + i] = ll - lu;
        }
    END_FOR_STAGE_ITEMS
    tsync();
    AbsMax ag, ab, ad, am;
    double musum = 0.0;
    // r_g = H y + g - A' pi - C' lam over the stage windows
    FOR_STAGE_ITEMS(N + 1, p.nw_max, n, j)
        const StageInfo& s = c.st[n];
        if (j < s.nw) {
            const double* w = y + s.u_off;
            const int nu = s.nu;
            double h1 = 0.0, h2 = 0.0, g;
            if (j < nu) {  // R u + S x  (view.py:368-377)
                for (int k = 0; k < nu; ++k) h1 = fma(fget(c, OCPQP_F_R, s, j * nu + k, 0.0), w[k], h1);
                for (int k = 0; k < s.nx; ++k) h2 = fma(fget(c, OCPQP_F_S, s, j * s.nx + k, 0.0), w[nu + k], h2);
                g = fget(c, OCPQP_F_r, s, j, 0.0);
            } else {       // S' u + Q x
                const int jx = j - nu;
                for (int k = 0; k < nu; ++k) h1 = fma(fget(c, OCPQP_F_S, s, k * s.nx + jx, 0.0), w[k], h1);
                for (int k = 0; k < s.nx; ++k) h2 = fma(fget(c, OCPQP_F_Q, s, jx * s.nx + k, 0.0), w[nu + k], h2);
                g = fget(c, OCPQP_F_q, s, jx, 0.0);
            }
            double r = homog ? h1 + h2 : (h1 + h2) + g;
            // at_pi (view.py:400-409): +pi_{n-1} on x_n, -B'pi_n / -A'pi_n on (u_n, x_n)
            double atp = 0.0;
            if (j >= nu && n > 0) atp = pi[c.st[n - 1].pi_off + (j - nu)];
            if (n < N) {
                double a = 0.0;
                const double* pn = pi + s.pi_off;
                if (j < nu)
                    for (int k = 0; k < s.nxn; ++k) a = fma(Bget(c, s, k, j), pn[k], a);
                else
                    for (int k = 0; k < s.nxn; ++k) a = fma(Aget(c, s, k, j - nu), pn[k], a);
                atp -= a;
            }
            r -= atp;
            r -= rows_t(c, s, j, crow + s.m_off);
            r_g[s.u_off + j] = r;
            ag.add(r);
        }
    END_FOR_STAGE_ITEMS
    if (p.ns_tot) {
        // slack components: Z s + z - (lam_row + lam_slack_bound) (view.py:145-153, 207-229)
        FOR_STAGE_ITEMS(N + 1, p.ns_max, n, j)
            const StageInfo& s = c.st[n];
            if (j < s.ns) {
                const int row = p.idxs[s.is_off + j];
                const int kl = s.c_off + row, ku = s.c_off + s.m + row;
                const int ksl = s.c_off + 2 * s.m + j, ksu = ksl + s.ns;
                const double lsl = (act[kl] != 0.0 ? lam[kl] : 0.0) + (act[ksl] != 0.0 ? lam[ksl] : 0.0);
                const double lsu = (act[ku] != 0.0 ? lam[ku] : 0.0) + (act[ksu] != 0.0 ? lam[ksu] : 0.0);
                const int yl = p.nv + s.s_off + j, yu = p.nv + p.ns_tot + s.s_off + j;
                const double gl = homog ? 0.0 : fget(c, OCPQP_F_zl, s, j, 0.0);
                const double gu = homog ? 0.0 : fget(c, OCPQP_F_zu, s, j, 0.0);
                const double rl = (fget(c, OCPQP_F_Zl, s, j, 0.0) * y[yl] + gl) - lsl;
                const double ru = (fget(c, OCPQP_F_Zu, s, j, 0.0) * y[yu] + gu) - lsu;
                r_g[yl] = rl;
                r_g[yu] = ru;
                ag.add(rl);
                ag.add(ru);
            }
        END_FOR_STAGE_ITEMS
    }
    // r_b = -(x_{n+1} - A x - B u) + b (view.py:411-427)
    FOR_STAGE_ITEMS(N, p.nx_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.nxn) {
            const double* u = y + s.u_off;
            const double* x = y + s.x_off;
            const double xn = y[c.st[n + 1].x_off + i];
            double ax = 0.0, bu = 0.0;
            for (int k = 0; k < s.nx; ++k) ax = fma(Aget(c, s, i, k), x[k], ax);
            for (int k = 0; k < s.nu; ++k) bu = fma(Bget(c, s, i, k), u[k], bu);
            const double r = homog ? -((xn - ax) - bu) : -((xn - ax) - bu) + fget(c, OCPQP_F_b, s, i, 0.0);
            r_b[s.pi_off + i] = r;
            ab.add(r);
        }
    END_FOR_STAGE_ITEMS
    // r_d = act ? -C y + d + t : 0 ;  r_m = act ? lam t : 0
    FOR_STAGE_ITEMS(N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double rd = 0.0, rm = 0.0;
            if (act[kk] != 0.0) {
                const double cy = slot_cy(c, s, k, rowv, y);
                if (homog) {
                    rd = -cy + t[kk];
                    rm = tI[kk] * lam[kk] + lamI[kk] * t[kk];
                } else {
                    rd = (-cy + dvec[kk]) + t[kk];
                    rm = lam[kk] * t[kk];
                    musum += rm;
                }
            }
            r_d[kk] = rd;
            if (r_m) r_m[kk] = rm;
            ad.add(rd);
            am.add(rm);
        }
    END_FOR_STAGE_ITEMS
    ResNorms out;
    out.g = team_absmax(ag, c.red);
    out.b = team_absmax(ab, c.red);
    out.d = team_absmax(ad, c.red);
    out.m = team_absmax(am, c.red);
    const double tot = team_sum(musum, c.red);
    out.mu = c.n_act > 0.0 ? tot / c.n_act : 0.0;
    return out;
}

// ---------------------------------------------------------------------------
// dense team kernels
// ---------------------------------------------------------------------------
// In-place lower Cholesky of the n x n matrix at L (leading dim ld); the upper
// triangle is zeroed.  Fails (returns false) on a pivot that is not > 0,
// including NaN, like LAPACK potrf behind linalg.cholesky_factor (linalg.py:81-118).
__device__ bool team_chol(double* L, int n, int ld, int* flag, bool keep_upper = false) {
    // Two barriers per column: every thread reads the pivot and takes the
    // (identical) square root itself; the diagonal is written back during the
    // trailing update, which reads only the scaled column.
    (void)flag;
    const int tid = threadIdx.x, T = blockDim.x;
    for (int k = 0; k < n; ++k) {
        const double d = L[k * ld + k];
        if (!(d > 0.0)) {
            tsync();
            return false;
        }
        const double dk = sqrt(d);
        // the scaled column is mirrored into row k's (unused, finally zeroed)
        // upper part, so the trailing update reads it contiguously
        for (int i = k + 1 + tid; i < n; i += T) {
            const double v = L[i * ld + k] / dk;
            L[i * ld + k] = v;
            L[k * ld + i] = v;
        }
        tsync();
        if (tid == 0) L[k * ld + k] = dk;
        // rows round-robin over warps, columns j <= i over lanes
        const int lane = tid & 31, nwarp = (T + 31) >> 5;
        const double* __restrict__ ck = L + k * ld;
        if (n - k > 4 * nwarp) {
            // four rows per warp pass: their loads are independent, so four
            // L2 / L1 round trips overlap (same arithmetic per element)
            for (int i0 = k + 1 + 4 * (tid >> 5); i0 < n; i0 += 4 * nwarp) {
                double lik[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) lik[q] = i0 + q < n ? L[(i0 + q) * ld + k] : 0.0;
                const int imax = min(i0 + 3, n - 1);
                for (int j = k + 1 + lane; j <= imax; j += 32) {
                    const double c = ck[j];
                    double v[4];
#pragma unroll
                    for (int q = 0; q < 4; ++q) v[q] = (i0 + q < n && j <= i0 + q) ? L[(i0 + q) * ld + j] : 0.0;
#pragma unroll
                    for (int q = 0; q < 4; ++q)
                        if (i0 + q < n && j <= i0 + q) L[(i0 + q) * ld + j] = v[q] - lik[q] * c;
                }
            }
        } else {
            for (int i = k + 1 + (tid >> 5); i < n; i += nwarp) {
                double* Li = L + i * ld;
                const double lik = Li[k];
                for (int j = k + 1 + lane; j <= i; j += 32) Li[j] -= lik * ck[j];
            }
        }
        tsync();
    }
    // keep_upper: the caller still reads L' from the upper triangle (row k holds
    // column k of L) and zeroes it itself
    if (!keep_upper) {
        for (int idx = tid; idx < n * n; idx += T) {
            const int i = idx / n, j = idx - i * n;
            if (j > i) L[i * ld + j] = 0.0;
        }
        tsync();
    }
    return true;
}

// The same factorization with the matrix held as a packed lower triangle in the
// scratch buffer `sm` (the stage's T1 buffer, shared memory when the plan placed
// it): every column step then costs shared-memory round trips instead of L2
// ones.  Same operations and order per element as team_chol.  keep_upper as there.
__device__ bool team_chol_packed(double* L, int n, double* sm, bool keep_upper) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int lane = tid & 31, nwarp = (T + 31) >> 5;
    auto at = [&](int i, int j) -> double& { return sm[i * (i + 1) / 2 + j]; };
    for (int e = tid; e < n * n; e += T) {
        const int i = e / n, j = e - i * n;
        if (j <= i) at(i, j) = L[e];
    }
    tsync();
    bool ok = true;
    for (int k = 0; k < n; ++k) {
        const double d = at(k, k);
        if (!(d > 0.0)) {
            ok = false;
            break;
        }
        const double dk = sqrt(d);
        for (int i = k + 1 + tid; i < n; i += T) at(i, k) = at(i, k) / dk;
        tsync();
        if (tid == 0) at(k, k) = dk;   // read by nobody in this column step
        for (int i = k + 1 + (tid >> 5); i < n; i += nwarp) {
            const double lik = at(i, k);
            for (int j = k + 1 + lane; j <= i; j += 32) at(i, j) -= lik * at(j, k);
        }
        tsync();
    }
    tsync();
    if (!ok) return false;
    for (int e = tid; e < n * n; e += T) {
        const int i = e / n, j = e - i * n;
        L[e] = j <= i ? at(i, j) : (keep_upper ? at(j, i) : 0.0);
    }
    tsync();
    return true;
}

// serial cho_solve x = (L L')^{-1} b for one thread (kkt_ocp.py:66-67)
__device__ __forceinline__ void cho_solve_serial(const double* L, int n, double* x) {
    for (int i = 0; i < n; ++i) {
        double s = x[i];
        for (int k = 0; k < i; ++k) s -= L[i * n + k] * x[k];
        x[i] = s / L[i * n + i];
    }
    for (int i = n - 1; i >= 0; --i) {
        double s = x[i];
        for (int k = i + 1; k < n; ++k) s -= L[k * n + i] * x[k];
        x[i] = s / L[i * n + i];
    }
}

// The same cho_solve by one whole warp for n <= 32, right-looking (lane i owns
// x_i; one broadcast per pivot instead of n serial dot products; the backward
// sweep sums in descending k).  out = sgn * x.
__device__ __forceinline__ void warp_cho_solve(const double* L, int n, const double* xin,
                                               double* out, double sgn) {
    const int lane = threadIdx.x & 31;
    double z = lane < n ? xin[lane] : 0.0;
    for (int k = 0; k < n; ++k) {
        if (lane == k) z = z / L[k * n + k];
        const double zk = __shfl_sync(0xffffffffu, z, k);
        if (lane > k && lane < n) z = fma(-L[lane * n + k], zk, z);
    }
    for (int k = n - 1; k >= 0; --k) {
        if (lane == k) z = z / L[k * n + k];
        const double zk = __shfl_sync(0xffffffffu, z, k);
        if (lane < k) z = fma(-L[k * n + lane], zk, z);
    }
    if (lane < n) out[lane] = sgn * z;
}

// warp_cho_solve for 32 < n <= 128: lane owns x_{lane + 32 q}, q < 4 (dense QPs
// after full condensing: n = nv up to a few hundred go serial beyond this).
__device__ __forceinline__ double wsel4(int q, double a, double b, double c, double d) {
    return q == 0 ? a : q == 1 ? b : q == 2 ? c : d;
}
__device__ void warp_cho_solve4(const double* L, int n, const double* xin, double* out,
                                double sgn) {
    // Each lane holds the reciprocal pivots of its rows (computed in parallel,
    // off the chain) and column k+1 of L is loaded while step k runs: a step
    // is one multiply, one shuffle and one FMA.
    const int lane = threadIdx.x & 31;
    double z[4], lc[4], rd[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        z[q] = i < n ? xin[i] : 0.0;
        rd[q] = i < n ? 1.0 / L[i * n + i] : 0.0;
        lc[q] = (i > 0 && i < n) ? L[i * n] : 0.0;
    }
    for (int k = 0; k < n; ++k) {
        const int kq = k >> 5, kl = k & 31;
        double ln[4];
        const int k1 = k + 1;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = lane + 32 * q;
            ln[q] = (i > k1 && i < n) ? L[i * n + k1] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q == kq && lane == kl) z[q] = z[q] * rd[q];
        const double zk = __shfl_sync(0xffffffffu, wsel4(kq, z[0], z[1], z[2], z[3]), kl);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = lane + 32 * q;
            if (i > k && i < n) z[q] = fma(-lc[q], zk, z[q]);
            lc[q] = ln[q];
        }
    }
    // backward: row k of L (entries i < k) prefetched one step ahead
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const int i = lane + 32 * q;
        lc[q] = (i < n - 1) ? L[(n - 1) * n + i] : 0.0;
    }
    for (int k = n - 1; k >= 0; --k) {
        const int kq = k >> 5, kl = k & 31;
        const int k1 = k - 1;
        double ln[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = lane + 32 * q;
            ln[q] = (i < k1) ? L[k1 * n + i] : 0.0;
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
            if (q == kq && lane == kl) z[q] = z[q] * rd[q];
        const double zk = __shfl_sync(0xffffffffu, wsel4(kq, z[0], z[1], z[2], z[3]), kl);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int i = lane + 32 * q;
            if (i < k) z[q] = fma(-lc[q], zk, z[q]);
            lc[q] = ln[q];
        }
    }
#pragma unroll
    for (int q = 0; q < 4; ++q)
        if (lane + 32 * q < n) out[lane + 32 * q] = sgn * z[q];
}

// Jg' diag(coef) Jg added into the symmetric stage matrix Mb (nw x nw; the
// SYRK of add_reduced_hessian, kkt_common.py:100-115) plus reg on the
// diagonal.  Kept out of line: the generic kernel is register-bound.
__device__ __noinline__ void rows_syrk(const Ctx& c, const StageInfo& s, const double* cg,
                                       double* Mb, int nw, int ng, double reg) {
    const int tid = threadIdx.x, T = blockDim.x;
    if (ng >= 32 && nw >= 64) {
        // Jg' diag(coef) Jg on the FP64 tensor cores (DMMA m8n8k4): one warp per
        // 16 x 16 block (2 x 2 tiles) of the lower block triangle -- four
        // operand loads feed four DMMAs (half the L2 traffic of one tile per
        // warp) on four independent accumulator pairs; k = general rows in
        // steps of 4, mirrored in the epilogue.  Fragment layout as below.
        const int lane = tid & 31, warp = tid >> 5, nwarp = T >> 5;
        const int gr = lane >> 2, tg = lane & 3;
        const int nb16 = (nw + 15) >> 4, nblk = nb16 * (nb16 + 1) / 2;
        const int nu = s.nu, nx = s.nx;
        const double* Dp = fptr(c, OCPQP_F_D, s);
        const double* Cp = fptr(c, OCPQP_F_C, s);
        // First general row with a nonzero in each 16-column block: the rows of a
        // condensed stage are block lower triangular (the state of block stage k
        // depends on u_0 .. u_{k-1} only), so the leading rows of most column
        // blocks are exact zeros and the k loop of a block pair can start at the
        // later of the two (41 % fewer DMMAs on the condensed config-4 stage; the
        // skipped terms are exact zeros).  One warp scans a column block, 32 rows
        // x 16 columns per step.
        __shared__ int s_first[16];
        if (nb16 <= 16) {
            for (int cb = warp; cb < nb16; cb += nwarp) {
                const int col = cb * 16 + (lane & 15), rsub = lane >> 4;
                const bool cin = col < nw;
                const double* cp = col < nu ? Dp + col : Cp + (col - nu);
                const int ld = col < nu ? nu : nx;
                int first = ng;
                for (int r0 = 0; r0 < ng && first == ng; r0 += 32) {
                    unsigned hit = 0;
#pragma unroll
                    for (int q = 0; q < 16; ++q) {
                        const int r = r0 + 2 * q + rsub;
                        if (cin && r < ng && cp[r * ld] != 0.0) hit |= 1u << q;
                    }
#pragma unroll
                    for (int o = 16; o > 0; o >>= 1) hit |= __shfl_xor_sync(0xffffffffu, hit, o);
                    if (hit) first = r0 + 2 * (__ffs(hit) - 1);
                }
                if (lane == 0) s_first[cb] = first;
            }
        } else if (tid < 16) {
            s_first[tid] = 0;
        }
        __syncthreads();
        for (int t = warp; t < nblk; t += nwarp) {
            int bi = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while (bi * (bi + 1) / 2 > t) --bi;
            while ((bi + 1) * (bi + 2) / 2 <= t) ++bi;
            const int bj = t - bi * (bi + 1) / 2;
            const int rs = nb16 <= 16 ? (max(s_first[bi], s_first[bj]) & ~3) : 0;
            const double* ca[2];
            const double* cb[2];
            int la[2], lb[2];
            bool ina[2], inb[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int ia = bi * 16 + 8 * h + gr, jb = bj * 16 + 8 * h + gr;
                ina[h] = ia < nw;
                inb[h] = jb < nw;
                ca[h] = ia < nu ? Dp + ia : Cp + (ia - nu);
                cb[h] = jb < nu ? Dp + jb : Cp + (jb - nu);
                la[h] = ia < nu ? nu : nx;
                lb[h] = jb < nu ? nu : nx;
            }
            double d[2][2][2];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int g = 0; g < 2; ++g) d[h][g][0] = d[h][g][1] = 0.0;
#pragma unroll 2
            for (int r0 = rs; r0 < ng; r0 += 4) {
                const int r = r0 + tg;
                const bool rin = r < ng;
                const double w = rin ? cg[r] : 0.0;
                double av[2], bv[2];
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    av[h] = (rin && ina[h]) ? ca[h][r * la[h]] : 0.0;
                    bv[h] = (rin && inb[h]) ? w * cb[h][r * lb[h]] : 0.0;
                }
#pragma unroll
                for (int h = 0; h < 2; ++h)
#pragma unroll
                    for (int g = 0; g < 2; ++g)
                        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                                     : "+d"(d[h][g][0]), "+d"(d[h][g][1])
                                     : "d"(av[h]), "d"(bv[g]));
            }
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int g = 0; g < 2; ++g)
#pragma unroll
                    for (int e = 0; e < 2; ++e) {
                        const int i = bi * 16 + 8 * h + gr, j = bj * 16 + 8 * g + 2 * tg + e;
                        if (i < nw && j <= i) {
                            double hh = d[h][g][e] + Mb[i * nw + j];
                            if (i == j && reg != 0.0) hh += reg;
                            Mb[i * nw + j] = hh;
                            Mb[j * nw + i] = hh;
                        }
                    }
        }
    } else if (ng >= 32 && nw >= 24) {
        // Jg' diag(coef) Jg on the FP64 tensor cores (DMMA m8n8k4): one warp
        // per 8x8 tile of the lower tile triangle, k = general rows in
        // steps of 4, mirrored in the epilogue.  Fragments: A row = lane/4,
        // col = lane%4; B row = lane%4, col = lane/4; D row = lane/4, cols
        // 2*(lane%4)+{0,1}.  (Dense QPs from full condensing: ng >> nw.)
        const int lane = tid & 31, warp = tid >> 5, nwarp = T >> 5;
        const int gr = lane >> 2, tg = lane & 3;
        const int nt = (nw + 7) >> 3, ntile = nt * (nt + 1) / 2;
        for (int t = warp; t < ntile; t += nwarp) {
            int ti = (int)((sqrt(8.0 * t + 1.0) - 1.0) * 0.5);
            while (ti * (ti + 1) / 2 > t) --ti;
            while ((ti + 1) * (ti + 2) / 2 <= t) ++ti;
            const int tj = t - ti * (ti + 1) / 2;
            const int ia = ti * 8 + gr, jb = tj * 8 + gr;
            // this lane's columns of Jg = [D C] (row stride nu or nx)
            const int nu = s.nu, nx = s.nx;
            const double* Dp = fptr(c, OCPQP_F_D, s);
            const double* Cp = fptr(c, OCPQP_F_C, s);
            const double* ca = ia < nu ? Dp + ia : Cp + (ia - nu);
            const double* cb = jb < nu ? Dp + jb : Cp + (jb - nu);
            const int la = ia < nu ? nu : nx, lb = jb < nu ? nu : nx;
            double d0 = 0.0, d1 = 0.0;
#pragma unroll 4   // the operand loads of four k steps in flight
            for (int r0 = 0; r0 < ng; r0 += 4) {
                const int r = r0 + tg;
                const bool rin = r < ng;
                const double av = (rin && ia < nw) ? ca[r * la] : 0.0;
                const double bv = (rin && jb < nw) ? cg[r] * cb[r * lb] : 0.0;
                asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                             : "+d"(d0), "+d"(d1)
                             : "d"(av), "d"(bv));
            }
            const int i = ti * 8 + gr;
#pragma unroll
            for (int e = 0; e < 2; ++e) {
                const int j = tj * 8 + 2 * tg + e;
                if (i < nw && j <= i) {
                    double h = (e ? d1 : d0) + Mb[i * nw + j];
                    if (i == j && reg != 0.0) h += reg;
                    Mb[i * nw + j] = h;
                    Mb[j * nw + i] = h;
                }
            }
        }
    } else {
        // Jg' diag(coef) Jg over 4x4 register blocks of the lower block
        // triangle, mirrored (the SYRK of add_reduced_hessian): 8 loads per
        // 16 FMAs instead of 2 per FMA -- the dominant term of dense QPs
        // (full condensing: ng >> nw)
        const int nbk = (nw + 3) >> 2;
        const int nblk = nbk * (nbk + 1) / 2;
        for (int b = tid; b < nblk; b += T) {
            int bi = (int)((sqrt(8.0 * b + 1.0) - 1.0) * 0.5);
            while (bi * (bi + 1) / 2 > b) --bi;
            while ((bi + 1) * (bi + 2) / 2 <= b) ++bi;
            const int bj = b - bi * (bi + 1) / 2;
            const int i0 = bi * 4, j0 = bj * 4;
            double acc[4][4];
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int e = 0; e < 4; ++e) acc[a][e] = 0.0;
            for (int r = 0; r < ng; ++r) {
                const double w = cg[r];
                double ji[4], cj[4];
#pragma unroll
                for (int a = 0; a < 4; ++a) {
                    ji[a] = (i0 + a < nw) ? Jgget(c, s, r, i0 + a) : 0.0;
                    cj[a] = (j0 + a < nw) ? w * Jgget(c, s, r, j0 + a) : 0.0;
                }
#pragma unroll
                for (int a = 0; a < 4; ++a)
#pragma unroll
                    for (int e = 0; e < 4; ++e) acc[a][e] = fma(ji[a], cj[e], acc[a][e]);
            }
#pragma unroll
            for (int a = 0; a < 4; ++a)
#pragma unroll
                for (int e = 0; e < 4; ++e) {
                    const int i = i0 + a, j = j0 + e;
                    if (i < nw && j <= i) {
                        double h = acc[a][e] + Mb[i * nw + j];
                        if (i == j && reg != 0.0) h += reg;
                        Mb[i * nw + j] = h;
                        Mb[j * nw + i] = h;
                    }
                }
        }
    }
}

// ---------------------------------------------------------------------------
// C(i, j) = sum_k a(k, i) b(k, j), i < M, j < N, k ascending with one fma chain
// per output (the arithmetic of the one-output-per-thread loops it replaces),
// over 4 x 4 register tiles: 8 operand loads per 16 FMAs, the loads of a k step
// independent of each other.  Operand columns are given as (pointer, stride):
// ca(i) / cb(j) return the address of element (0, i) / (0, j) and the stride
// between consecutive k, so the k loop carries no index arithmetic beyond two
// multiply-adds per operand.  epi(i, j, acc) stores.  Large stages only (the
// condensed config-4 stage: 160 x 160 x 60).
struct ColRef {
    const double* p;
    int ld;
};
template <class FA, class FB, class FE>
__device__ __forceinline__ void team_gemm_tn(int M, int N, int K, FA ca, FB cb, FE epi) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int tn = (N + 3) >> 2, nt = ((M + 3) >> 2) * tn;
    for (int t = tid; t < nt; t += T) {
        const int i0 = (t / tn) * 4, j0 = (t - (t / tn) * tn) * 4;
        ColRef ra[4], rb[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            // out-of-range columns re-read the tile's first one (finite data; never stored)
            ra[q] = ca(i0 + q < M ? i0 + q : i0);
            rb[q] = cb(j0 + q < N ? j0 + q : j0);
        }
        double acc[4][4];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int r = 0; r < 4; ++r) acc[q][r] = 0.0;
#pragma unroll 2
        for (int k = 0; k < K; ++k) {
            double av[4], bv[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                av[q] = ra[q].p[k * ra[q].ld];
                bv[q] = rb[q].p[k * rb[q].ld];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
#pragma unroll
                for (int r = 0; r < 4; ++r) acc[q][r] = fma(av[q], bv[r], acc[q][r]);
        }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int r = 0; r < 4; ++r)
                if (i0 + q < M && j0 + r < N) epi(i0 + q, j0 + r, acc[q][r]);
    }
}
// stages large enough for the tiled paths (every thread gets several tiles)
__device__ __forceinline__ bool big_stage(int nw) { return nw * nw >= 16 * (int)blockDim.x; }

// ---------------------------------------------------------------------------
// Householder QR of the m x n (m >= n) row-major stack S in place (LAPACK
// dgeqr2 / dlarfg reflectors, the arithmetic of np.linalg.qr(mode="r")), then
// qr_cholesky's rank test and row-sign normalisation (linalg.py:152-187).
// Returns false on RankDeficient.  Column-parallel reflector application.
// ---------------------------------------------------------------------------
// The same reflectors by warp 0 alone when the stack fits one warp (m <= 32):
// lane i owns row i, column sums by shuffles, only __syncwarp between steps
// (the block-wide version spends its time in barriers at these sizes).
__device__ void warp_qr_reflectors(double* S, int m, int n) {
    const int lane = threadIdx.x & 31;
    const bool own = lane < m;
    for (int k = 0; k < n; ++k) {
        const double sk = (own && lane > k) ? S[lane * n + k] : 0.0;
        double ss = sk * sk;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        if (ss == 0.0) continue;    // H = I (tau = 0)
        const double alpha = S[k * n + k];
        const double beta = -copysign(hypot(alpha, sqrt(ss)), alpha);
        const double tau = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        const double vk = (own && lane > k) ? sk * sc : 0.0;   // reflector entry of this row
        if (own && lane > k) S[lane * n + k] = vk;
        for (int j = k + 1; j < n; ++j) {
            double w = (own && lane > k) ? vk * S[lane * n + j] : 0.0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            w = (S[k * n + j] + w) * tau;
            __syncwarp();
            if (own && lane > k) S[lane * n + j] = fma(-w, vk, S[lane * n + j]);
            if (lane == k) S[k * n + j] -= w;
            __syncwarp();
        }
        if (lane == k) S[k * n + k] = beta;
        __syncwarp();
    }
}

__device__ __noinline__ bool team_qr(Ctx& c, double* S, int m, int n) {
    const int tid = threadIdx.x, T = blockDim.x;
    if (m <= 32) {
        if (tid < 32) warp_qr_reflectors(S, m, n);
        tsync();
    } else
    for (int k = 0; k < n; ++k) {
        double ss = 0.0;
        for (int i = k + 1 + tid; i < m; i += T) ss = fma(S[i * n + k], S[i * n + k], ss);
        ss = team_sum(ss, c.red);   // same value in every thread
        if (ss == 0.0) continue;    // H = I (tau = 0)
        const double alpha = S[k * n + k];
        const double beta = -copysign(hypot(alpha, sqrt(ss)), alpha);
        const double tau = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        for (int i = k + 1 + tid; i < m; i += T) S[i * n + k] *= sc;
        tsync();
        // reflector application: one warp per column j, lanes over the rows
        // (the dot product v'S[:, j] by a shuffle reduction)
        {
            const int lane = tid & 31, nwarp = (T + 31) >> 5;
            for (int j = k + 1 + (tid >> 5); j < n; j += nwarp) {
                double w = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) w = fma(S[i * n + k], S[i * n + j], w);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
                w = (S[k * n + j] + w) * tau;
                for (int i = k + 1 + lane; i < m; i += 32) S[i * n + j] = fma(-w, S[i * n + k], S[i * n + j]);
                if (lane == 0) S[k * n + j] -= w;
            }
        }
        if (tid == 0) S[k * n + k] = beta;
        tsync();
    }
    double dmax = 0.0;
    for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(S[i * n + i]));
    const double tol = (m > n ? m : n) * 2.220446049250313e-16 * dmax;
    int bad = 0;
    for (int i = 0; i < n; ++i)
        if (!(fabs(S[i * n + i]) > tol)) bad = 1;
    tsync();
    if (bad) return false;
    for (int i = tid; i < n; i += T) {
        const double sg = S[i * n + i] < 0.0 ? -1.0 : 1.0;
        for (int j = 0; j < n; ++j) S[i * n + j] = j < i ? 0.0 : sg * S[i * n + j];
    }
    tsync();
    return true;
}

enum { LINALG_OK = 0, LINALG_NPD = 1, LINALG_RANK = 2 };

// classical stage (kkt_ocp.py:231-251); the stage Hessian M~ is in Mb (== G
// when it need not survive the stage).  LINALG_OK / LINALG_NPD.
__device__ int stage_classical(Ctx& c, int n, const double* Mb, long long& flops) {
    const int N = c.N;
    const int tid = threadIdx.x, T = blockDim.x;
    const StageInfo& s = c.st[n];
    const int nu = s.nu, nx = s.nx, nw = s.nw, nxn = s.nxn;
    double* G = c.w[WS_G];
    double* T1 = c.w[WS_T1];
    double* Pall = c.w[WS_P];
    if (c.w[WS_HASLP] && tid == 0) c.w[WS_HASLP][n] = 0.0;
    if (n < N) {
        const double* Pn = Pall + c.st[n + 1].P_off;
        const double* An = fptr(c, OCPQP_F_A, s);
        const double* Bn = fptr(c, OCPQP_F_B, s);
        const bool big = big_stage(nw);
        auto BAcol = [&](int j) { return j < nu ? ColRef{Bn + j, nu} : ColRef{An + (j - nu), nx}; };
        if (big) {
            team_gemm_tn(nxn, nw, nxn, [&](int i) { return ColRef{Pn + i * nxn, 1}; }, BAcol,
                         [&](int i, int j, double v) { T1[i * nw + j] = v; });
            tsync();
            team_gemm_tn(nw, nw, nxn, BAcol, [&](int j) { return ColRef{T1 + j, nw}; },
                         [&](int i, int j, double v) { G[i * nw + j] = v + Mb[i * nw + j]; });
        } else {
        // T1 = P[n+1] [B A]  (nx' x nw): column j of [B A] read with stride
        for (int idx = tid; idx < nxn * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            const double* col = j < nu ? Bn + j : An + (j - nu);
            const int ld = j < nu ? nu : nx;
            double a = 0.0;
            for (int k = 0; k < nxn; ++k) a = fma(Pn[i * nxn + k], col[k * ld], a);
            T1[idx] = a;
        }
        tsync();
        // G = [B A]' T1 + M~
        for (int idx = tid; idx < nw * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            const double* col = i < nu ? Bn + i : An + (i - nu);
            const int ld = i < nu ? nu : nx;
            double a = 0.0;
            for (int k = 0; k < nxn; ++k) a = fma(col[k * ld], T1[k * nw + j], a);
            G[idx] = a + Mb[idx];
        }
        }
        flops += 2ll * nxn * nw * nxn + 2ll * nw * nw * nxn;
        tsync();
    } else if (Mb != G) {
        for (int idx = tid; idx < nw * nw; idx += T) G[idx] = Mb[idx];
        tsync();
    }
    double* P = Pall + s.P_off;
    if (nu) {
        double* L = c.w[WS_L] + s.L_off;
        double* K = c.w[WS_K] + s.K_off;
        for (int idx = tid; idx < nu * nu; idx += T) {
            const int i = idx / nu, j = idx - i * nu;
            L[idx] = G[i * nw + j];
        }
        tsync();
        flops += (long long)nu * nu * nu / 3;
        const bool bigk = nu >= 32 && (long long)nu * nx <= (long long)nxn * nw && n < N;
        // large stages: factor in the T1 buffer (free between G and the K solve)
        const bool packed = nu >= 32 && n < N && (long long)nu * (nu + 1) / 2 <= (long long)nxn * nw &&
                            __isShared(T1);   // only pays when the plan placed T1 in shared memory
        if (!(packed ? team_chol_packed(L, nu, T1, bigk) : team_chol(L, nu, nu, c.iflag, bigk)))
            return LINALG_NPD;
        if (bigk) {
            // K = -L'^{-1} L^{-1} G_ux (kkt_ocp.py:240-243), right-looking: the
            // lane quad 4c..4c+3 owns column j, lane q its rows q, q + 4, ...;
            // per pivot one division, the quad's FMAs on the rows still open
            // (four rows per batch: loads first, then stores) and a quad-wide
            // __syncwarp.  The column lives in T1 (free between G and the P
            // update; shared memory when the plan placed it); both sweeps read
            // row i of L, whose upper part still holds column i (team_chol).
            const int q = tid & 3;
            const unsigned qmask = 0xFu << (tid & 28);
            double* __restrict__ Y = T1;
            double* __restrict__ rinv = T1 + nu * nx;   // 1 / L_ii (behind the columns)
            const double* __restrict__ Lr = L;
            const bool have_rinv = (long long)nu * nx + nu <= (long long)nxn * nw;
            if (have_rinv) {
                for (int i = tid; i < nu; i += T) rinv[i] = 1.0 / Lr[i * nu + i];
                tsync();
            }
            for (int j = tid >> 2; j < nx; j += T >> 2) {
                for (int i = q; i < nu; i += 4) Y[i * nx + j] = G[i * nw + nu + j];
                __syncwarp(qmask);
                for (int i = 0; i < nu; ++i) {
                    // row i + 1 of L -> L1 while this pivot runs (each row is touched
                    // for the first time at its pivot: an L2 round trip per batch otherwise)
                    if (i + 1 < nu && (tid & 31) * 16 < nu)
                        asm volatile("prefetch.global.L1 [%0];\n" ::"l"(Lr + (i + 1) * nu + (tid & 31) * 16));
                    const double y = have_rinv ? Y[i * nx + j] * rinv[i] : Y[i * nx + j] / Lr[i * nu + i];
                    const double* Li = Lr + i * nu;
                    for (int k = i + 1 + ((q - (i + 1)) & 3); k < nu; k += 32) {
                        double l[8], v[8];
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int kk = k + 4 * r;
                            l[r] = kk < nu ? Li[kk] : 0.0;
                            v[r] = kk < nu ? Y[kk * nx + j] : 0.0;
                        }
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int kk = k + 4 * r;
                            if (kk < nu) Y[kk * nx + j] = fma(-l[r], y, v[r]);
                        }
                    }
                    __syncwarp(qmask);
                    if (q == (i & 3)) Y[i * nx + j] = y;
                }
                __syncwarp(qmask);
                for (int i = nu - 1; i >= 0; --i) {
                    if (i > 0 && (tid & 31) * 16 < nu)
                        asm volatile("prefetch.global.L1 [%0];\n" ::"l"(Lr + (i - 1) * nu + (tid & 31) * 16));
                    const double y = have_rinv ? Y[i * nx + j] * rinv[i] : Y[i * nx + j] / Lr[i * nu + i];
                    const double* Li = Lr + i * nu;
                    for (int k = q; k < i; k += 32) {
                        double l[8], v[8];
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int kk = k + 4 * r;
                            l[r] = kk < i ? Li[kk] : 0.0;
                            v[r] = kk < i ? Y[kk * nx + j] : 0.0;
                        }
#pragma unroll
                        for (int r = 0; r < 8; ++r) {
                            const int kk = k + 4 * r;
                            if (kk < i) Y[kk * nx + j] = fma(-l[r], y, v[r]);
                        }
                    }
                    __syncwarp(qmask);
                    if (q == (i & 3)) K[i * nx + j] = -y;
                }
            }
            tsync();
            for (int idx = tid; idx < nu * nu; idx += T) {
                const int i = idx / nu, j = idx - i * nu;
                if (j > i) L[idx] = 0.0;
            }
        } else
        // K = -L'^{-1} L^{-1} G_ux  (kkt_ocp.py:240-243), one column per thread
        for (int j = tid; j < nx; j += T) {
            for (int i = 0; i < nu; ++i) {
                double a = G[i * nw + nu + j];
                for (int k = 0; k < i; ++k) a -= L[i * nu + k] * K[k * nx + j];
                K[i * nx + j] = a / L[i * nu + i];
            }
            for (int i = nu - 1; i >= 0; --i) {
                double a = K[i * nx + j];
                for (int k = i + 1; k < nu; ++k) a -= L[k * nu + i] * K[k * nx + j];
                K[i * nx + j] = a / L[i * nu + i];
            }
            for (int i = 0; i < nu; ++i) K[i * nx + j] = -K[i * nx + j];
        }
        flops += 2ll * nu * nu * nx;
        tsync();
        // P = G_xx + G_ux' K (kkt_ocp.py:244)
        if (big_stage(nw)) {
            team_gemm_tn(nx, nx, nu, [&](int i) { return ColRef{G + nu + i, nw}; },
                         [&](int j) { return ColRef{K + j, nx}; },
                         [&](int i, int j, double v) { T1[i * nx + j] = v + G[(nu + i) * nw + nu + j]; });
        } else
        for (int idx = tid; idx < nx * nx; idx += T) {
            const int i = idx / nx, j = idx - i * nx;
            double a = 0.0;
            for (int k = 0; k < nu; ++k) a = fma(G[k * nw + nu + i], K[k * nx + j], a);
            T1[idx] = a + G[(nu + i) * nw + nu + j];
        }
        flops += 2ll * nx * nx * nu;
    } else {
        for (int idx = tid; idx < nx * nx; idx += T) {
            const int i = idx / nx, j = idx - i * nx;
            T1[idx] = G[(nu + i) * nw + nu + j];
        }
    }
    tsync();
    // symmetrise (kkt_ocp.py:251)
    for (int idx = tid; idx < nx * nx; idx += T) {
        const int i = idx / nx, j = idx - i * nx;
        P[idx] = 0.5 * (T1[idx] + T1[j * nx + i]);
    }
    tsync();
    return LINALG_OK;
}

// square-root / QR stage (kkt_ocp.py:206-230) and _split_stage_factor
// (:83-91); M~ in WS_MST (extended workspace).  LINALG_OK / NPD / RANK.
__device__ int stage_sqrt(Ctx& c, int n, bool use_qr, bool classical, long long& flops) {
    const int N = c.N;
    const int tid = threadIdx.x, T = blockDim.x;
    const StageInfo& s = c.st[n];
    const int nu = s.nu, nx = s.nx, nw = s.nw, nxn = s.nxn;
    const bool hasW = n < N;
    const double* M = c.w[WS_MST];
    double* W = c.w[WS_T1];     // nxn x nw: W = L_{n+1}' [B A]
    double* LG = c.w[WS_G];     // nw x nw lower
    double* QR = c.w[WS_QR];
    double* LPs = c.w[WS_LPS];
    double* haslp = c.w[WS_HASLP];
    if (hasW) {
        const double* Ln;
        if (haslp[n + 1] != 0.0) {
            Ln = LPs + c.st[n + 1].P_off;
        } else {
            // per-stage QR retry inside a classical sweep (kkt_ocp.py:210-212)
            const double* Pn = c.w[WS_P] + c.st[n + 1].P_off;
            for (int idx = tid; idx < nxn * nxn; idx += T) QR[idx] = Pn[idx];
            tsync();
            flops += (long long)nxn * nxn * nxn / 3;
            if (!team_chol(QR, nxn, nxn, c.iflag)) return LINALG_NPD;
            Ln = QR;
        }
        for (int idx = tid; idx < nxn * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            double a = 0.0;
            for (int k = i; k < nxn; ++k) a = fma(Ln[k * nxn + i], BAget(c, s, k, j), a);
            W[idx] = a;
        }
        flops += 2ll * nxn * nw * nxn;
        tsync();
    }
    if (use_qr) {
        for (int idx = tid; idx < nw * nw; idx += T) LG[idx] = M[idx];
        tsync();
        flops += (long long)nw * nw * nw / 3;
        if (!team_chol(LG, nw, nw, c.iflag)) return LINALG_NPD;
        const int mr = nw + (hasW ? nxn : 0);
        for (int idx = tid; idx < mr * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            QR[idx] = i < nw ? LG[j * nw + i] : W[(i - nw) * nw + j];
        }
        tsync();
        const long long qf = 2ll * mr * nw * nw - (2ll * nw * nw * nw) / 3;
        flops += qf > 0 ? qf : 0;
        if (!team_qr(c, QR, mr, nw)) return LINALG_RANK;
        for (int idx = tid; idx < nw * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            LG[idx] = j <= i ? QR[j * nw + i] : 0.0;
        }
        tsync();
    } else {
        // G = W' W + M~ (matmul_acc(1, W, W, 1, M, transA), kkt_ocp.py:220)
        for (int idx = tid; idx < nw * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            double v = M[idx];
            if (hasW) {
                double a = 0.0;
                for (int k = 0; k < nxn; ++k) a = fma(W[k * nw + i], W[k * nw + j], a);
                v = a + v;
            }
            LG[idx] = v;
        }
        if (hasW) flops += 2ll * nw * nw * nxn;
        tsync();
        flops += (long long)nw * nw * nw / 3;
        if (!team_chol(LG, nw, nw, c.iflag)) return LINALG_NPD;
    }
    // split: L_uu, K = -L_uu^{-T} L_xu', L_P (kkt_ocp.py:83-91)
    double* LP = LPs + s.P_off;
    if (nu) {
        double* L = c.w[WS_L] + s.L_off;
        for (int idx = tid; idx < nu * nu; idx += T) {
            const int i = idx / nu, j = idx - i * nu;
            L[idx] = LG[i * nw + j];
        }
        tsync();
        double* K = c.w[WS_K] + s.K_off;
        for (int j = tid; j < nx; j += T) {
            for (int i = nu - 1; i >= 0; --i) {
                double a = LG[(nu + j) * nw + i];
                for (int k = i + 1; k < nu; ++k) a -= L[k * nu + i] * K[k * nx + j];
                K[i * nx + j] = a / L[i * nu + i];
            }
            for (int i = 0; i < nu; ++i) K[i * nx + j] = -K[i * nx + j];
        }
        flops += (long long)nu * nu * nx;
    }
    for (int idx = tid; idx < nx * nx; idx += T) {
        const int i = idx / nx, j = idx - i * nx;
        LP[idx] = LG[(nu + i) * nw + nu + j];
    }
    if (tid == 0) haslp[n] = 1.0;
    tsync();
    if (classical) {
        // explicit P for the classical stages below (kkt_ocp.py:227-229)
        double* P = c.w[WS_P] + s.P_off;
        for (int idx = tid; idx < nx * nx; idx += T) {
            const int i = idx / nx, j = idx - i * nx;
            const int kk = i < j ? i : j;
            double a = 0.0;
            for (int k = 0; k <= kk; ++k) a = fma(LP[i * nx + k], LP[j * nx + k], a);
            P[idx] = a;
        }
        tsync();
    }
    return LINALG_OK;
}

// ---------------------------------------------------------------------------
// riccati_factor (kkt_ocp.py:142-201; kkt_common.py:57-115).  Returns -1 on
// success, the failing stage on FactorizationFailed; -2 NonPositiveIterate,
// -3 singular soft-slack block, -4 RankDeficient escaping the QR factor.
// sqrt_variant / use_qr / stage_fb need the extended workspace.  flops follow
// the linalg.py counting rules.
// ---------------------------------------------------------------------------
__device__ int factor(Ctx& c, const double* lam, const double* t, double reg, long long& flops,
                      bool sqrt_variant = false, bool use_qr = false, bool stage_fb = false) {
    const KParams& p = *c.p;
    const int N = c.N;
    const int tid = threadIdx.x, T = blockDim.x;
    const double* act = c.w[WS_ACT];
    double* gam = c.w[WS_GAM];
    double* coef = c.w[WS_COEF];
    double* Dl = c.w[WS_DL];
    double* Du = c.w[WS_DU];
    double* G = c.w[WS_G];
    double* Pall = c.w[WS_P];
    const bool sqrt_mode = sqrt_variant || use_qr;
    double* Mb = (sqrt_mode || stage_fb) ? c.w[WS_MST] : G;
    // block_scales for every stage (kkt_common.py:57-97)
    int bad = 0;
    FOR_STAGE_ITEMS(N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double g = 0.0;
            if (act[kk] != 0.0) {
                if (lam[kk] <= 0.0 || t[kk] <= 0.0) bad = 1;
                g = lam[kk] / t[kk];
            }
            gam[kk] = g;
        }
    END_FOR_STAGE_ITEMS
    if (team_or(bad)) return -2;
    if (p.ns_tot) {
        int sing = 0;
        FOR_STAGE_ITEMS(N + 1, p.ns_max, n, j)
            const StageInfo& s = c.st[n];
            if (j < s.ns) {
                const int row = p.idxs[s.is_off + j];
                const double glo = gam[s.c_off + row], gup = gam[s.c_off + s.m + row];
                const double gslo = gam[s.c_off + 2 * s.m + j], gsup = gam[s.c_off + 2 * s.m + s.ns + j];
                const double dl = (fget(c, OCPQP_F_Zl, s, j, 0.0) + glo) + gslo;
                const double du = (fget(c, OCPQP_F_Zu, s, j, 0.0) + gup) + gsup;
                if (dl <= 0.0 || du <= 0.0) sing = 1;
                Dl[s.s_off + j] = dl;
                Du[s.s_off + j] = du;
            }
        END_FOR_STAGE_ITEMS
        if (team_or(sing)) return -3;
    }
    // effective per-row coefficients ge_lo + ge_up
    FOR_STAGE_ITEMS(N + 1, p.m_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.m) {
            double glo = gam[s.c_off + i], gup = gam[s.c_off + s.m + i];
            if (s.ns) {
                const int j = p.row_slack[s.m_off + i];
                if (j >= 0) {
                    const double dl = Dl[s.s_off + j], du = Du[s.s_off + j];
                    glo = glo * (dl - glo) / dl;
                    gup = gup * (du - gup) / du;
                }
            }
            coef[s.m_off + i] = glo + gup;
        }
    END_FOR_STAGE_ITEMS
    tsync();

    for (int n = N; n >= 0; --n) {
        const StageInfo& s = c.st[n];
        const int nw = s.nw, ng = s.ng;
        const double* cf = coef + s.m_off;
        // stage Hessian M~ (kkt_ocp.py:70-80 + add_reduced_hessian kkt_common.py:100-115)
        for (int idx = tid; idx < nw * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            double h = 0.5 * (Mraw(c, s, i, j) + Mraw(c, s, j, i));
            if (i == j) {
                const int kb = p.var_box[s.u_off + i];
                if (kb >= 0) h += cf[kb];
            }
            if (i == j && reg != 0.0 && !ng) h += reg;
            Mb[idx] = h;
        }
        tsync();
        if (ng) {
            rows_syrk(c, s, cf + s.nb, Mb, nw, ng, reg);
            flops += 2ll * nw * nw * ng;
            tsync();
        }
        // _factor_stage with the per-stage QR retry (kkt_ocp.py:180-191)
        const int rc = sqrt_mode ? stage_sqrt(c, n, use_qr, !sqrt_variant, flops)
                                 : stage_classical(c, n, Mb, flops);
        if (rc == LINALG_NPD) {
            if (stage_fb && !use_qr && stage_sqrt(c, n, true, !sqrt_variant, flops) == LINALG_OK)
                continue;
            return n;
        }
        if (rc == LINALG_RANK) return -4;
    }
    // L_P0 = chol(P[0]) (kkt_ocp.py:193-200)
    const int nx0 = c.st[0].nx;
    const bool lp0 = c.w[WS_HASLP] && c.w[WS_HASLP][0] != 0.0;
    if (nx0 && !sqrt_variant && !lp0) {
        double* LP0 = c.w[WS_LP0];
        const double* P0 = Pall + c.st[0].P_off;
        for (int idx = tid; idx < nx0 * nx0; idx += T) LP0[idx] = P0[idx];
        tsync();
        flops += (long long)nx0 * nx0 * nx0 / 3;
        if (!team_chol(LP0, nx0, nx0, c.iflag)) return 0;
    }
    return -1;
}

// ---------------------------------------------------------------------------
// Riccati solve (kkt_ocp.py:254-320) with fold_rhs / recover_block
// (kkt_common.py:118-163).  r_m is either rm_ext (masked by act) or computed
// as (lam t - tau) + corr * dlam_aff dt_aff on active slots (solver.py:207-258).
// Returns nonzero when the step contains a non-finite entry.
// ---------------------------------------------------------------------------
struct RmSpec {
    const double* ext;    // explicit r_m (Newton-step entry) or nullptr
    double tau;           // centering shift
    const double* dlam;   // affine step for the corrector term, or nullptr
    const double* dt;
    int absf = 0;         // absolute formulation: 1 affine (-comp), 2 direction (- 2 comp)
    double* out = nullptr;  // materialise the active r_m (0 elsewhere) for refinement
};

__device__ int solve(Ctx& c, const double* lam, const double* t, const double* r_g,
                     const double* r_b, const double* r_d, const RmSpec& rm,
                     double* dy, double* dpi, double* dlam, double* dt, long long& flops) {
    const KParams& p = *c.p;
    const int N = c.N;
    const int tid = threadIdx.x, T = blockDim.x;
    const double* act = c.w[WS_ACT];
    const double* gam = c.w[WS_GAM];
    const double* Dl = c.w[WS_DL];
    const double* Du = c.w[WS_DU];
    double* wall = c.w[WS_WALL];
    double* rtsl = c.w[WS_RTSL];
    double* rtsu = c.w[WS_RTSU];
    double* crow = c.w[WS_CROW];
    double* frow = c.w[WS_ROWV];
    double* rhat = c.w[WS_RHAT];
    const double* Pall = c.w[WS_P];
    const double* Kall = c.w[WS_K];
    const double* Lall = c.w[WS_L];
    double* pv = c.w[WS_PV];
    double* kff = c.w[WS_KFF];
    double* vec = c.w[WS_VEC];
    const double* haslp = c.w[WS_HASLP];   // nullptr without the extended workspace
    const double* LPs = c.w[WS_LPS];
    int nonfinite = 0;
    // fold: w_all = act ? (lam r_d - r_m) / t : 0
    FOR_STAGE_ITEMS(N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double w = 0.0, rmk = 0.0;
            if (act[kk] != 0.0) {
                if (rm.ext) {
                    rmk = rm.ext[kk];
                } else if (rm.absf == 1) {
                    rmk = -(lam[kk] * t[kk]);
                } else {
                    const double comp = lam[kk] * t[kk];
                    rmk = comp - rm.tau;
                    if (rm.dlam) rmk = rmk + rm.dlam[kk] * rm.dt[kk];
                    if (rm.absf == 2) rmk = rmk - 2.0 * comp;
                }
                w = (lam[kk] * r_d[kk] - rmk) / t[kk];
            }
            wall[kk] = w;
            if (rm.out) rm.out[kk] = rmk;
        }
    END_FOR_STAGE_ITEMS
    tsync();
    if (p.ns_tot) {
        FOR_STAGE_ITEMS(N + 1, p.ns_max, n, j)
            const StageInfo& s = c.st[n];
            if (j < s.ns) {
                const int row = p.idxs[s.is_off + j];
                const int c0 = s.c_off, m = s.m;
                const double a = (r_g[p.nv + s.s_off + j] - wall[c0 + row]) - wall[c0 + 2 * m + j];
                const double b = (r_g[p.nv + p.ns_tot + s.s_off + j] - wall[c0 + m + row]) -
                                 wall[c0 + 2 * m + s.ns + j];
                rtsl[s.s_off + j] = a;
                rtsu[s.s_off + j] = b;
            }
        END_FOR_STAGE_ITEMS
        tsync();
    }
    FOR_STAGE_ITEMS(N + 1, p.m_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.m) {
            crow[s.m_off + i] = wall[s.c_off + i] - wall[s.c_off + s.m + i];
            double fr = 0.0;
            if (s.ns) {
                const int j = p.row_slack[s.m_off + i];
                if (j >= 0)
                    fr = gam[s.c_off + i] * rtsl[s.s_off + j] / Dl[s.s_off + j] -
                         gam[s.c_off + s.m + i] * rtsu[s.s_off + j] / Du[s.s_off + j];
            }
            frow[s.m_off + i] = fr;
        }
    END_FOR_STAGE_ITEMS
    tsync();
    FOR_STAGE_ITEMS(N + 1, p.nw_max, n, j)
        const StageInfo& s = c.st[n];
        if (j < s.nw) {
            double r = r_g[s.u_off + j] - rows_t(c, s, j, crow + s.m_off);
            if (s.ns) r = r - rows_t(c, s, j, frow + s.m_off);
            rhat[s.u_off + j] = r;
        }
    END_FOR_STAGE_ITEMS
    tsync();
    // backward sweep (kkt_ocp.py:276-289)
    double* win = vec;                 // [nw]  (rr | rq)
    double* e = vec + p.nw_max;        // [nx']
    double* z = vec + p.nw_max + p.nx_max;  // serial scratch [max(nu, nx0)]
    for (int n = N; n >= 0; --n) {
        const StageInfo& s = c.st[n];
        const int nu = s.nu, nx = s.nx, nw = s.nw, nxn = s.nxn;
        if (n < N) {
            const double* rb = r_b + s.pi_off;
            const double* pvnext = pv + (c.st[n + 1].pv_off);
            if (haslp && haslp[n + 1] != 0.0) {
                // p_apply = L_P (L_P' v) (kkt_ocp.py:110-113)
                const double* Lp = LPs + c.st[n + 1].P_off;
                for (int i = tid; i < nxn; i += T) {
                    double a = 0.0;
                    for (int k = i; k < nxn; ++k) a = fma(Lp[k * nxn + i], rb[k], a);
                    z[i] = a;
                }
                tsync();
                for (int i = tid; i < nxn; i += T) {
                    double a = 0.0;
                    for (int k = 0; k <= i; ++k) a = fma(Lp[i * nxn + k], z[k], a);
                    e[i] = a + pvnext[i];
                }
            } else {
                const double* Pn = Pall + c.st[n + 1].P_off;
                for (int i = tid; i < nxn; i += T) {
                    double a = 0.0;
                    for (int k = 0; k < nxn; ++k) a = fma(Pn[i * nxn + k], rb[k], a);
                    e[i] = a + pvnext[i];
                }
            }
            tsync();
        }
        for (int j = tid; j < nw; j += T) {
            double a = rhat[s.u_off + j];
            if (n < N) {
                double b = 0.0;
                for (int k = 0; k < nxn; ++k) b = fma(BAget(c, s, k, j), e[k], b);
                a = a + b;
            }
            win[j] = a;
        }
        tsync();
        const double* K = Kall + s.K_off;
        double* pvc = pv + s.pv_off;
        for (int i = tid; i < nx; i += T) {
            double a = 0.0;
            for (int k = 0; k < nu; ++k) a = fma(K[k * nx + i], win[k], a);
            pvc[i] = win[nu + i] + a;
        }
        if (nu && nu <= 32 && tid >= T - 32) {
            warp_cho_solve(Lall + s.L_off, nu, win, kff + s.kff_off, -1.0);
        } else if (nu > 32 && nu <= 128 && tid >= T - 32) {
            warp_cho_solve4(Lall + s.L_off, nu, win, kff + s.kff_off, -1.0);
        } else if (nu > 128 && tid == T - 1) {
            const double* L = Lall + s.L_off;
            for (int i = 0; i < nu; ++i) z[i] = win[i];
            cho_solve_serial(L, nu, z);
            double* kf = kff + s.kff_off;
            for (int i = 0; i < nu; ++i) kf[i] = -z[i];
        }
        if (nu) flops += 2ll * nu * nu;
        tsync();
    }
    // x0 step (kkt_ocp.py:292)
    const int nx0 = c.st[0].nx;
    if (nx0) {
        const double* LP0 = (haslp && haslp[0] != 0.0) ? LPs + c.st[0].P_off : c.w[WS_LP0];
        if (nx0 <= 32) {
            if (tid < 32) warp_cho_solve(LP0, nx0, pv + c.st[0].pv_off, dy + c.st[0].x_off, -1.0);
        } else if (nx0 <= 128) {
            if (tid < 32) warp_cho_solve4(LP0, nx0, pv + c.st[0].pv_off, dy + c.st[0].x_off, -1.0);
        } else if (tid == 0) {
            for (int i = 0; i < nx0; ++i) z[i] = pv[c.st[0].pv_off + i];
            cho_solve_serial(LP0, nx0, z);
            for (int i = 0; i < nx0; ++i) dy[c.st[0].x_off + i] = -z[i];
        }
        flops += 2ll * nx0 * nx0;
        tsync();
    }
    // forward rollout (kkt_ocp.py:293-305); dpi is filled afterwards in parallel
    for (int n = 0; n <= N; ++n) {
        const StageInfo& s = c.st[n];
        const int nu = s.nu, nx = s.nx, nxn = s.nxn;
        const double* xi = dy + s.x_off;
        if (nu) {
            const double* K = Kall + s.K_off;
            const double* kf = kff + s.kff_off;
            for (int i = tid; i < nu; i += T) {
                double a = 0.0;
                for (int k = 0; k < nx; ++k) a = fma(K[i * nx + k], xi[k], a);
                dy[s.u_off + i] = a + kf[i];
            }
            tsync();
        }
        if (n < N) {
            const double* du = dy + s.u_off;
            const double* rb = r_b + s.pi_off;
            double* xn = dy + c.st[n + 1].x_off;
            for (int i = tid; i < nxn; i += T) {
                double ax = 0.0, bu = 0.0;
                for (int k = 0; k < nx; ++k) ax = fma(Aget(c, s, i, k), xi[k], ax);
                for (int k = 0; k < nu; ++k) bu = fma(Bget(c, s, i, k), du[k], bu);
                xn[i] = (ax + bu) + rb[i];
            }
            tsync();
        }
    }
    // dpi_n = P[n+1] x_{n+1} + pv[n+1]; square-root stages: L_P (L_P' x)
    double* zt = c.w[WS_ZT];
    if (haslp) {
        FOR_STAGE_ITEMS(N, p.nx_max, n, i)
            const StageInfo& s = c.st[n];
            if (i < s.nxn && haslp[n + 1] != 0.0) {
                const StageInfo& s1 = c.st[n + 1];
                const double* Lp = LPs + s1.P_off;
                const double* xn = dy + s1.x_off;
                double a = 0.0;
                for (int k = i; k < s.nxn; ++k) a = fma(Lp[k * s.nxn + i], xn[k], a);
                zt[s.pi_off + i] = a;
            }
        END_FOR_STAGE_ITEMS
        tsync();
    }
    FOR_STAGE_ITEMS(N, p.nx_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.nxn) {
            const StageInfo& s1 = c.st[n + 1];
            const double* xn = dy + s1.x_off;
            double a = 0.0;
            if (haslp && haslp[n + 1] != 0.0) {
                const double* Lp = LPs + s1.P_off;
                const double* zz = zt + s.pi_off;
                for (int k = 0; k <= i; ++k) a = fma(Lp[i * s.nxn + k], zz[k], a);
            } else {
                const double* Pn = Pall + s1.P_off;
                for (int k = 0; k < s.nxn; ++k) a = fma(Pn[i * s.nxn + k], xn[k], a);
            }
            const double v = a + pv[s1.pv_off + i];
            dpi[s.pi_off + i] = v;
            if (!isfinite(v)) nonfinite = 1;
        }
    END_FOR_STAGE_ITEMS
    for (int i = tid; i < p.nv; i += T)
        if (!isfinite(dy[i])) nonfinite = 1;
    // recover_block (kkt_common.py:140-163)
    double* rowv = c.w[WS_ROWV];
    rows_values(c, dy, rowv);
    tsync();
    if (p.ns_tot) {
        FOR_STAGE_ITEMS(N + 1, p.ns_max, n, j)
            const StageInfo& s = c.st[n];
            if (j < s.ns) {
                const int row = p.idxs[s.is_off + j];
                const double base = rowv[s.m_off + row];
                const double dsl = (-rtsl[s.s_off + j] - gam[s.c_off + row] * base) / Dl[s.s_off + j];
                const double dsu = (-rtsu[s.s_off + j] + gam[s.c_off + s.m + row] * base) / Du[s.s_off + j];
                dy[p.nv + s.s_off + j] = dsl;
                dy[p.nv + p.ns_tot + s.s_off + j] = dsu;
                if (!isfinite(dsl) || !isfinite(dsu)) nonfinite = 1;
            }
        END_FOR_STAGE_ITEMS
        tsync();
    }
    FOR_STAGE_ITEMS(N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double dl = 0.0, dtt = 0.0;
            if (act[kk] != 0.0) {
                const double cy = slot_cy(c, s, k, rowv, dy);
                dl = wall[kk] - gam[kk] * cy;
                dtt = -r_d[kk] + cy;
            }
            dlam[kk] = dl;
            dt[kk] = dtt;
            if (!isfinite(dl) || !isfinite(dtt)) nonfinite = 1;
        }
    END_FOR_STAGE_ITEMS
    return team_or(nonfinite);
}

// ---------------------------------------------------------------------------
// IPM vector kernels (ipm_core.py:201-272)
// ---------------------------------------------------------------------------
// max_step: largest alpha in (0,1] keeping lam, t >= 0, scaled by ftb
// The step is (dlam, dt), or (dlam - lam, dt - t) with `absd` (the absolute
// formulation's solution minus the iterate, ipm_core.py:275-283).
__device__ double max_step(Ctx& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double ftb, bool absd = false) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    double ratio = INFINITY;
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
        if (act[k] != 0.0) {
            const double dl = absd ? dlam[k] - lam[k] : dlam[k];
            const double dd = absd ? dt[k] - t[k] : dt[k];
            if (dl < 0.0) ratio = fmin(ratio, -lam[k] / dl);
            if (dd < 0.0) ratio = fmin(ratio, -t[k] / dd);
        }
    }
    ratio = team_min(ratio, c.red);
    return fmin(1.0, ftb * ratio);
}

// duality measure at lam + alpha dlam, t + alpha dt
__device__ double trial_mu(Ctx& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double alpha, bool absd = false) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    double s = 0.0;
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x)
        if (act[k] != 0.0) {
            const double dl = absd ? dlam[k] - lam[k] : dlam[k];
            const double dd = absd ? dt[k] - t[k] : dt[k];
            s += (lam[k] + alpha * dl) * (t[k] + alpha * dd);
        }
    s = team_sum(s, c.red);
    return c.n_act > 0.0 ? s / c.n_act : 0.0;
}

// every entry of the four vectors finite (QpSolution.isfinite, view.py:666-672)
__device__ bool team_finite4(Ctx& c, const double* y, const double* pi, const double* lam,
                             const double* t) {
    const KParams& p = *c.p;
    int bad = 0;
    for (int i = threadIdx.x; i < p.ny; i += blockDim.x) bad |= !isfinite(y[i]);
    for (int i = threadIdx.x; i < p.ne; i += blockDim.x) bad |= !isfinite(pi[i]);
    for (int i = threadIdx.x; i < p.nc; i += blockDim.x) bad |= !isfinite(lam[i]) || !isfinite(t[i]);
    return !team_or(bad);
}

// x -= base over the four vectors (recover_step_absolute)
__device__ void sub4(Ctx& c, double* y, double* pi, double* lam, double* t, const double* by,
                     const double* bpi, const double* blam, const double* bt) {
    const KParams& p = *c.p;
    for (int i = threadIdx.x; i < p.ny; i += blockDim.x) y[i] = y[i] - by[i];
    for (int i = threadIdx.x; i < p.ne; i += blockDim.x) pi[i] = pi[i] - bpi[i];
    for (int i = threadIdx.x; i < p.nc; i += blockDim.x) {
        lam[i] = lam[i] - blam[i];
        t[i] = t[i] - bt[i];
    }
    tsync();
}

__device__ void copy4(Ctx& c, double* y, double* pi, double* lam, double* t, const double* sy,
                      const double* spi, const double* slam, const double* st) {
    const KParams& p = *c.p;
    for (int i = threadIdx.x; i < p.ny; i += blockDim.x) y[i] = sy[i];
    for (int i = threadIdx.x; i < p.ne; i += blockDim.x) pi[i] = spi[i];
    for (int i = threadIdx.x; i < p.nc; i += blockDim.x) {
        lam[i] = slam[i];
        t[i] = st[i];
    }
    tsync();
}

// max |kkt_rhs_flat(r_g, r_b, r_d, r_m)| with NaN propagation (solver.py:331-333)
__device__ double rhs_norm(Ctx& c, const double* rg, const double* rb, const double* rd,
                           const double* rm) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    AbsMax a;
    for (int i = threadIdx.x; i < p.ny; i += blockDim.x) a.add(rg[i]);
    for (int i = threadIdx.x; i < p.ne; i += blockDim.x) a.add(rb[i]);
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
        a.add(act[k] != 0.0 ? rd[k] : 0.0);
        a.add(act[k] != 0.0 ? rm[k] : 0.0);
    }
    return team_absmax(a, c.red);
}

// refinement residual kkt_apply_vec(delta) + rhs into WS_RF* (ipm_core.py:335);
// returns its max |.|
__device__ double refine_residual(Ctx& c, const double* lam, const double* t, const double* rg,
                                  const double* rb, const double* rd, const double* rm,
                                  const double* dy, const double* dpi, const double* dl,
                                  const double* dt) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    double *ry = c.w[WS_RFY], *rpi = c.w[WS_RFPI], *rl = c.w[WS_RFLAM], *rt = c.w[WS_RFT];
    residuals(c, dy, dpi, dl, dt, ry, rpi, rl, rt, lam, t);
    AbsMax a;
    for (int i = threadIdx.x; i < p.ny; i += blockDim.x) { ry[i] = ry[i] + rg[i]; a.add(ry[i]); }
    for (int i = threadIdx.x; i < p.ne; i += blockDim.x) { rpi[i] = rpi[i] + rb[i]; a.add(rpi[i]); }
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
        rl[k] = rl[k] + (act[k] != 0.0 ? rd[k] : 0.0);
        rt[k] = rt[k] + (act[k] != 0.0 ? rm[k] : 0.0);
        a.add(rl[k]);
        a.add(rt[k]);
    }
    return team_absmax(a, c.red);   // includes the barriers that publish WS_RF*
}

// ---------------------------------------------------------------------------
// context construction
// ---------------------------------------------------------------------------
__device__ void make_ctx(Ctx& c, const KParams& p, int q, double* gslot, double* smem,
                         double* red, int* iflag) {
    double* gslot2 = p.ws2 ? p.ws2 + (long long)blockIdx.x * p.ws2_slot : nullptr;
    c.p = &p;
    c.st = p.st;
    c.N = p.N;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f)
        c.f[f] = p.f[f] ? p.f[f] + (long long)q * p.bs[f] : nullptr;
    for (int b = 0; b < WS_EXT0; ++b)
        c.w[b] = ((p.smem_mask >> b) & 1u) ? smem + p.smem_off[b] : gslot + p.ws_off[b];
    for (int b = WS_EXT0; b < WS_NUM; ++b) c.w[b] = gslot2 ? gslot2 + p.ws_off[b] : nullptr;
    c.red = red;
    c.iflag = iflag;
    c.n_act = 0.0;
}

// initial iterate (solver.py:113-142)
__device__ void init_iterate(Ctx& c, const OcpIpmArgC& arg, double* y, double* pi,
                             double* lam, double* t) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    const double* dvec = c.w[WS_DVEC];
    double* rowv = c.w[WS_ROWV];
    const int warm = arg.warm_start;
    if (warm == 0) {
        for (int i = threadIdx.x; i < p.ny; i += blockDim.x) y[i] = 0.0;
    }
    if (warm != 2) {
        for (int i = threadIdx.x; i < p.ne; i += blockDim.x) pi[i] = 0.0;
    }
    tsync();
    rows_values(c, y, rowv);
    tsync();
    double floor = arg.t0;
    if (warm == 2) {
        // floor = max(1e-8, t_min, min(1, max(gap_d, gap_b)))  (solver.py:125-134)
        double gd = 0.0, gb = 0.0;
        FOR_STAGE_ITEMS(c.N + 1, p.nc_max, n, k)
            const StageInfo& s = c.st[n];
            if (k < s.nc) {
                const int kk = s.c_off + k;
                if (act[kk] != 0.0) gd = fmax(gd, dvec[kk] - slot_cy(c, s, k, rowv, y));
            }
        END_FOR_STAGE_ITEMS
        FOR_STAGE_ITEMS(c.N, p.nx_max, n, i)
            const StageInfo& s = c.st[n];
            if (i < s.nxn) {
                const double* u = y + s.u_off;
                const double* x = y + s.x_off;
                double ax = 0.0, bu = 0.0;
                for (int k = 0; k < s.nx; ++k) ax = fma(Aget(c, s, i, k), x[k], ax);
                for (int k = 0; k < s.nu; ++k) bu = fma(Bget(c, s, i, k), u[k], bu);
                const double r = -((y[c.st[n + 1].x_off + i] - ax) - bu) + fget(c, OCPQP_F_b, s, i, 0.0);
                gb = fmax(gb, fabs(r));
            }
        END_FOR_STAGE_ITEMS
        gd = team_max(gd, c.red);
        gb = team_max(gb, c.red);
        floor = fmax(fmax(1e-8, arg.t_min), fmin(1.0, fmax(gd, gb)));
    }
    const double lfloor = fmax(1e-8, arg.lam_min);
    FOR_STAGE_ITEMS(c.N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double tv = 0.0, lv = 0.0;
            if (act[kk] != 0.0) {
                const double cy = (warm == 0) ? 0.0 : slot_cy(c, s, k, rowv, y);
                tv = fmax(cy - dvec[kk], floor);
                lv = (warm == 2) ? fmax(lam[kk], lfloor) : arg.mu0 / tv;
            }
            t[kk] = tv;
            lam[kk] = lv;
        }
    END_FOR_STAGE_ITEMS
    tsync();
}

// ---------------------------------------------------------------------------
// iterative_refinement (ipm_core.py:317-359) through _refine (solver.py:311-321):
// refines the direction d = (dy, dpi, dl, dt) in place against the rhs
// (rg, rb, rd, rm; rm materialised, 0 on inactive slots).  The corrections are
// solved into (cy, cpi, cl, ct).  Returns the final (best) residual norm.
// ---------------------------------------------------------------------------
__device__ __noinline__ double refine(Ctx& c, const double* lam, const double* t, const double* rg,
                         const double* rb, const double* rd, const double* rm, double* dy,
                         double* dpi, double* dl, double* dt, double* cy, double* cpi, double* cl,
                         double* ct, int max_steps, double stop_ratio, long long& flops) {
    const KParams& p = *c.p;
    const double rn = rhs_norm(c, rg, rb, rd, rm);
    const double sc = isnan(rn) ? 1.0 : fmax(1.0, rn);
    double best = refine_residual(c, lam, t, rg, rb, rd, rm, dy, dpi, dl, dt);
    if (max_steps <= 0 || best <= stop_ratio * sc) return best;
    double *by = c.w[WS_BY], *bpi = c.w[WS_BPI], *bl = c.w[WS_BLAM], *bt = c.w[WS_BT];
    copy4(c, by, bpi, bl, bt, dy, dpi, dl, dt);
    double norm = best;
    int grew = 0;
    for (int st = 0; st < max_steps; ++st) {
        RmSpec rs{c.w[WS_RFT], 0.0, nullptr, nullptr};
        solve(c, lam, t, c.w[WS_RFY], c.w[WS_RFPI], c.w[WS_RFLAM], rs, cy, cpi, cl, ct, flops);
        for (int i = threadIdx.x; i < p.ny; i += blockDim.x) dy[i] = dy[i] + cy[i];
        for (int i = threadIdx.x; i < p.ne; i += blockDim.x) dpi[i] = dpi[i] + cpi[i];
        for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
            dl[k] = dl[k] + cl[k];
            dt[k] = dt[k] + ct[k];
        }
        tsync();
        const double nn = refine_residual(c, lam, t, rg, rb, rd, rm, dy, dpi, dl, dt);
        if (nn < best) {
            copy4(c, by, bpi, bl, bt, dy, dpi, dl, dt);
            best = nn;
        }
        grew = (nn >= norm) ? grew + 1 : 0;
        norm = nn;
        if (nn <= stop_ratio * sc) break;
        if (grew >= 2) break;
    }
    copy4(c, dy, dpi, dl, dt, by, bpi, bl, bt);
    return best;
}

// ---------------------------------------------------------------------------
// _factor_with_policy (solver.py:145-164): -1 ok (used_qr set), >= 0 Failure,
// < -1 an exception of the reference (NonPositiveIterate / SingularSlackBlock /
// RankDeficient).
// ---------------------------------------------------------------------------
__device__ int factor_policy(Ctx& c, const OcpIpmArgC& arg, const double* lam, const double* t,
                             long long& flops, bool& used_qr) {
    bool use_qr = arg.use_qr_always != 0;
    const bool sv = arg.riccati_variant != 0, fb = arg.use_qr_fallback != 0;
    int fs = factor(c, lam, t, arg.reg_prim, flops, sv, use_qr, fb);
    if (fs == -1) { used_qr = use_qr; return -1; }
    if (fs < -1) return fs;
    if (fb && !use_qr) {
        fs = factor(c, lam, t, arg.reg_prim, flops, sv, true, fb);
        if (fs == -1) { used_qr = true; return -1; }
        if (fs < -1) return fs;
        use_qr = true;
    }
    const double reg2 = arg.reg_prim > 0.0 ? 2.0 * arg.reg_prim : 1e-8;
    fs = factor(c, lam, t, reg2, flops, sv, use_qr, fb);
    if (fs == -1) used_qr = use_qr;
    return fs;
}

__device__ __forceinline__ int raise_status(int fs) {
    return fs == -2 ? OCPQP_STATUS_NONPOSITIVE_ITERATE
         : fs == -3 ? OCPQP_STATUS_SINGULAR_SLACK
         : fs == -4 ? OCPQP_STATUS_RANK_DEFICIENT : OCPQP_STATUS_FAILURE;
}

// ---------------------------------------------------------------------------
// the fused IPM solve of one QP (solver.py:180-308), every mode: speed
// (classical or square-root Riccati), balance / robust (QR array algorithm,
// fallback ladder, iterative refinement), speed_abs (absolute formulation)
// ---------------------------------------------------------------------------
__device__ void ipm_one(Ctx& c, const SolveParams& sp, int q) {
    const KParams& p = *c.p;
    const OcpIpmArgC& arg = sp.arg;
    double* y = sp.y + (long long)q * p.ny;
    double* pi = sp.pi + (long long)q * p.ne;
    double* lam = sp.lam + (long long)q * p.nc;
    double* t = sp.t + (long long)q * p.nc;
    double* trace = sp.trace ? sp.trace + (long long)q * arg.iter_max * 8 : nullptr;
    double* r_g = c.w[WS_RG];
    double* r_b = c.w[WS_RB];
    double* r_d = c.w[WS_RD];
    double *ay = c.w[WS_AFF_Y], *api = c.w[WS_AFF_PI], *alam = c.w[WS_AFF_LAM], *at = c.w[WS_AFF_T];
    double *dy = c.w[WS_DIR_Y], *dpi = c.w[WS_DIR_PI], *dlam = c.w[WS_DIR_LAM], *dt = c.w[WS_DIR_T];
    const double* act = c.w[WS_ACT];
    const bool absf = arg.abs_form != 0, crp = arg.comp_res_pred != 0;

    setup_constraints(c);
    // an escape from the team kernel resumes at its iteration and iterate
    const long long* meta = p.esc_meta ? p.esc_meta + 3ll * q : nullptr;
    if (!meta) init_iterate(c, arg, y, pi, lam, t);
    if (absf) {
        // g_full = view.grad(), b_vec = view.b() (solver.py:184-186): the residual
        // operators at the zero point
        double *zy = c.w[WS_BY], *zpi = c.w[WS_BPI], *zl = c.w[WS_BLAM], *zt = c.w[WS_BT];
        for (int i = threadIdx.x; i < p.ny; i += blockDim.x) zy[i] = 0.0;
        for (int i = threadIdx.x; i < p.ne; i += blockDim.x) zpi[i] = 0.0;
        for (int i = threadIdx.x; i < p.nc; i += blockDim.x) { zl[i] = 0.0; zt[i] = 0.0; }
        tsync();
        residuals(c, zy, zpi, zl, zt, c.w[WS_GF], c.w[WS_BF], c.w[WS_RFLAM], nullptr);
    }
    const double* rg = absf ? c.w[WS_GF] : r_g;
    const double* rb = absf ? c.w[WS_BF] : r_b;
    const double* rd = absf ? c.w[WS_DVEC] : r_d;

    long long flops = meta ? meta[1] : 0;
    double alpha_last = meta ? __longlong_as_double(meta[2]) : 1.0;
    int it = meta ? (int)meta[0] : 0;
    int status = -1;
    ResNorms res{qnan(), qnan(), qnan(), qnan(), qnan()};
    while (true) {
        double mu;
        if (crp) {
            res = residuals(c, y, pi, lam, t, r_g, r_b, r_d, nullptr);
            mu = res.mu;
        } else {
            // duality_measure of the iterate (ipm_core.py:201-214)
            double sm = 0.0;
            for (int k = threadIdx.x; k < p.nc; k += blockDim.x)
                if (act[k] != 0.0) sm += lam[k] * t[k];
            sm = team_sum(sm, c.red);
            mu = c.n_act > 0.0 ? sm / c.n_act : 0.0;
            if (!team_finite4(c, y, pi, lam, t)) { status = OCPQP_STATUS_NAN; break; }
        }
        // check_termination (ipm_core.py:286-314)
        if (crp && (!isfinite(res.g) || !isfinite(res.b) || !isfinite(res.d) || !isfinite(res.m))) {
            status = OCPQP_STATUS_NAN;
        } else if (!isfinite(mu)) {
            status = OCPQP_STATUS_NAN;
        } else if (alpha_last < arg.alpha_min) {
            status = OCPQP_STATUS_MINSTEP;
        } else if (mu <= arg.tol_comp &&
                   (arg.mu_only_exit || !crp ||
                    (res.g <= arg.tol_stat && res.b <= arg.tol_eq && res.d <= arg.tol_ineq &&
                     res.m <= arg.tol_comp))) {
            status = OCPQP_STATUS_SUCCESS;
        } else if (it >= arg.iter_max) {
            status = OCPQP_STATUS_MAXITER;
        }
        if (status >= 0) break;
        bool used_qr = false;
        const int fs = factor_policy(c, arg, lam, t, flops, used_qr);
        if (fs != -1) { status = raise_status(fs); break; }
        // affine prediction (solver.py:207-226)
        RmSpec ra{nullptr, 0.0, nullptr, nullptr, absf ? 1 : 0,
                  arg.itref_pred_max > 0 ? c.w[WS_RMD] : nullptr};
        int nf = solve(c, lam, t, rg, rb, rd, ra, ay, api, alam, at, flops);
        if (arg.itref_pred_max > 0) {
            tsync();
            refine(c, lam, t, rg, rb, rd, c.w[WS_RMD], ay, api, alam, at, dy, dpi, dlam, dt,
                   arg.itref_pred_max, arg.itref_stop_ratio, flops);
        }
        if (absf) {
            sub4(c, ay, api, alam, at, y, pi, lam, t);
            nf = !team_finite4(c, ay, api, alam, at);
        } else if (arg.itref_pred_max > 0) {
            nf = !team_finite4(c, ay, api, alam, at);
        }
        if (nf) { status = OCPQP_STATUS_NAN; break; }
        const double alpha_aff = max_step(c, lam, t, alam, at, 1.0);
        const double mu_aff = trial_mu(c, lam, t, alam, at, alpha_aff);
        double sigma = 0.0;
        if (mu > 0.0) sigma = fmin(1.0, fmax(0.0, pow(mu_aff / mu, 3.0)));
        const double tau = sigma * mu;
        // combined predictor-corrector direction; rm_dir materialised for refinement
        const bool refine_dir = arg.itref_corr_max > 0;
        double* rmd = refine_dir ? c.w[WS_RMD] : nullptr;
        RmSpec rs{nullptr, tau, nullptr, nullptr, absf ? 2 : 0, rmd};
        if (arg.pred_corr) { rs.dlam = alam; rs.dt = at; }
        nf = solve(c, lam, t, rg, rb, rd, rs, dy, dpi, dlam, dt, flops);
        if (arg.pred_corr && arg.cond_pred_corr) {
            const double a_t = max_step(c, lam, t, dlam, dt, 1.0, absf);
            const double mu_t = trial_mu(c, lam, t, dlam, dt, a_t, absf);
            if (!(mu_t <= arg.corr_ratio * mu_aff)) {
                RmSpec rc{nullptr, tau, nullptr, nullptr, absf ? 2 : 0, rmd};
                nf = solve(c, lam, t, rg, rb, rd, rc, dy, dpi, dlam, dt, flops);
            }
        }
        if (refine_dir) {
            tsync();
            double ir = refine(c, lam, t, rg, rb, rd, rmd, dy, dpi, dlam, dt, ay, api, alam, at,
                               arg.itref_corr_max, arg.itref_stop_ratio, flops);
            if (arg.use_qr_fallback && !used_qr) {
                const double rn = rhs_norm(c, rg, rb, rd, rmd);
                if (ir > arg.qr_fallback_ratio * (isnan(rn) ? 1.0 : fmax(1.0, rn))) {
                    // refactor by the QR array algorithm (solver.py:266-280)
                    const int f2 = factor(c, lam, t, arg.reg_prim, flops, arg.riccati_variant != 0,
                                          true, arg.use_qr_fallback != 0);
                    if (f2 == -1) {
                        RmSpec rx{rmd, 0.0, nullptr, nullptr};
                        solve(c, lam, t, rg, rb, rd, rx, dy, dpi, dlam, dt, flops);
                        tsync();
                        refine(c, lam, t, rg, rb, rd, rmd, dy, dpi, dlam, dt, ay, api, alam, at,
                               arg.itref_corr_max, arg.itref_stop_ratio, flops);
                    } else if (f2 < -1) {
                        status = raise_status(f2);
                        break;
                    }
                }
            }
        }
        if (absf) sub4(c, dy, dpi, dlam, dt, y, pi, lam, t);
        if (absf || refine_dir) nf = !team_finite4(c, dy, dpi, dlam, dt);
        if (nf) { status = OCPQP_STATUS_NAN; break; }
        const double alpha = max_step(c, lam, t, dlam, dt, arg.ftb);
        // update_iterate_delta (ipm_core.py:253-272)
        for (int i = threadIdx.x; i < p.ny; i += blockDim.x) y[i] += alpha * dy[i];
        for (int i = threadIdx.x; i < p.ne; i += blockDim.x) pi[i] += alpha * dpi[i];
        for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
            double lv = lam[k] + alpha * dlam[k];
            double tv = t[k] + alpha * dt[k];
            if (act[k] != 0.0) {
                lv = fmax(lv, arg.lam_min);
                tv = fmax(tv, arg.t_min);
            }
            lam[k] = lv;
            t[k] = tv;
        }
        if (trace && threadIdx.x == 0 && it < arg.iter_max) {
            double* tr = trace + (long long)it * 8;
            tr[0] = alpha_aff; tr[1] = alpha; tr[2] = mu; tr[3] = sigma;
            tr[4] = res.g; tr[5] = res.b; tr[6] = res.d; tr[7] = res.m;
        }
        tsync();
        alpha_last = alpha;
        ++it;
    }
    // final residuals (solver.py:300): with per-iteration residuals every exit
    // leaves the loop before the iterate changes, so they are the last ones
    if (!crp) res = residuals(c, y, pi, lam, t, r_g, r_b, r_d, nullptr);
    if (threadIdx.x == 0) {
        sp.status[q] = status;
        sp.iters[q] = it;
        double* r = sp.res + (long long)q * 5;
        r[0] = res.g; r[1] = res.b; r[2] = res.d; r[3] = res.m; r[4] = res.mu;
        sp.flops[q] = flops;
    }
}

__global__ void __launch_bounds__(512) k_ipm_solve(KParams p, SolveParams sp) {
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ int iflag[4];
    __shared__ int s_q;
    double* gslot = p.ws + (long long)blockIdx.x * p.ws_slot;
    while (true) {
        if (threadIdx.x == 0) {
            const int i = atomicAdd(p.counter, 1);
            // escape list of the team kernel (balance mode), or every QP
            s_q = p.esc_list ? (i < *p.esc_count ? p.esc_list[i] : p.B) : i;
        }
        tsync();
        const int q = s_q;
        tsync();
        if (q >= p.B) break;
        Ctx c;
        make_ctx(c, p, q, gslot, smem, red, iflag);
        ipm_one(c, sp, q);
        tsync();
    }
}

// Newton step at a given iterate (riccati_factor + solve), static QP -> slot map
__global__ void __launch_bounds__(512) k_newton_step(KParams p, double reg, const double* lam0,
                                                     const double* t0, const double* rg,
                                                     const double* rb, const double* rd,
                                                     const double* rm, double* sy, double* spi,
                                                     double* slam, double* st_, int* fail) {
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ int iflag[4];
    double* gslot = p.ws + (long long)blockIdx.x * p.ws_slot;
    for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
        Ctx c;
        make_ctx(c, p, q, gslot, smem, red, iflag);
        setup_constraints(c);
        const double* lam = lam0 + (long long)q * p.nc;
        const double* t = t0 + (long long)q * p.nc;
        long long fl = 0;
        const int fs = factor(c, lam, t, reg, fl);
        double* dy = sy + (long long)q * p.ny;
        double* dpi = spi + (long long)q * p.ne;
        double* dl = slam + (long long)q * p.nc;
        double* dtt = st_ + (long long)q * p.nc;
        if (fs == -1) {
            RmSpec rs{rm + (long long)q * p.nc, 0.0, nullptr, nullptr};
            solve(c, lam, t, rg + (long long)q * p.ny, rb + (long long)q * p.ne,
                  rd + (long long)q * p.nc, rs, dy, dpi, dl, dtt, fl);
        } else {
            for (int i = threadIdx.x; i < p.ny; i += blockDim.x) dy[i] = 0.0;
            for (int i = threadIdx.x; i < p.ne; i += blockDim.x) dpi[i] = 0.0;
            for (int i = threadIdx.x; i < p.nc; i += blockDim.x) { dl[i] = 0.0; dtt[i] = 0.0; }
        }
        if (threadIdx.x == 0) fail[q] = fs;
        tsync();
    }
}

// residuals of a batch of points
__global__ void __launch_bounds__(512) k_residuals(KParams p, const double* y0, const double* pi0,
                                                   const double* lam0, const double* t0,
                                                   double* rg, double* rb, double* rd, double* rm,
                                                   double* norms) {
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ int iflag[4];
    double* gslot = p.ws + (long long)blockIdx.x * p.ws_slot;
    for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
        Ctx c;
        make_ctx(c, p, q, gslot, smem, red, iflag);
        setup_constraints(c);
        double* g = rg ? rg + (long long)q * p.ny : c.w[WS_RG];
        double* b = rb ? rb + (long long)q * p.ne : c.w[WS_RB];
        double* d = rd ? rd + (long long)q * p.nc : c.w[WS_RD];
        double* m = rm ? rm + (long long)q * p.nc : nullptr;
        ResNorms r = residuals(c, y0 + (long long)q * p.ny, pi0 + (long long)q * p.ne,
                               lam0 + (long long)q * p.nc, t0 + (long long)q * p.nc, g, b, d, m);
        if (threadIdx.x == 0) {
            double* o = norms + (long long)q * 5;
            o[0] = r.g; o[1] = r.b; o[2] = r.d; o[3] = r.m; o[4] = r.mu;
        }
        tsync();
    }
}

// ---------------------------------------------------------------------------
// _shift_guess (mass_spring.py:152-195): one-stage shift of a solution for the
// next closed-loop MPC solve.  Stage n takes stage n+1's x, u, pi, lam, t
// (where the block sizes agree), the last input repeats, the terminal state is
// rolled once more through the dynamics, and the stage-0 multipliers of the
// initial-state box rows are rebuilt from the stage-0 stationarity gap.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(512) k_shift_guess(KParams p, const double* sy, const double* spi,
                                                     const double* slam, const double* st_,
                                                     double* gy, double* gpi, double* glam,
                                                     double* gt) {
    extern __shared__ double smem[];
    __shared__ double red[32];
    __shared__ int iflag[4];
    double* gslot = p.ws + (long long)blockIdx.x * p.ws_slot;
    const int N = p.N;
    for (int q = blockIdx.x; q < p.B; q += gridDim.x) {
        Ctx c;
        make_ctx(c, p, q, gslot, smem, red, iflag);
        setup_constraints(c);
        const double* y = sy + (long long)q * p.ny;
        const double* pi = spi + (long long)q * p.ne;
        const double* lam = slam + (long long)q * p.nc;
        const double* t = st_ + (long long)q * p.nc;
        double* Y = gy + (long long)q * p.ny;
        double* PI = gpi + (long long)q * p.ne;
        double* LAM = glam + (long long)q * p.nc;
        double* T = gt + (long long)q * p.nc;
        // g = copy of sol, then the stage shift (reads sol only)
        for (int i = threadIdx.x; i < p.ny; i += blockDim.x) Y[i] = y[i];
        for (int i = threadIdx.x; i < p.ne; i += blockDim.x) PI[i] = pi[i];
        for (int i = threadIdx.x; i < p.nc; i += blockDim.x) { LAM[i] = lam[i]; T[i] = t[i]; }
        tsync();
        if (N >= 1) {
            FOR_STAGE_ITEMS(N - 1, p.nc_max + p.nw_max + p.nx_max, n, k)
                const StageInfo& s = c.st[n];
                const StageInfo& s1 = c.st[n + 1];
                if (k < p.nx_max) {                       // x(n) = x(n+1), pi(n) = pi(n+1)
                    if (k < s.nx) Y[s.x_off + k] = y[s1.x_off + k];
                    if (k < s.nxn && k < s1.nxn) PI[s.pi_off + k] = pi[s1.pi_off + k];
                } else if (k < p.nx_max + p.nw_max) {     // u(n) = u(n+1) when the shapes agree
                    const int j = k - p.nx_max;
                    if (s.nu == s1.nu && j < s.nu) Y[s.u_off + j] = y[s1.u_off + j];
                } else {                                  // lam / t blocks when the shapes agree
                    const int j = k - p.nx_max - p.nw_max;
                    if (s.nc == s1.nc && j < s.nc) {
                        LAM[s.c_off + j] = lam[s1.c_off + j];
                        T[s.c_off + j] = t[s1.c_off + j];
                    }
                }
            END_FOR_STAGE_ITEMS
            const StageInfo& sl = c.st[N - 1];
            for (int i = threadIdx.x; i < sl.nx; i += blockDim.x) Y[sl.x_off + i] = y[c.st[N].x_off + i];
            tsync();
            // x(N) = A x(N-1) + B u(N-1) + b of the shifted guess
            for (int i = threadIdx.x; i < sl.nxn; i += blockDim.x) {
                double ax = 0.0, bu = 0.0;
                for (int k = 0; k < sl.nx; ++k) ax = fma(Aget(c, sl, i, k), Y[sl.x_off + k], ax);
                for (int k = 0; k < sl.nu; ++k) bu = fma(Bget(c, sl, i, k), Y[sl.u_off + k], bu);
                Y[c.st[N].x_off + i] = (ax + bu) + fget(c, OCPQP_F_b, sl, i, 0.0);
            }
            tsync();
        }
        // stage-0 initial-state rows: zero their multipliers, take the gap
        const StageInfo& s0 = c.st[0];
        for (int i = threadIdx.x; i < s0.nb; i += blockDim.x)
            if (p.idxb[s0.ib_off + i] >= s0.nu) {
                LAM[s0.c_off + i] = 0.0;
                LAM[s0.c_off + s0.m + i] = 0.0;
            }
        tsync();
        residuals(c, Y, PI, LAM, T, c.w[WS_RG], c.w[WS_RB], c.w[WS_RD], nullptr);
        const double* rg = c.w[WS_RG];
        for (int i = threadIdx.x; i < s0.nb; i += blockDim.x) {
            const int k = p.idxb[s0.ib_off + i];
            if (k >= s0.nu) {
                const double gap = rg[s0.x_off + (k - s0.nu)];
                if (gap >= 0.0) LAM[s0.c_off + i] = gap;
                else LAM[s0.c_off + s0.m + i] = -gap;
                T[s0.c_off + i] = 0.0;
                T[s0.c_off + s0.m + i] = 0.0;
            }
        }
        tsync();
    }
}

// ---------------------------------------------------------------------------
// host-side launchers (called from ocpqp_capi.cu)
// ---------------------------------------------------------------------------
cudaError_t launch_ipm_solve(const KParams& p, const SolveParams& sp, int grid, int threads,
                             size_t smem, cudaStream_t stream) {
    cudaError_t e = cudaFuncSetAttribute(k_ipm_solve, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.counter, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    k_ipm_solve<<<grid, threads, smem, stream>>>(p, sp);
    return cudaGetLastError();
}

cudaError_t launch_newton_step(const KParams& p, double reg, const double* lam, const double* t,
                               const double* rg, const double* rb, const double* rd,
                               const double* rm, double* sy, double* spi, double* slam,
                               double* st, int* fail, int grid, int threads, cudaStream_t stream) {
    k_newton_step<<<grid, threads, 0, stream>>>(p, reg, lam, t, rg, rb, rd, rm, sy, spi, slam, st,
                                                fail);
    return cudaGetLastError();
}

cudaError_t launch_residuals(const KParams& p, const double* y, const double* pi,
                             const double* lam, const double* t, double* rg, double* rb,
                             double* rd, double* rm, double* norms, int grid, int threads,
                             cudaStream_t stream) {
    k_residuals<<<grid, threads, 0, stream>>>(p, y, pi, lam, t, rg, rb, rd, rm, norms);
    return cudaGetLastError();
}

cudaError_t launch_shift_guess(const KParams& p, const double* sy, const double* spi,
                               const double* slam, const double* st, double* gy, double* gpi,
                               double* glam, double* gt, int grid, int threads,
                               cudaStream_t stream) {
    k_shift_guess<<<grid, threads, 0, stream>>>(p, sy, spi, slam, st, gy, gpi, glam, gt);
    return cudaGetLastError();
}

// One block per field A..r: bit f of *mask is set when field f is broadcast
// (batch stride 0) and every stage the shaped kernels read holds the same bits
// as stage 0 (A, B, b, S, R, r: stages 0..N-1; Q, q: 0..N).
struct StageFields {
    const double* f[OCPQP_F_lb];
    long long bs[OCPQP_F_lb];
};

__global__ void k_stage_invariant(StageFields sf, int N, int nx, int nu, int* mask) {
    const int fi = blockIdx.x;
    const double* a = sf.f[fi];
    if (!a || sf.bs[fi] != 0) return;
    const int sz[OCPQP_F_lb] = {nx * nx, nx * nu, nx, nx * nx, nu * nx, nu * nu, nx, nu};
    const int last = (fi == OCPQP_F_Q || fi == OCPQP_F_q) ? N : N - 1;
    const long long L = sz[fi];
    int diff = 0;
    for (long long i = threadIdx.x; i < L * last; i += blockDim.x)
        diff |= __double_as_longlong(a[L + i]) != __double_as_longlong(a[i % L]);
    if (!__syncthreads_or(diff) && threadIdx.x == 0) atomicOr(mask, 1 << fi);
}

__global__ void k_pack_ba(const double* A, long long bsA, const double* B, long long bsB, int N,
                          int nx, int nu, double* out, long long out_bs, long long total, int trans,
                          long long copies, int stage_major) {
    const int nw = nx + nu;
    const long long per_qp = (long long)N * nx * nw;
    for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
         e += (long long)gridDim.x * blockDim.x) {
        const long long q = e / per_qp;
        const long long r = e - q * per_qp;
        const int n = (int)(r / (nx * nw));
        const int rem = (int)(r - (long long)n * nx * nw);
        int k, j;   // element (k, j) of [B A]: row-major (k, j) or transposed (j, k)
        if (trans) { j = rem / nx; k = rem - j * nx; }
        else { k = rem / nw; j = rem - k * nw; }
        // QP-major [copies][N][stage] or stage-major [N][copies][stage]
        const long long o = stage_major ? ((long long)n * copies + q) * nx * nw + rem : q * out_bs + r;
        out[o] = j < nu ? B[q * bsB + ((long long)n * nx + k) * nu + j]
                        : A[q * bsA + ((long long)n * nx + k) * nx + (j - nu)];
    }
}

cudaError_t launch_pack_ba(const double* A, long long bsA, const double* B, long long bsB, int Bn,
                           int N, int nx, int nu, double* out, long long out_bs, cudaStream_t stream,
                           int trans, int stage_major) {
    const long long copies = out_bs == 0 ? 1 : Bn;
    const long long total = copies * N * (long long)nx * (nx + nu);
    if (total == 0) return cudaSuccess;
    const int threads = 256;
    const long long blocks = std::min<long long>((total + threads - 1) / threads, 148ll * 16);
    k_pack_ba<<<(int)blocks, threads, 0, stream>>>(A, bsA, B, bsB, N, nx, nu, out, out_bs, total, trans,
                                                   copies, stage_major);
    return cudaGetLastError();
}

cudaError_t launch_stage_invariant(const double* const* f, const long long* bs, int N, int nx,
                                   int nu, int* mask, cudaStream_t stream) {
    cudaError_t e = cudaMemsetAsync(mask, 0, sizeof(int), stream);
    if (e != cudaSuccess) return e;
    StageFields sf;
    for (int i = 0; i < OCPQP_F_lb; ++i) { sf.f[i] = f[i]; sf.bs[i] = bs[i]; }
    k_stage_invariant<<<OCPQP_F_lb, 256, 0, stream>>>(sf, N, nx, nu, mask);
    return cudaGetLastError();
}

int ipm_occupancy(int threads, size_t smem) {
    int nb = 0;
    cudaFuncSetAttribute(k_ipm_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ipm_solve, threads, smem) != cudaSuccess)
        return 0;
    return nb;
}

}  // namespace ocpqp
