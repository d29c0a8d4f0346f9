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

__device__ __forceinline__ double fget(const Ctx& c, int F, const StageInfo& s, int idx,
                                       double dflt) {
    const double* b = c.f[F];
    return b ? b[s.foff[F] + idx] : dflt;
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
            } else {
                const int g = i - s.nb;
                v = 0.0;
                for (int j = 0; j < s.nw; ++j) v = fma(Jgget(c, s, g, j), w[j], v);
            }
            rowv[s.m_off + i] = v;
        }
    END_FOR_STAGE_ITEMS
}

__device__ __forceinline__ double rows_t(const Ctx& c, const StageInfo& s, int j,
                                         const double* coeff /* stage rows */) {
    const int kb = c.p->var_box[s.u_off + j];
    double out = kb >= 0 ? coeff[kb] : 0.0;
    if (s.ng) {
        double g = 0.0;
        for (int r = 0; r < s.ng; ++r) g = fma(Jgget(c, s, r, j), coeff[s.nb + r], g);
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

__device__ ResNorms residuals(Ctx& c, const double* y, const double* pi, const double* lam,
                              const double* t, double* r_g, double* r_b, double* r_d,
                              double* r_m /* may be null */) {
    const KParams& p = *c.p;
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
            double r = (h1 + h2) + g;
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
                const double rl = (fget(c, OCPQP_F_Zl, s, j, 0.0) * y[yl] + fget(c, OCPQP_F_zl, s, j, 0.0)) - lsl;
                const double ru = (fget(c, OCPQP_F_Zu, s, j, 0.0) * y[yu] + fget(c, OCPQP_F_zu, s, j, 0.0)) - lsu;
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
            const double r = -((xn - ax) - bu) + fget(c, OCPQP_F_b, s, i, 0.0);
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
                rd = (-cy + dvec[kk]) + t[kk];
                rm = lam[kk] * t[kk];
                musum += rm;
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
__device__ bool team_chol(double* L, int n, int ld, int* flag) {
    const int tid = threadIdx.x, T = blockDim.x;
    for (int k = 0; k < n; ++k) {
        if (tid == 0) {
            const double d = L[k * ld + k];
            const int ok = d > 0.0;
            if (ok) L[k * ld + k] = sqrt(d);
            *flag = ok;
        }
        tsync();
        if (!*flag) return false;
        const double dk = L[k * ld + k];
        for (int i = k + 1 + tid; i < n; i += T) L[i * ld + k] /= dk;
        tsync();
        const int rem = n - k - 1;
        for (int idx = tid; idx < rem * rem; idx += T) {
            const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
            if (j <= i) L[i * ld + j] -= L[i * ld + k] * L[j * ld + k];
        }
        tsync();
    }
    for (int idx = tid; idx < n * n; idx += T) {
        const int i = idx / n, j = idx - i * n;
        if (j > i) L[i * ld + j] = 0.0;
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

// ---------------------------------------------------------------------------
// classical Riccati factor (kkt_ocp.py:142-201, 231-251; kkt_common.py:57-115)
// returns -1 on success, the failing stage otherwise; -2 non-positive iterate,
// -3 singular soft-slack block.  flops follow linalg.py counting rules.
// ---------------------------------------------------------------------------
__device__ int factor(Ctx& c, const double* lam, const double* t, double reg, long long& flops) {
    const KParams& p = *c.p;
    const int N = c.N;
    const int tid = threadIdx.x, T = blockDim.x;
    const double* act = c.w[WS_ACT];
    double* gam = c.w[WS_GAM];
    double* coef = c.w[WS_COEF];
    double* Dl = c.w[WS_DL];
    double* Du = c.w[WS_DU];
    double* G = c.w[WS_G];
    double* T1 = c.w[WS_T1];
    double* Pall = c.w[WS_P];
    double* Kall = c.w[WS_K];
    double* Lall = c.w[WS_L];
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
        const int nu = s.nu, nx = s.nx, nw = s.nw, nxn = s.nxn, ng = s.ng;
        const double* cf = coef + s.m_off;
        // stage Hessian M~ (kkt_ocp.py:70-80 + add_reduced_hessian kkt_common.py:100-115)
        for (int idx = tid; idx < nw * nw; idx += T) {
            const int i = idx / nw, j = idx - i * nw;
            double h = 0.5 * (Mraw(c, s, i, j) + Mraw(c, s, j, i));
            if (i == j) {
                const int kb = p.var_box[s.u_off + i];
                if (kb >= 0) h += cf[kb];
            }
            if (ng) {
                double a = 0.0;
                for (int r = 0; r < ng; ++r)
                    a = fma(Jgget(c, s, r, i), cf[s.nb + r] * Jgget(c, s, r, j), a);
                h = a + h;
            }
            if (i == j && reg != 0.0) h += reg;
            G[idx] = h;
        }
        if (ng) flops += 2ll * nw * nw * ng;
        tsync();
        if (n < N) {
            const double* Pn = Pall + c.st[n + 1].P_off;
            // T1 = P[n+1] [B A]  (nx' x nw)
            for (int idx = tid; idx < nxn * nw; idx += T) {
                const int i = idx / nw, j = idx - i * nw;
                double a = 0.0;
                for (int k = 0; k < nxn; ++k) a = fma(Pn[i * nxn + k], BAget(c, s, k, j), a);
                T1[idx] = a;
            }
            tsync();
            // G = [B A]' T1 + M~
            for (int idx = tid; idx < nw * nw; idx += T) {
                const int i = idx / nw, j = idx - i * nw;
                double a = 0.0;
                for (int k = 0; k < nxn; ++k) a = fma(BAget(c, s, k, i), T1[k * nw + j], a);
                G[idx] = a + G[idx];
            }
            flops += 2ll * nxn * nw * nxn + 2ll * nw * nw * nxn;
            tsync();
        }
        double* P = Pall + s.P_off;
        if (nu) {
            double* L = Lall + s.L_off;
            double* K = Kall + s.K_off;
            for (int idx = tid; idx < nu * nu; idx += T) {
                const int i = idx / nu, j = idx - i * nu;
                L[idx] = G[i * nw + j];
            }
            tsync();
            flops += (long long)nu * nu * nu / 3;
            if (!team_chol(L, nu, nu, c.iflag)) return n;
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
    }
    // L_P0 = chol(P[0]) (kkt_ocp.py:193-200)
    const int nx0 = c.st[0].nx;
    if (nx0) {
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
    int nonfinite = 0;
    // fold: w_all = act ? (lam r_d - r_m) / t : 0
    FOR_STAGE_ITEMS(N + 1, p.nc_max, n, k)
        const StageInfo& s = c.st[n];
        if (k < s.nc) {
            const int kk = s.c_off + k;
            double w = 0.0;
            if (act[kk] != 0.0) {
                double rmk;
                if (rm.ext) {
                    rmk = rm.ext[kk];
                } else {
                    rmk = lam[kk] * t[kk] - rm.tau;
                    if (rm.dlam) rmk = rmk + rm.dlam[kk] * rm.dt[kk];
                }
                w = (lam[kk] * r_d[kk] - rmk) / t[kk];
            }
            wall[kk] = w;
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
            const double* Pn = Pall + c.st[n + 1].P_off;
            const double* rb = r_b + s.pi_off;
            const double* pvnext = pv + (c.st[n + 1].pv_off);
            for (int i = tid; i < nxn; i += T) {
                double a = 0.0;
                for (int k = 0; k < nxn; ++k) a = fma(Pn[i * nxn + k], rb[k], a);
                e[i] = a + pvnext[i];
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
        if (nu && tid == T - 1) {
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
        if (tid == 0) {
            const double* LP0 = c.w[WS_LP0];
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
    // dpi_n = P[n+1] x_{n+1} + pv[n+1]
    FOR_STAGE_ITEMS(N, p.nx_max, n, i)
        const StageInfo& s = c.st[n];
        if (i < s.nxn) {
            const StageInfo& s1 = c.st[n + 1];
            const double* Pn = Pall + s1.P_off;
            const double* xn = dy + s1.x_off;
            double a = 0.0;
            for (int k = 0; k < s.nxn; ++k) a = fma(Pn[i * s.nxn + k], xn[k], a);
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
__device__ double max_step(Ctx& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double ftb) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    double ratio = INFINITY;
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x) {
        if (act[k] != 0.0) {
            if (dlam[k] < 0.0) ratio = fmin(ratio, -lam[k] / dlam[k]);
            if (dt[k] < 0.0) ratio = fmin(ratio, -t[k] / dt[k]);
        }
    }
    ratio = team_min(ratio, c.red);
    return fmin(1.0, ftb * ratio);
}

// duality measure at lam + alpha dlam, t + alpha dt
__device__ double trial_mu(Ctx& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double alpha) {
    const KParams& p = *c.p;
    const double* act = c.w[WS_ACT];
    double s = 0.0;
    for (int k = threadIdx.x; k < p.nc; k += blockDim.x)
        if (act[k] != 0.0) s += (lam[k] + alpha * dlam[k]) * (t[k] + alpha * dt[k]);
    s = team_sum(s, c.red);
    return c.n_act > 0.0 ? s / c.n_act : 0.0;
}

// ---------------------------------------------------------------------------
// context construction
// ---------------------------------------------------------------------------
__device__ void make_ctx(Ctx& c, const KParams& p, int q, double* gslot, double* smem,
                         double* red, int* iflag) {
    c.p = &p;
    c.st = p.st;
    c.N = p.N;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f)
        c.f[f] = p.f[f] ? p.f[f] + (long long)q * p.bs[f] : nullptr;
    for (int b = 0; b < WS_NUM; ++b)
        c.w[b] = ((p.smem_mask >> b) & 1u) ? smem + p.smem_off[b] : gslot + p.ws_off[b];
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
// the fused IPM solve of one QP (solver.py:180-308, speed mode)
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

    setup_constraints(c);
    init_iterate(c, arg, y, pi, lam, t);

    long long flops = 0;
    double alpha_last = 1.0;
    int it = 0;
    int status = -1;
    ResNorms res;
    const double reg2 = arg.reg_prim > 0.0 ? 2.0 * arg.reg_prim : 1e-8;
    while (true) {
        res = residuals(c, y, pi, lam, t, r_g, r_b, r_d, nullptr);
        const double mu = res.mu;
        // check_termination (ipm_core.py:286-314)
        if (!isfinite(res.g) || !isfinite(res.b) || !isfinite(res.d) || !isfinite(res.m) ||
            !isfinite(mu)) {
            status = OCPQP_STATUS_NAN;
        } else if (alpha_last < arg.alpha_min) {
            status = OCPQP_STATUS_MINSTEP;
        } else if (mu <= arg.tol_comp && res.g <= arg.tol_stat && res.b <= arg.tol_eq &&
                   res.d <= arg.tol_ineq && res.m <= arg.tol_comp) {
            status = OCPQP_STATUS_SUCCESS;
        } else if (it >= arg.iter_max) {
            status = OCPQP_STATUS_MAXITER;
        }
        if (status >= 0) break;
        // factorization with the speed-mode ladder (solver.py:145-164)
        int fs = factor(c, lam, t, arg.reg_prim, flops);
        if (fs >= 0) fs = factor(c, lam, t, reg2, flops);
        if (fs == -2) { status = OCPQP_STATUS_NONPOSITIVE_ITERATE; break; }
        if (fs == -3) { status = OCPQP_STATUS_SINGULAR_SLACK; break; }
        if (fs >= 0) { status = OCPQP_STATUS_FAILURE; break; }
        // affine prediction
        RmSpec rs{nullptr, 0.0, nullptr, nullptr};
        if (solve(c, lam, t, r_g, r_b, r_d, rs, ay, api, alam, at, flops)) {
            status = OCPQP_STATUS_NAN;
            break;
        }
        const double alpha_aff = max_step(c, lam, t, alam, at, 1.0);
        const double mu_aff = trial_mu(c, lam, t, alam, at, alpha_aff);
        double sigma = 0.0;
        if (mu > 0.0) sigma = fmin(1.0, fmax(0.0, pow(mu_aff / mu, 3.0)));
        const double tau = sigma * mu;
        // combined predictor-corrector direction
        rs.tau = tau;
        if (arg.pred_corr) { rs.dlam = alam; rs.dt = at; }
        int nf = solve(c, lam, t, r_g, r_b, r_d, rs, dy, dpi, dlam, dt, flops);
        if (arg.pred_corr && arg.cond_pred_corr) {
            const double a_t = max_step(c, lam, t, dlam, dt, 1.0);
            const double mu_t = trial_mu(c, lam, t, dlam, dt, a_t);
            if (!(mu_t <= arg.corr_ratio * mu_aff)) {
                RmSpec rc{nullptr, tau, nullptr, nullptr};
                nf = solve(c, lam, t, r_g, r_b, r_d, rc, dy, dpi, dlam, dt, flops);
            }
        }
        if (nf) { status = OCPQP_STATUS_NAN; break; }
        const double alpha = max_step(c, lam, t, dlam, dt, arg.ftb);
        // update_iterate_delta (ipm_core.py:253-272)
        const double* act = c.w[WS_ACT];
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
    // the final residuals (solver.py:300) are those of the last evaluation: every
    // exit path leaves the loop before updating the iterate
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
        if (threadIdx.x == 0) s_q = atomicAdd(p.counter, 1);
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

int ipm_occupancy(int threads, size_t smem) {
    int nb = 0;
    cudaFuncSetAttribute(k_ipm_solve, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_ipm_solve, threads, smem) != cudaSuccess)
        return 0;
    return nb;
}

}  // namespace ocpqp
