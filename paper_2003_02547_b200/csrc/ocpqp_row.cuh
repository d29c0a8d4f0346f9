// Row-owner fused OCP-QP IPM kernel for sm_100a (fp64), NX <= 32.
//
// Same algorithm as ocpqp_ipm.cu -- the speed-mode loop of the reference
// (solver.py:180-308) with the classical Riccati factor/solve of
// kkt_ocp.py:142-320 and kkt_common.py:57-163 -- mapped for small and medium
// stage sizes:
//   * a team of G in {8, 16, 32} lanes owns one QP; lane a owns row a of the
//     cost-to-go P, of G_xx and of T1 = P[B A], column a of G_ux and K, and
//     component a of every per-stage vector, so the Riccati recursion runs on
//     register-resident rows with team shuffles instead of element-indexed
//     loops;
//   * 32/G teams share a warp and walk their QPs in lockstep (a warp claims
//     32/G QPs at once), so an 8-state chain keeps all 32 lanes busy;
//   * teams never use CTA barriers: every synchronisation is a __syncwarp on
//     the team's lane mask, and per-team buffers live in shared memory when
//     they fit, else in the team's global slot (L2-resident).
// Stage shape (NX, NU, NG, NB) is compile-time for stages 0..N-1; the
// terminal stage has nu = 0 and runtime nb, ng.
#pragma once
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ocpqp_internal.h"

namespace ocpqp {
namespace rowk {

constexpr unsigned FULL = 0xffffffffu;

template <int G>
struct Team {
    unsigned mask;
    int lane;
    __device__ __forceinline__ Team() {
        lane = threadIdx.x & (G - 1);
        if constexpr (G == 32) mask = FULL;
        else mask = ((1u << G) - 1u) << ((threadIdx.x & 31) & ~(G - 1));
    }
    __device__ __forceinline__ void sync() const { __syncwarp(mask); }
    __device__ __forceinline__ double shfl(double v, int src) const {
        return __shfl_sync(mask, v, src, G);
    }
    __device__ __forceinline__ double sum(double v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(mask, v, o, G);
        return v;
    }
    __device__ __forceinline__ double max(double v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(mask, v, o, G));
        return v;
    }
    __device__ __forceinline__ double min(double v) const {
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(mask, v, o, G));
        return v;
    }
    __device__ __forceinline__ int any(int v) const { return __any_sync(mask, v); }
};

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

struct AbsMax {
    double m = 0.0;
    int nan = 0;
    __device__ __forceinline__ void add(double x) {
        if (isnan(x)) nan = 1;
        else m = fmax(m, fabs(x));
    }
};

template <int G>
__device__ __forceinline__ double absmax(const Team<G>& T, const AbsMax& a) {
    const int nan = T.any(a.nan);
    const double m = T.max(a.m);
    return nan ? qnan() : m;
}

// Cholesky of an NN x NN matrix whose row i is held by lane i (entries j <= i
// used).  Pivot test of LAPACK potrf (linalg.py:81-118): fails unless > 0.
template <int NN, int G>
__device__ __forceinline__ bool chol_rows(const Team<G>& T, double (&row)[NN]) {
    const int lane = T.lane;
#pragma unroll
    for (int k = 0; k < NN; ++k) {
        const double piv = T.shfl(row[k], k);
        if (!(piv > 0.0)) return false;
        const double dkk = sqrt(piv);
        const double inv = 1.0 / dkk;
        const double lik = lane == k ? dkk : row[k] * inv;
        if (lane >= k) row[k] = lik;
#pragma unroll
        for (int j = k + 1; j < NN; ++j) {
            const double ljk = T.shfl(lik, j);
            if (lane >= j) row[j] = fma(-lik, ljk, row[j]);
        }
    }
    return true;
}

// z <- (L L')^{-1} z with z_i on lane i (i < NN), L row-major in memory.
template <int NN, int G>
__device__ __forceinline__ double cho_solve_lanes(const Team<G>& T, const double* L, double z) {
    const int lane = T.lane;
    const double dii = lane < NN ? L[lane * NN + lane] : 1.0;
#pragma unroll
    for (int k = 0; k < NN; ++k) {
        if (lane == k) z = z / dii;
        const double zk = T.shfl(z, k);
        if (lane > k && lane < NN) z = fma(-L[lane * NN + k], zk, z);
    }
#pragma unroll
    for (int k = NN - 1; k >= 0; --k) {
        if (lane == k) z = z / dii;
        const double zk = T.shfl(z, k);
        if (lane < k) z = fma(-L[k * NN + lane], zk, z);
    }
    return z;
}

struct RCtx {
    const double* f[OCPQP_NUM_FIELDS];
    double* w[WS_EXT0];  // base workspace only (speed mode)
    double* tile;
    double n_act;
};

template <int NX_, int NU_, int NG_, int NB_, int G_, int WPB_>
struct RShape {
    static constexpr int NX = NX_, NU = NU_, NG = NG_, NB = NB_, G = G_, WPB = WPB_;
    static constexpr int NW = NU + NX, M = NB + NG;
    static constexpr int TPW = 32 / G, TEAMS = TPW * WPB, THREADS = 32 * WPB;
    // per-team tile: T1 rows (NX x NW), K (NU x NX), L (NU x NU), rinv (NU)
    static constexpr int TILE = NX * NW + NU * NX + NU * NU + NU + 8;
    static_assert(NX <= G && NU <= G, "row kernel needs NX, NU <= team size");
    static_assert(NB == NW, "row kernel instantiated for full box rows on stages 0..N-1");
};

template <class S>
struct RKern {
    static constexpr int NX = S::NX, NU = S::NU, NG = S::NG, NB = S::NB, NW = S::NW, M = S::M, G = S::G;
    using TeamT = Team<G>;

    struct Dims {
        int N, NBN, NGN, MN, nc, nv, ne, msum;
        __device__ __forceinline__ int slot_stage(int k) const {
            const int n = k / (2 * M);
            return n < N ? n : N;
        }
        __device__ __forceinline__ int row_stage(int r) const {
            const int n = r / M;
            return n < N ? n : N;
        }
        __device__ __forceinline__ int xoff(int n) const { return n * NW + (n < N ? NU : 0); }
    };

    // ---- data access (uniform-stage formula offsets) ----
    __device__ static __forceinline__ const double* A(const RCtx& c, int n) { return c.f[OCPQP_F_A] + n * NX * NX; }
    __device__ static __forceinline__ const double* Bm(const RCtx& c, int n) { return c.f[OCPQP_F_B] + n * NX * NU; }
    __device__ static __forceinline__ const double* bv(const RCtx& c, int n) { return c.f[OCPQP_F_b] + n * NX; }
    __device__ static __forceinline__ const double* Q(const RCtx& c, int n) { return c.f[OCPQP_F_Q] + n * NX * NX; }
    __device__ static __forceinline__ const double* Sm(const RCtx& c, int n) { return c.f[OCPQP_F_S] + n * NU * NX; }
    __device__ static __forceinline__ const double* R(const RCtx& c, int n) { return c.f[OCPQP_F_R] + n * NU * NU; }
    __device__ static __forceinline__ const double* qv(const RCtx& c, int n) { return c.f[OCPQP_F_q] + n * NX; }
    __device__ static __forceinline__ const double* rv(const RCtx& c, int n) { return c.f[OCPQP_F_r] + n * NU; }
    __device__ static __forceinline__ const double* Cm(const RCtx& c, int n) { return c.f[OCPQP_F_C] + n * NG * NX; }
    __device__ static __forceinline__ const double* Dm(const RCtx& c, int n) { return c.f[OCPQP_F_D] + n * NG * NU; }

    // box row of window variable j at the terminal stage (runtime idxb)
    __device__ static __forceinline__ int box_row_N(const KParams& p, const Dims& d, int j) {
        return p.var_box[d.N * NW + j];
    }

    // lam_lo - lam_up (masked) of row i of stage n
    __device__ static __forceinline__ double lam_diff(const double* lam, const double* dv,
                                                      int coff, int m, int i) {
        const double ll = isnan(dv[coff + i]) ? 0.0 : lam[coff + i];
        const double lu = isnan(dv[coff + m + i]) ? 0.0 : lam[coff + m + i];
        return ll - lu;
    }

    // value of row i (box or general) of stage n for the window w
    __device__ static __forceinline__ double row_value(const RCtx& c, const KParams& p, const Dims& d,
                                                       int n, int i, const double* w) {
        if (n < d.N) {
            if (i < NB) return w[i];
            const double* Dr = Dm(c, n) + (i - NB) * NU;
            const double* Cr = Cm(c, n) + (i - NB) * NX;
            double v = 0.0;
#pragma unroll
            for (int j = 0; j < NU; ++j) v = fma(Dr[j], w[j], v);
#pragma unroll 8
            for (int j = 0; j < NX; ++j) v = fma(Cr[j], w[NU + j], v);
            return v;
        }
        if (i < d.NBN) return w[p.idxb[d.N * NB + i]];
        const double* Cr = Cm(c, n) + (i - d.NBN) * NX;
        double v = 0.0;
        for (int j = 0; j < NX; ++j) v = fma(Cr[j], w[j], v);
        return v;
    }

    // ---------------- setup: d (NaN = inactive side) ----------------
    __device__ static void setup(RCtx& c, const TeamT& T, const KParams& p, const Dims& d) {
        double* dv = c.w[WS_DVEC];
        double cnt = 0.0;
        for (int k = T.lane; k < d.nc; k += G) {
            const int n = d.slot_stage(k);
            const int m = n < d.N ? M : d.MN;
            const int nb = n < d.N ? NB : d.NBN;
            const int kk = k - n * 2 * M;
            const int lo = kk < m;
            const int i = lo ? kk : kk - m;
            double bound;
            if (i < nb) bound = c.f[lo ? OCPQP_F_lb : OCPQP_F_ub][n * NB + i];
            else bound = c.f[lo ? OCPQP_F_lg : OCPQP_F_ug][n * NG + (i - nb)];
            const double mk = c.f[lo ? OCPQP_F_maskl : OCPQP_F_masku][n * M + i];
            const bool a = (mk != 0.0) && isfinite(bound);
            dv[k] = a ? (lo ? bound : -bound) : qnan();
            cnt += a ? 1.0 : 0.0;
        }
        c.n_act = T.sum(cnt);
        T.sync();
    }

    struct Res {
        double g, b, d, m, mu;
    };

    // ---------------- residuals (view.py:272-288) ----------------
    __device__ static Res residuals(RCtx& c, const TeamT& T, const KParams& p, const Dims& d,
                                    const double* y, const double* pi, const double* lam,
                                    const double* t) {
        const double* dv = c.w[WS_DVEC];
        double* r_g = c.w[WS_RG];
        double* r_b = c.w[WS_RB];
        double* r_d = c.w[WS_RD];
        const int a = T.lane;
        AbsMax ag, ab, ad, am;
        for (int n = 0; n < d.N; ++n) {
            const double* u = y + n * NW;
            const double* x = u + NU;
            const double* pn = pi + n * NX;
            const int coff = n * 2 * M;
            if (a < NX) {
                // x row (view.py:368-377, 400-409)
                const double* Qr = Q(c, n) + a * NX;
                const double* Sc = Sm(c, n) + a;
                const double* Ac = A(c, n) + a;
                double h1 = 0.0, h2 = 0.0, at = 0.0;
#pragma unroll
                for (int k = 0; k < NU; ++k) h1 = fma(Sc[k * NX], u[k], h1);
#pragma unroll 8
                for (int k = 0; k < NX; ++k) h2 = fma(Qr[k], x[k], h2);
#pragma unroll 8
                for (int k = 0; k < NX; ++k) at = fma(Ac[k * NX], pn[k], at);
                double atp = (n > 0 ? pi[(n - 1) * NX + a] : 0.0) - at;
                double ct = lam_diff(lam, dv, coff, M, NU + a);
                if constexpr (NG > 0) {
                    const double* Cc = Cm(c, n) + a;
                    double gsum = 0.0;
                    for (int r = 0; r < NG; ++r)
                        gsum = fma(Cc[r * NX], lam_diff(lam, dv, coff, M, NB + r), gsum);
                    ct += gsum;
                }
                const double r = (((h1 + h2) + qv(c, n)[a]) - atp) - ct;
                r_g[n * NW + NU + a] = r;
                ag.add(r);
                // r_b (view.py:411-427)
                const double* Ar = A(c, n) + a * NX;
                const double* Br = Bm(c, n) + a * NU;
                double ax = 0.0, bu = 0.0;
#pragma unroll 8
                for (int k = 0; k < NX; ++k) ax = fma(Ar[k], x[k], ax);
#pragma unroll
                for (int k = 0; k < NU; ++k) bu = fma(Br[k], u[k], bu);
                const double xn = y[d.xoff(n + 1) + a];
                const double rb = -((xn - ax) - bu) + bv(c, n)[a];
                r_b[n * NX + a] = rb;
                ab.add(rb);
            }
            if (a < NU) {
                const double* Rr = R(c, n) + a * NU;
                const double* Sr = Sm(c, n) + a * NX;
                const double* Bc = Bm(c, n) + a;
                double h1 = 0.0, h2 = 0.0, at = 0.0;
#pragma unroll
                for (int k = 0; k < NU; ++k) h1 = fma(Rr[k], u[k], h1);
#pragma unroll 8
                for (int k = 0; k < NX; ++k) h2 = fma(Sr[k], x[k], h2);
#pragma unroll 8
                for (int k = 0; k < NX; ++k) at = fma(Bc[k * NU], pn[k], at);
                double ct = lam_diff(lam, dv, coff, M, a);
                if constexpr (NG > 0) {
                    const double* Dc = Dm(c, n) + a;
                    double gsum = 0.0;
                    for (int r = 0; r < NG; ++r)
                        gsum = fma(Dc[r * NU], lam_diff(lam, dv, coff, M, NB + r), gsum);
                    ct += gsum;
                }
                const double r = (((h1 + h2) + rv(c, n)[a]) - (-at)) - ct;
                r_g[n * NW + a] = r;
                ag.add(r);
            }
        }
        {   // terminal stage (nu = 0)
            const int n = d.N;
            const double* x = y + n * NW;
            const int coff = n * 2 * M;
            if (a < NX) {
                const double* Qr = Q(c, n) + a * NX;
                double h2 = 0.0;
#pragma unroll 8
                for (int k = 0; k < NX; ++k) h2 = fma(Qr[k], x[k], h2);
                const double atp = d.N > 0 ? pi[(n - 1) * NX + a] : 0.0;
                const int kb = box_row_N(p, d, a);
                double ct = kb >= 0 ? lam_diff(lam, dv, coff, d.MN, kb) : 0.0;
                if (NG > 0 && d.NGN > 0) {
                    const double* Cc = Cm(c, n) + a;
                    double gsum = 0.0;
                    for (int r = 0; r < d.NGN; ++r)
                        gsum = fma(Cc[r * NX], lam_diff(lam, dv, coff, d.MN, d.NBN + r), gsum);
                    ct += gsum;
                }
                const double r = (((0.0 + h2) + qv(c, n)[a]) - atp) - ct;
                r_g[n * NW + a] = r;
                ag.add(r);
            }
        }
        double musum = 0.0;
        for (int k = T.lane; k < d.nc; k += G) {
            double rd = 0.0, rm = 0.0;
            const double dk = dv[k];
            if (!isnan(dk)) {
                const int n = d.slot_stage(k);
                const int m = n < d.N ? M : d.MN;
                const int kk = k - n * 2 * M;
                const double rvv = row_value(c, p, d, n, kk < m ? kk : kk - m, y + n * NW);
                const double cy = kk < m ? rvv : -rvv;
                rd = (-cy + dk) + t[k];
                rm = lam[k] * t[k];
                musum += rm;
            }
            r_d[k] = rd;
            ad.add(rd);
            am.add(rm);
        }
        Res o;
        o.g = absmax(T, ag);
        o.b = absmax(T, ab);
        o.d = absmax(T, ad);
        o.m = absmax(T, am);
        const double tot = T.sum(musum);
        o.mu = c.n_act > 0.0 ? tot / c.n_act : 0.0;
        T.sync();
        return o;
    }

    // ---------------- classical Riccati factor ----------------
    // -1 ok; failing stage; -2 non-positive iterate.  flops per linalg.py rules.
    __device__ static int factor(RCtx& c, const TeamT& T, const KParams& p, const Dims& d,
                                 const double* lam, const double* t, double reg, long long& flops) {
        const int a = T.lane;
        const double* dv = c.w[WS_DVEC];
        double* gam = c.w[WS_GAM];
        double* coef = c.w[WS_COEF];
        double* Pst = c.w[WS_P];
        double* Kst = c.w[WS_K];
        double* Lst = c.w[WS_L];
        double* T1 = c.tile;                    // NX x NW (also Pt: NX x NX)
        double* Ks = T1 + NX * NW;              // NU x NX
        double* Ls = Ks + NU * NX;              // NU x NU
        double* rinv = Ls + NU * NU;            // NU
        int bad = 0;
        for (int k = a; k < d.nc; k += G) {
            double g = 0.0;
            if (!isnan(dv[k])) {
                if (lam[k] <= 0.0 || t[k] <= 0.0) bad = 1;
                g = lam[k] / t[k];
            }
            gam[k] = g;
        }
        if (T.any(bad)) return -2;
        T.sync();
        for (int r = a; r < d.msum; r += G) {
            const int n = d.row_stage(r);
            const int m = n < d.N ? M : d.MN;
            const int i = r - n * M;
            const int k = n * 2 * M + i;
            coef[r] = gam[k] + gam[k + m];
        }
        T.sync();
        const int N = d.N;
        double prow[NX];
        // terminal stage: P_N = sym(M~_N)
        {
            const int n = N;
            const double* Qn = Q(c, n);
            const double* cf = coef + n * M;
            if (a < NX) {
                const int kb = box_row_N(p, d, a);
#pragma unroll
                for (int b = 0; b < NX; ++b) {
                    double h = 0.5 * (Qn[a * NX + b] + Qn[b * NX + a]);
                    if (b == a && kb >= 0) h += cf[kb];
                    if (NG > 0 && d.NGN > 0) {
                        const double* Cn = Cm(c, n);
                        double s = 0.0;
                        for (int r = 0; r < d.NGN; ++r)
                            s = fma(Cn[r * NX + a], cf[d.NBN + r] * Cn[r * NX + b], s);
                        h = s + h;
                    }
                    if (b == a && reg != 0.0) h += reg;
                    T1[a * NX + b] = h;
                }
            }
            if (NG > 0 && d.NGN > 0) flops += 2ll * NX * NX * d.NGN;
            T.sync();
            if (a < NX) {
                double* Pn = Pst + n * NX * NX + a * NX;
#pragma unroll
                for (int b = 0; b < NX; ++b) {
                    const double v = 0.5 * (T1[a * NX + b] + T1[b * NX + a]);
                    prow[b] = v;
                    Pn[b] = v;
                }
            }
            T.sync();
        }
        for (int n = N - 1; n >= 0; --n) {
            const double* An = A(c, n);
            const double* Bn = Bm(c, n);
            // T1 row a = P_{n+1}[a,:] [B A]  (kkt_ocp.py:232)
            if (a < NX) {
#pragma unroll
                for (int j = 0; j < NU; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NX; ++k) s = fma(prow[k], Bn[k * NU + j], s);
                    T1[a * NW + j] = s;
                }
#pragma unroll 4
                for (int j = 0; j < NX; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NX; ++k) s = fma(prow[k], An[k * NX + j], s);
                    T1[a * NW + NU + j] = s;
                }
            }
            flops += 2ll * NX * NW * NX + 2ll * NW * NW * NX;
            if (NG > 0) flops += 2ll * NW * NW * NG;
            T.sync();
            // G = [B A]' T1 + M~  (kkt_ocp.py:233, 70-80; kkt_common.py:100-115)
            const double* Qn = Q(c, n);
            const double* Rn = R(c, n);
            const double* Sn = Sm(c, n);
            const double* cf = coef + n * M;
            double gxx[NX], gux[NU], guu[NU];
            if (a < NX) {
                const double* Ac = An + a;
#pragma unroll
                for (int b = 0; b < NX; ++b) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NX; ++k) s = fma(Ac[k * NX], T1[k * NW + NU + b], s);
                    double h = 0.5 * (Qn[a * NX + b] + Qn[b * NX + a]);
                    if (b == a) h += cf[NU + a];
                    if constexpr (NG > 0) {
                        const double* Cn = Cm(c, n);
                        double g = 0.0;
                        for (int r = 0; r < NG; ++r)
                            g = fma(Cn[r * NX + a], cf[NB + r] * Cn[r * NX + b], g);
                        h = g + h;
                    }
                    if (b == a && reg != 0.0) h += reg;
                    gxx[b] = s + h;
                }
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NX; ++k) s = fma(Bn[k * NU + i], T1[k * NW + NU + a], s);
                    double h = Sn[i * NX + a];
                    if constexpr (NG > 0) {
                        const double* Cn = Cm(c, n);
                        const double* Dn = Dm(c, n);
                        double g = 0.0;
                        for (int r = 0; r < NG; ++r)
                            g = fma(Dn[r * NU + i], cf[NB + r] * Cn[r * NX + a], g);
                        h = g + h;
                    }
                    gux[i] = s + h;
                }
            }
            if (a < NU) {
#pragma unroll
                for (int j = 0; j < NU; ++j) {
                    double s = 0.0;
#pragma unroll
                    for (int k = 0; k < NX; ++k) s = fma(Bn[k * NU + a], T1[k * NW + j], s);
                    double h = 0.5 * (Rn[a * NU + j] + Rn[j * NU + a]);
                    if (j == a) h += cf[a];
                    if constexpr (NG > 0) {
                        const double* Dn = Dm(c, n);
                        double g = 0.0;
                        for (int r = 0; r < NG; ++r)
                            g = fma(Dn[r * NU + a], cf[NB + r] * Dn[r * NU + j], g);
                        h = g + h;
                    }
                    if (j == a && reg != 0.0) h += reg;
                    guu[j] = s + h;
                }
            } else {
#pragma unroll
                for (int j = 0; j < NU; ++j) guu[j] = 0.0;
            }
            // chol(G_uu), lanes own rows
            flops += (long long)NU * NU * NU / 3;
            if (!chol_rows<NU, G>(T, guu)) return n;
            double* Ln = Lst + n * NU * NU;
            if (a < NU) {
#pragma unroll
                for (int j = 0; j < NU; ++j) {
                    const double v = j <= a ? guu[j] : 0.0;
                    Ls[a * NU + j] = v;
                    Ln[a * NU + j] = v;
                }
                rinv[a] = 1.0 / guu[a];
            }
            T.sync();
            // K column a = -L'^{-1} L^{-1} G_ux[:, a]  (kkt_ocp.py:240-243)
            double* Kn = Kst + n * NU * NX;
            if (a < NX) {
                double z[NU];
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    double s = gux[i];
#pragma unroll
                    for (int k = 0; k < i; ++k) s = fma(-Ls[i * NU + k], z[k], s);
                    z[i] = s * rinv[i];
                }
#pragma unroll
                for (int i = NU - 1; i >= 0; --i) {
                    double s = z[i];
#pragma unroll
                    for (int k = i + 1; k < NU; ++k) s = fma(-Ls[k * NU + i], z[k], s);
                    z[i] = s * rinv[i];
                }
#pragma unroll
                for (int i = 0; i < NU; ++i) {
                    Ks[i * NX + a] = -z[i];
                    Kn[i * NX + a] = -z[i];
                }
            }
            flops += 2ll * NU * NU * NX + 2ll * NX * NX * NU;
            T.sync();
            // P = G_xx + G_ux' K, symmetrised (kkt_ocp.py:244, 251)
            if (a < NX) {
#pragma unroll
                for (int b = 0; b < NX; ++b) {
                    double s = 0.0;
#pragma unroll
                    for (int i = 0; i < NU; ++i) s = fma(gux[i], Ks[i * NX + b], s);
                    T1[a * NX + b] = s + gxx[b];
                }
            }
            T.sync();
            if (a < NX) {
                double* Pn = Pst + n * NX * NX + a * NX;
#pragma unroll
                for (int b = 0; b < NX; ++b) {
                    const double v = 0.5 * (T1[a * NX + b] + T1[b * NX + a]);
                    prow[b] = v;
                    Pn[b] = v;
                }
            }
            T.sync();
        }
        // L_P0 = chol(P_0) (kkt_ocp.py:193-200)
        flops += (long long)NX * NX * NX / 3;
        if (a >= NX) {
#pragma unroll
            for (int b = 0; b < NX; ++b) prow[b] = 0.0;
        }
        if (!chol_rows<NX, G>(T, prow)) return 0;
        if (a < NX) {
            double* LP0 = c.w[WS_LP0] + a * NX;
#pragma unroll
            for (int b = 0; b < NX; ++b) LP0[b] = b <= a ? prow[b] : 0.0;
        }
        T.sync();
        return -1;
    }

    // Jc' crow at window variable j of stage n (rows_w_t, view.py:99-105)
    __device__ static __forceinline__ double ct_rows(const RCtx& c, const KParams& p, const Dims& d,
                                                     int n, int j, const double* crow) {
        const double* cr = crow + n * M;
        if (n < d.N) {
            double out = cr[j];
            if constexpr (NG > 0) {
                double g = 0.0;
                if (j < NU) {
                    const double* Dc = Dm(c, n) + j;
                    for (int r = 0; r < NG; ++r) g = fma(Dc[r * NU], cr[NB + r], g);
                } else {
                    const double* Cc = Cm(c, n) + (j - NU);
                    for (int r = 0; r < NG; ++r) g = fma(Cc[r * NX], cr[NB + r], g);
                }
                out += g;
            }
            return out;
        }
        const int kb = box_row_N(p, d, j);
        double out = kb >= 0 ? cr[kb] : 0.0;
        if (NG > 0 && d.NGN > 0) {
            const double* Cc = Cm(c, n) + j;
            double g = 0.0;
            for (int r = 0; r < d.NGN; ++r) g = fma(Cc[r * NX], cr[d.NBN + r], g);
            out += g;
        }
        return out;
    }

    // recover_block (kkt_common.py:140-163) for the slots of stage n
    __device__ static __forceinline__ int recover_stage(const RCtx& c, const TeamT& T, const KParams& p,
                                                        const Dims& d, int n, const double* dy,
                                                        double* dlam, double* dt) {
        const double* dv = c.w[WS_DVEC];
        const double* gam = c.w[WS_GAM];
        const double* wall = c.w[WS_WALL];
        const double* r_d = c.w[WS_RD];
        const int m = n < d.N ? M : d.MN;
        const int coff = n * 2 * M;
        int nf = 0;
        for (int kk = T.lane; kk < 2 * m; kk += G) {
            const int k = coff + kk;
            double dl = 0.0, dtt = 0.0;
            if (!isnan(dv[k])) {
                const double rvv = row_value(c, p, d, n, kk < m ? kk : kk - m, dy + n * NW);
                const double cy = kk < m ? rvv : -rvv;
                dl = wall[k] - gam[k] * cy;
                dtt = -r_d[k] + cy;
            }
            dlam[k] = dl;
            dt[k] = dtt;
            nf |= !isfinite(dl) || !isfinite(dtt);
        }
        return nf;
    }

    // ---------------- Riccati solve (kkt_ocp.py:254-320) ----------------
    __device__ static int solve(RCtx& c, const TeamT& T, const KParams& p, const Dims& d,
                                const double* lam, const double* t, const double* rm_ext, double tau,
                                const double* dla, const double* dta, double* dy, double* dpi,
                                double* dlam, double* dt, long long& flops) {
        const int a = T.lane;
        const double* dv = c.w[WS_DVEC];
        const double* r_g = c.w[WS_RG];
        const double* r_b = c.w[WS_RB];
        const double* r_d = c.w[WS_RD];
        double* wall = c.w[WS_WALL];
        double* crow = c.w[WS_CROW];
        const double* Pst = c.w[WS_P];
        const double* Kst = c.w[WS_K];
        const double* Lst = c.w[WS_L];
        double* pvst = c.w[WS_PV];
        double* kffst = c.w[WS_KFF];
        int nf = 0;
        // fold_rhs (kkt_common.py:118-137)
        for (int k = a; k < d.nc; k += G) {
            double w = 0.0;
            if (!isnan(dv[k])) {
                double rmk;
                if (rm_ext) {
                    rmk = rm_ext[k];
                } else {
                    rmk = lam[k] * t[k] - tau;
                    if (dla) rmk = rmk + dla[k] * dta[k];
                }
                w = (lam[k] * r_d[k] - rmk) / t[k];
            }
            wall[k] = w;
        }
        T.sync();
        for (int r = a; r < d.msum; r += G) {
            const int n = d.row_stage(r);
            const int m = n < d.N ? M : d.MN;
            const int k = n * 2 * M + (r - n * M);
            crow[r] = wall[k] - wall[k + m];
        }
        T.sync();
        const int N = d.N;
        // backward sweep (kkt_ocp.py:276-289)
        double pvr = 0.0;
        if (a < NX) {
            pvr = r_g[N * NW + a] - ct_rows(c, p, d, N, a, crow);
            pvst[N * NX + a] = pvr;
        }
        for (int n = N - 1; n >= 0; --n) {
            const double* Pn = Pst + (n + 1) * NX * NX;
            const double* rb = r_b + n * NX;
            double e = 0.0;
            if (a < NX) {
                const double* Pr = Pn + a * NX;
#pragma unroll 8
                for (int k = 0; k < NX; ++k) e = fma(Pr[k], rb[k], e);
                e = e + pvr;
            }
            const double* An = A(c, n);
            const double* Bn = Bm(c, n);
            double sq = 0.0, su = 0.0;
#pragma unroll 8
            for (int k = 0; k < NX; ++k) {
                const double ek = T.shfl(e, k);
                if (a < NX) sq = fma(An[k * NX + a], ek, sq);
                if (a < NU) su = fma(Bn[k * NU + a], ek, su);
            }
            double rq = 0.0, rr = 0.0;
            if (a < NX) rq = (r_g[n * NW + NU + a] - ct_rows(c, p, d, n, NU + a, crow)) + sq;
            if (a < NU) rr = (r_g[n * NW + a] - ct_rows(c, p, d, n, a, crow)) + su;
            // kff = -(L L')^{-1} rr
            const double kf = -cho_solve_lanes<NU, G>(T, Lst + n * NU * NU, rr);
            if (a < NU) kffst[n * NU + a] = kf;
            // pv = rq + K' rr
            const double* Kn = Kst + n * NU * NX;
            double s = 0.0;
#pragma unroll
            for (int i = 0; i < NU; ++i) {
                const double ri = T.shfl(rr, i);
                if (a < NX) s = fma(Kn[i * NX + a], ri, s);
            }
            pvr = rq + s;
            if (a < NX) pvst[n * NX + a] = pvr;
        }
        flops += 2ll * NU * NU * N + 2ll * NX * NX;
        // x0 step (kkt_ocp.py:292)
        double xi = -cho_solve_lanes<NX, G>(T, c.w[WS_LP0], pvr);
        T.sync();
        // forward rollout (kkt_ocp.py:293-305) with per-stage recovery
        for (int n = 0; n < N; ++n) {
            if (a < NX) dy[n * NW + NU + a] = xi;
            const double* Kn = Kst + n * NU * NX;
            double du = 0.0;
#pragma unroll 8
            for (int k = 0; k < NX; ++k) {
                const double xk = T.shfl(xi, k);
                if (a < NU) du = fma(Kn[a * NX + k], xk, du);
            }
            if (a < NU) {
                du = du + kffst[n * NU + a];
                dy[n * NW + a] = du;
            }
            nf |= !isfinite(du) || !isfinite(xi);
            const double* An = A(c, n);
            const double* Bn = Bm(c, n);
            double ax = 0.0, bu = 0.0;
#pragma unroll 8
            for (int k = 0; k < NX; ++k) {
                const double xk = T.shfl(xi, k);
                if (a < NX) ax = fma(An[a * NX + k], xk, ax);
            }
#pragma unroll
            for (int i = 0; i < NU; ++i) {
                const double ui = T.shfl(du, i);
                if (a < NX) bu = fma(Bn[a * NU + i], ui, bu);
            }
            const double xn = (ax + bu) + (a < NX ? r_b[n * NX + a] : 0.0);
            // dpi_n = P_{n+1} x_{n+1} + pv_{n+1}
            const double* Pr = Pst + (n + 1) * NX * NX + a * NX;
            double s = 0.0;
#pragma unroll 8
            for (int k = 0; k < NX; ++k) {
                const double xk = T.shfl(xn, k);
                if (a < NX) s = fma(Pr[k], xk, s);
            }
            if (a < NX) {
                const double v = s + pvst[(n + 1) * NX + a];
                dpi[n * NX + a] = v;
                nf |= !isfinite(v);
            }
            T.sync();
            nf |= recover_stage(c, T, p, d, n, dy, dlam, dt);
            xi = xn;
        }
        if (a < NX) dy[N * NW + a] = xi;
        nf |= !isfinite(xi);
        T.sync();
        nf |= recover_stage(c, T, p, d, N, dy, dlam, dt);
        return T.any(nf);
    }

    __device__ static double max_step(const RCtx& c, const TeamT& T, const Dims& d, const double* lam,
                                      const double* t, const double* dlam, const double* dt, double ftb) {
        const double* dv = c.w[WS_DVEC];
        double ratio = INFINITY;
        for (int k = T.lane; k < d.nc; k += G) {
            if (!isnan(dv[k])) {
                if (dlam[k] < 0.0) ratio = fmin(ratio, -lam[k] / dlam[k]);
                if (dt[k] < 0.0) ratio = fmin(ratio, -t[k] / dt[k]);
            }
        }
        ratio = T.min(ratio);
        return fmin(1.0, ftb * ratio);
    }

    __device__ static double trial_mu(const RCtx& c, const TeamT& T, const Dims& d, const double* lam,
                                      const double* t, const double* dlam, const double* dt, double alpha) {
        const double* dv = c.w[WS_DVEC];
        double s = 0.0;
        for (int k = T.lane; k < d.nc; k += G)
            if (!isnan(dv[k])) s += (lam[k] + alpha * dlam[k]) * (t[k] + alpha * dt[k]);
        s = T.sum(s);
        return c.n_act > 0.0 ? s / c.n_act : 0.0;
    }

    // ---------------- the IPM loop of one QP (solver.py:180-308) ----------------
    __device__ static void ipm_one(RCtx& c, const TeamT& T, const KParams& p, const Dims& d,
                                   const SolveParams& sp, int q) {
        const OcpIpmArgC& arg = sp.arg;
        const int a = T.lane;
        double* gy = sp.y + (long long)q * d.nv;
        double* gpi = sp.pi + (long long)q * d.ne;
        double* glam = sp.lam + (long long)q * d.nc;
        double* gt = sp.t + (long long)q * d.nc;
        double* y = c.w[WS_IY];
        double* pi = c.w[WS_IPI];
        double* lam = c.w[WS_ILAM];
        double* t = c.w[WS_IT];
        double* alam = c.w[WS_AFF_LAM];
        double* at = c.w[WS_AFF_T];
        double *dy = c.w[WS_DIR_Y], *dpi = c.w[WS_DIR_PI], *dlam = c.w[WS_DIR_LAM], *dt = c.w[WS_DIR_T];
        const double* dv = c.w[WS_DVEC];
        setup(c, T, p, d);
        const int warm = arg.warm_start;
        for (int i = a; i < d.nv; i += G) y[i] = warm ? gy[i] : 0.0;
        for (int i = a; i < d.ne; i += G) pi[i] = warm == 2 ? gpi[i] : 0.0;
        T.sync();
        // initial iterate (solver.py:113-142)
        double floor = arg.t0;
        if (warm == 2) {
            double gd = 0.0, gb = 0.0;
            for (int k = a; k < d.nc; k += G) {
                if (!isnan(dv[k])) {
                    const int n = d.slot_stage(k);
                    const int m = n < d.N ? M : d.MN;
                    const int kk = k - n * 2 * M;
                    const double rvv = row_value(c, p, d, n, kk < m ? kk : kk - m, y + n * NW);
                    gd = fmax(gd, dv[k] - (kk < m ? rvv : -rvv));
                }
            }
            for (int e = a; e < d.ne; e += G) {
                const int n = e / NX, i = e - n * NX;
                const double* u = y + n * NW;
                const double* Ar = A(c, n) + i * NX;
                const double* Br = Bm(c, n) + i * NU;
                double ax = 0.0, bu = 0.0;
                for (int k = 0; k < NX; ++k) ax = fma(Ar[k], u[NU + k], ax);
                for (int k = 0; k < NU; ++k) bu = fma(Br[k], u[k], bu);
                gb = fmax(gb, fabs(-((y[d.xoff(n + 1) + i] - ax) - bu) + bv(c, n)[i]));
            }
            gd = T.max(gd);
            gb = T.max(gb);
            floor = fmax(fmax(1e-8, arg.t_min), fmin(1.0, fmax(gd, gb)));
        }
        const double lfloor = fmax(1e-8, arg.lam_min);
        for (int k = a; k < d.nc; k += G) {
            double tv = 0.0, lv = 0.0;
            if (!isnan(dv[k])) {
                double cy = 0.0;
                if (warm) {
                    const int n = d.slot_stage(k);
                    const int m = n < d.N ? M : d.MN;
                    const int kk = k - n * 2 * M;
                    const double rvv = row_value(c, p, d, n, kk < m ? kk : kk - m, y + n * NW);
                    cy = kk < m ? rvv : -rvv;
                }
                tv = fmax(cy - dv[k], floor);
                lv = warm == 2 ? fmax(glam[k], lfloor) : arg.mu0 / tv;
            }
            t[k] = tv;
            lam[k] = lv;
        }
        T.sync();
        double* trace = sp.trace ? sp.trace + (long long)q * arg.iter_max * 8 : nullptr;
        long long flops = 0;
        double alpha_last = 1.0;
        int it = 0, status = -1;
        Res res;
        const double reg2 = arg.reg_prim > 0.0 ? 2.0 * arg.reg_prim : 1e-8;
        long long ph[DBG_KEPT] = {0, 0, 0, 0, 0, 0, 0, 0};
        const long long t_start = clock64();
        long long tc = t_start;
        while (true) {
            res = residuals(c, T, p, d, y, pi, lam, t);
            const double mu = res.mu;
            if (!isfinite(res.g) || !isfinite(res.b) || !isfinite(res.d) || !isfinite(res.m) || !isfinite(mu))
                status = OCPQP_STATUS_NAN;
            else if (alpha_last < arg.alpha_min)
                status = OCPQP_STATUS_MINSTEP;
            else if (mu <= arg.tol_comp && res.g <= arg.tol_stat && res.b <= arg.tol_eq &&
                     res.d <= arg.tol_ineq && res.m <= arg.tol_comp)
                status = OCPQP_STATUS_SUCCESS;
            else if (it >= arg.iter_max)
                status = OCPQP_STATUS_MAXITER;
            if (p.dbg) { const long long n_ = clock64(); ph[DBG_RES] += n_ - tc; tc = n_; }
            if (status >= 0) break;
            int fs = factor(c, T, p, d, lam, t, arg.reg_prim, flops);
            if (fs >= 0) { T.sync(); fs = factor(c, T, p, d, lam, t, reg2, flops); }
            if (fs == -2) { status = OCPQP_STATUS_NONPOSITIVE_ITERATE; break; }
            if (fs >= 0) { status = OCPQP_STATUS_FAILURE; break; }
            if (p.dbg) { const long long n_ = clock64(); ph[DBG_FACTOR] += n_ - tc; tc = n_; }
            if (solve(c, T, p, d, lam, t, nullptr, 0.0, nullptr, nullptr, dy, dpi, alam, at, flops)) {
                status = OCPQP_STATUS_NAN;
                break;
            }
            T.sync();
            if (p.dbg) { const long long n_ = clock64(); ph[DBG_SOLVE_AFF] += n_ - tc; tc = n_; }
            const double alpha_aff = max_step(c, T, d, lam, t, alam, at, 1.0);
            const double mu_aff = trial_mu(c, T, d, lam, t, alam, at, alpha_aff);
            double sigma = 0.0;
            if (mu > 0.0) sigma = fmin(1.0, fmax(0.0, pow(mu_aff / mu, 3.0)));
            const double tau = sigma * mu;
            int nf = solve(c, T, p, d, lam, t, nullptr, tau, arg.pred_corr ? alam : nullptr,
                           arg.pred_corr ? at : nullptr, dy, dpi, dlam, dt, flops);
            T.sync();
            if (arg.pred_corr && arg.cond_pred_corr) {
                const double a_t = max_step(c, T, d, lam, t, dlam, dt, 1.0);
                const double mu_t = trial_mu(c, T, d, lam, t, dlam, dt, a_t);
                if (!(mu_t <= arg.corr_ratio * mu_aff)) {
                    nf = solve(c, T, p, d, lam, t, nullptr, tau, nullptr, nullptr, dy, dpi, dlam, dt, flops);
                    T.sync();
                }
            }
            if (p.dbg) { const long long n_ = clock64(); ph[DBG_SOLVE_DIR] += n_ - tc; tc = n_; }
            if (nf) { status = OCPQP_STATUS_NAN; break; }
            const double alpha = max_step(c, T, d, lam, t, dlam, dt, arg.ftb);
            for (int i = a; i < d.nv; i += G) y[i] += alpha * dy[i];
            for (int i = a; i < d.ne; i += G) pi[i] += alpha * dpi[i];
            for (int k = a; k < d.nc; k += G) {
                double lv = lam[k] + alpha * dlam[k];
                double tv = t[k] + alpha * dt[k];
                if (!isnan(dv[k])) {
                    lv = fmax(lv, arg.lam_min);
                    tv = fmax(tv, arg.t_min);
                }
                lam[k] = lv;
                t[k] = tv;
            }
            if (trace && a == 0 && it < arg.iter_max) {
                double* tr = trace + (long long)it * 8;
                tr[0] = alpha_aff; tr[1] = alpha; tr[2] = mu; tr[3] = sigma;
                tr[4] = res.g; tr[5] = res.b; tr[6] = res.d; tr[7] = res.m;
            }
            T.sync();
            alpha_last = alpha;
            ++it;
            if (p.dbg) { const long long n_ = clock64(); ph[DBG_STEP] += n_ - tc; tc = n_; }
        }
        T.sync();
        for (int i = a; i < d.nv; i += G) gy[i] = y[i];
        for (int i = a; i < d.ne; i += G) gpi[i] = pi[i];
        for (int k = a; k < d.nc; k += G) { glam[k] = lam[k]; gt[k] = t[k]; }
        if (a == 0) {
            sp.status[q] = status;
            sp.iters[q] = it;
            double* r = sp.res + (long long)q * 5;
            r[0] = res.g; r[1] = res.b; r[2] = res.d; r[3] = res.m; r[4] = res.mu;
            sp.flops[q] = flops;
            if (p.dbg) {
                ph[DBG_TOTAL] = clock64() - t_start;
                ph[DBG_ITERS] = it;
                for (int i = 0; i < DBG_KEPT; ++i) p.dbg[(long long)q * DBG_NUM + i] = ph[i];
            }
        }
    }
};

// KParams.stage_smem = per-team tile offset within the team's smem region,
// KParams.team_stride = doubles of smem per team.
template <class S>
__global__ void __launch_bounds__(S::THREADS) k_row_solve(KParams p, SolveParams sp) {
    extern __shared__ double smem[];
    __shared__ RCtx ctx[S::TEAMS];
    const int warp = threadIdx.x >> 5;
    const int tiw = (threadIdx.x & 31) / S::G;          // team in warp
    const int team = warp * S::TPW + tiw;
    Team<S::G> T;
    RCtx& c = ctx[team];
    double* tsm = smem + (long long)team * p.team_stride;
    double* gslot = p.ws + ((long long)blockIdx.x * S::TEAMS + team) * p.ws_slot;
    for (int b = T.lane; b < WS_EXT0; b += S::G)
        c.w[b] = ((p.smem_mask >> b) & 1ull) ? tsm + p.smem_off[b] : gslot + p.ws_off[b];
    if (T.lane == 0) c.tile = tsm + p.stage_smem;
    typename RKern<S>::Dims d;
    d.N = p.N; d.NBN = p.NBN; d.NGN = p.NGN; d.MN = p.NBN + p.NGN;
    d.nc = p.nc; d.nv = p.nv; d.ne = p.ne; d.msum = p.msum;
    __syncwarp();
    while (true) {
        int base = 0;
        if ((threadIdx.x & 31) == 0) base = atomicAdd(p.counter, S::TPW);
        base = __shfl_sync(FULL, base, 0);
        if (base >= p.B) break;
        const int q = base + tiw;
        if (q < p.B) {
            for (int f = T.lane; f < OCPQP_NUM_FIELDS; f += S::G)
                c.f[f] = p.f[f] + (long long)q * p.bs[f];
            T.sync();
            RKern<S>::ipm_one(c, T, p, d, sp, q);
        }
        __syncwarp();
    }
}

template <class S>
int row_team_tile() { return S::TILE; }

template <class S>
cudaError_t row_launch(const KParams& p, const SolveParams& sp, int grid, size_t smem, cudaStream_t st) {
    cudaError_t e = cudaFuncSetAttribute(k_row_solve<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    e = cudaMemsetAsync(p.counter, 0, sizeof(int), st);
    if (e != cudaSuccess) return e;
    k_row_solve<S><<<grid, S::THREADS, smem, st>>>(p, sp);
    return cudaGetLastError();
}

template <class S>
int row_occupancy(size_t smem) {
    int nb = 0;
    cudaFuncSetAttribute(k_row_solve<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k_row_solve<S>, S::THREADS, smem) != cudaSuccess)
        return 0;
    return nb;
}

}  // namespace rowk
}  // namespace ocpqp
