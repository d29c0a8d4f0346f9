// Dense QPs with equality constraints on the GPU (fp64, sm_100a).
//
// The reference's dense backend (kkt_dense.py:117-256) behind its IPM loop
// (solver.py:180-308, speed-mode sequence of SURVEY Appendix A) for
//   min 1/2 v'Hv + g'v  s.t.  A v = b,  box rows lb <= v[idxb] <= ub,
//                              general rows lg <= C v <= ug       (qp_data.py:426-500)
// with the two equality-handling methods of DenseKktFactor:
//   schur       Hred = H + C' diag(gamma) C (+ box gamma, + reg_prim I),
//               L = chol(Hred), W = L^{-1} A', M = W'W + reg_dual I, Lm = chol(M);
//               solve: z = Hred^{-1} rhat, dpi = M^{-1}(r_b + A z),
//                      dv = Hred^{-1}(A' dpi - rhat)                 (kkt_dense.py:166-185, 226-231)
//   null_space  [Q1 Z] R = qr(A') (Householder), Hz = Z' Hred Z, Lz = chol(Hz);
//               solve: v_p = Q1 Ra^{-T} r_b, q = -Hz^{-1} Z'(rhat + Hred v_p),
//                      dv = v_p + Z q, dpi = Ra^{-1} Q1'(Hred dv + rhat) (kkt_dense.py:153-165, 217-225)
// One CTA per QP (persistent over the batch), workspace per resident CTA in
// global memory (L1/L2-resident at the sizes this path serves).  Counted flops
// follow the reference's flop_counter rules (linalg.py:41-78): cholesky n^3//3,
// triangular solves n^2 m, matmul_acc 2mnk; inline products uncounted.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "ocpqp_internal.h"

namespace ocpqp {
namespace densek {

constexpr unsigned FULL = 0xffffffffu;

__device__ __forceinline__ double qnan() { return __longlong_as_double(0x7ff8000000000000ll); }

__device__ double tsum(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    __syncthreads();
    return s;
}
__device__ double tmin(double v, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmin(v, __shfl_xor_sync(FULL, v, o));
    __syncthreads();
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
    __syncthreads();
    double s = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) s = fmin(s, red[i]);
    __syncthreads();
    return s;
}
// max |x| with NaN propagation
__device__ double tabsmax(double m, int nan, double* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(FULL, m, o));
    nan = __syncthreads_or(nan);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
    __syncthreads();
    double s = red[0];
    for (int i = 1; i < (int)(blockDim.x >> 5); ++i) s = fmax(s, red[i]);
    __syncthreads();
    return nan ? qnan() : s;
}

// In-place lower Cholesky of the n x n matrix at L (row stride ld); upper
// triangle zeroed.  Pivot test as LAPACK potrf: a pivot not > 0 fails.
__device__ bool tchol(double* L, int n, int ld, int* flag) {
    const int tid = threadIdx.x, T = blockDim.x;
    for (int k = 0; k < n; ++k) {
        if (tid == 0) {
            const double d = L[k * ld + k];
            *flag = d > 0.0;
            if (d > 0.0) L[k * ld + k] = sqrt(d);
        }
        __syncthreads();
        if (!*flag) return false;
        const double lkk = L[k * ld + k];
        for (int i = k + 1 + tid; i < n; i += T) L[i * ld + k] /= lkk;
        __syncthreads();
        const int rem = n - k - 1;
        for (int idx = tid; idx < rem * rem; idx += T) {
            const int i = k + 1 + idx / rem, j = k + 1 + idx % rem;
            if (j <= i) L[i * ld + j] = fma(-L[i * ld + k], L[j * ld + k], L[i * ld + j]);
        }
        __syncthreads();
    }
    for (int idx = tid; idx < n * n; idx += T) {
        const int i = idx / n, j = idx - i * n;
        if (j > i) L[i * ld + j] = 0.0;
    }
    __syncthreads();
    return true;
}

// x <- L^{-1} x (lower, trans = 0) or L^{-T} x (trans = 1), by warp 0 with
// lane-split dot products (scipy solve_triangular semantics, n x n, stride ld)
__device__ void wtrsv(const double* L, int n, int ld, double* x, bool trans, bool upper = false) {
    if (threadIdx.x >= 32) return;
    const int lane = threadIdx.x;
    // effective lower-triangular access: lower & !trans, or upper & trans
    const bool fwd = (!upper && !trans) || (upper && trans);
    for (int s = 0; s < n; ++s) {
        const int i = fwd ? s : n - 1 - s;
        double acc = 0.0;
        if (fwd) {
            for (int k = lane; k < i; k += 32) {
                const double lik = upper ? L[k * ld + i] : L[i * ld + k];
                acc = fma(lik, x[k], acc);
            }
        } else {
            for (int k = i + 1 + lane; k < n; k += 32) {
                const double lki = upper ? L[i * ld + k] : L[k * ld + i];
                acc = fma(lki, x[k], acc);
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
        if (lane == 0) x[i] = (x[i] - acc) / L[i * ld + i];
        __syncwarp();
    }
}

struct DKParams {
    int B, nv, ne, nb, ng, nc, m;
    int method;                 // 0 schur, 1 null_space
    const int* idxb;            // [nb]
    const double* f[11];        // H g A b lb ub C lg ug maskl masku
    long long bs[11];
    double* ws;
    long long ws_slot;
    int* counter;
    double reg_dual;            // IpmArg.reg_dual (ipm_core.py; Schur complement shift)
};
enum { DH = 0, DG, DA, DBV, DLB, DUB, DC, DLG, DUG, DML, DMU };

// workspace offsets (doubles) within a slot
struct WS {
    long long act, gam, tinv, wall, rd, rg, rb, rhat, v, pi, lam, t, dv, dpi, dlam, dt, alam, at,
        tv1, tv2, te1, te2, rowv, L, W, M, Q, R, Hz, HZ, HRZ, end;
};
__host__ __device__ inline WS ws_layout(int nv, int ne, int nc, int m) {
    WS w;
    long long o = 0;
    auto take = [&](long long n) { const long long r = o; o += (n + 1) & ~1ll; return r; };
    w.act = take(nc); w.gam = take(nc); w.tinv = take(nc); w.wall = take(nc); w.rd = take(nc);
    w.rg = take(nv); w.rb = take(ne); w.rhat = take(nv);
    w.v = take(nv); w.pi = take(ne); w.lam = take(nc); w.t = take(nc);
    w.dv = take(nv); w.dpi = take(ne); w.dlam = take(nc); w.dt = take(nc);
    w.alam = take(nc); w.at = take(nc);
    w.tv1 = take(nv); w.tv2 = take(nv); w.te1 = take(ne); w.te2 = take(ne); w.rowv = take(m);
    w.L = take((long long)nv * nv); w.W = take((long long)nv * ne); w.M = take((long long)ne * ne);
    w.Q = take((long long)nv * nv); w.R = take((long long)ne * ne);
    const long long nz = nv - ne > 0 ? nv - ne : 0;
    w.Hz = take(nz * nz); w.HZ = take((long long)nv * nz); w.HRZ = take((long long)nv * nz);
    w.end = o;
    return w;
}

struct C {
    const DKParams* p;
    const double* f[11];
    double* w;
    WS o;
    int nv, ne, nb, ng, nc, m;
    double n_act;
    double* red;
    int* flag;
    __device__ double* V(long long off) const { return w + off; }
    __device__ double H(int i, int j) const { return f[DH][i * nv + j]; }
    __device__ double A(int i, int j) const { return f[DA][i * nv + j]; }
    __device__ double Cg(int r, int j) const { return f[DC][r * nv + j]; }
};

// row value of constraint row r (box rows first, then general rows)
__device__ double rowval(const C& c, int r, const double* v) {
    if (r < c.nb) return v[c.p->idxb[r]];
    double s = 0.0;
    const int g = r - c.nb;
    for (int j = 0; j < c.nv; ++j) s = fma(c.Cg(g, j), v[j], s);
    return s;
}

// Jc' coeff (coeff per row), variable j
__device__ double rows_t(const C& c, int j, const double* coeff) {
    double s = 0.0;
    for (int r = 0; r < c.nb; ++r)
        if (c.p->idxb[r] == j) s += coeff[r];
    double gsum = 0.0;
    for (int g = 0; g < c.ng; ++g) gsum = fma(c.Cg(g, j), coeff[c.nb + g], gsum);
    return s + gsum;
}

// setup: d (NaN = inactive side) and the active count (view.py:108-129, 156-157)
__device__ void setup(C& c) {
    double* dv = c.V(c.o.act);
    double cnt = 0.0;
    for (int k = threadIdx.x; k < c.nc; k += blockDim.x) {
        const bool lo = k < c.m;
        const int r = lo ? k : k - c.m;
        const double bound = r < c.nb ? c.f[lo ? DLB : DUB][r] : c.f[lo ? DLG : DUG][r - c.nb];
        const double mask = c.f[lo ? DML : DMU][r];
        const bool a = (mask != 0.0) && isfinite(bound);
        dv[k] = a ? (lo ? bound : -bound) : qnan();
        cnt += a ? 1.0 : 0.0;
    }
    const double tot = tsum(cnt, c.red);
    if (threadIdx.x == 0) c.n_act = tot;
}

struct Res {
    double g, b, d, m, mu;
};

// residuals (view.py:272-288 on the DenseView, view.py:295-336)
__device__ Res residuals(C& c, const double* v, const double* pi, const double* lam, const double* t) {
    const double* dvec = c.V(c.o.act);
    double* rowv = c.V(c.o.rowv);
    double* rg = c.V(c.o.rg);
    double* rb = c.V(c.o.rb);
    double* rd = c.V(c.o.rd);
    double* crow = c.V(c.o.wall);   // lam_lo - lam_up per row (scratch, m <= nc)
    for (int r = threadIdx.x; r < c.m; r += blockDim.x) {
        rowv[r] = rowval(c, r, v);
        const double ll = !isnan(dvec[r]) ? lam[r] : 0.0;
        const double lu = !isnan(dvec[r + c.m]) ? lam[r + c.m] : 0.0;
        crow[r] = ll - lu;
    }
    __syncthreads();
    double mg = 0.0, mb = 0.0, md = 0.0, mm = 0.0, musum = 0.0;
    int ng_ = 0, nb_ = 0, nd_ = 0, nm_ = 0;
    for (int j = threadIdx.x; j < c.nv; j += blockDim.x) {
        double h = 0.0;
        for (int k = 0; k < c.nv; ++k) h = fma(c.H(j, k), v[k], h);
        double atp = 0.0;
        for (int i = 0; i < c.ne; ++i) atp = fma(c.A(i, j), pi[i], atp);
        const double r = ((h + c.f[DG][j]) - atp) - rows_t(c, j, crow);
        rg[j] = r;
        if (isnan(r)) ng_ = 1; else mg = fmax(mg, fabs(r));
    }
    for (int i = threadIdx.x; i < c.ne; i += blockDim.x) {
        double av = 0.0;
        for (int k = 0; k < c.nv; ++k) av = fma(c.A(i, k), v[k], av);
        const double r = -av + c.f[DBV][i];
        rb[i] = r;
        if (isnan(r)) nb_ = 1; else mb = fmax(mb, fabs(r));
    }
    for (int k = threadIdx.x; k < c.nc; k += blockDim.x) {
        double d = 0.0, mmv = 0.0;
        if (!isnan(dvec[k])) {
            const double cy = k < c.m ? rowv[k] : -rowv[k - c.m];
            d = (-cy + dvec[k]) + t[k];
            mmv = lam[k] * t[k];
            musum += mmv;
        }
        rd[k] = d;
        if (isnan(d)) nd_ = 1; else md = fmax(md, fabs(d));
        if (isnan(mmv)) nm_ = 1; else mm = fmax(mm, fabs(mmv));
    }
    Res o;
    o.g = tabsmax(mg, ng_, c.red);
    o.b = tabsmax(mb, nb_, c.red);
    o.d = tabsmax(md, nd_, c.red);
    o.m = tabsmax(mm, nm_, c.red);
    const double s = tsum(musum, c.red);
    o.mu = c.n_act > 0.0 ? s / c.n_act : 0.0;
    return o;
}

// factor (kkt_dense.py:117-165): returns 0 ok, 1 not positive definite /
// rank deficient (FactorizationFailed), 2 non-positive iterate
__device__ int factor(C& c, const double* lam, const double* t, double reg, double reg_dual,
                      long long& flops) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int nv = c.nv, ne = c.ne;
    const double* dvec = c.V(c.o.act);
    double* gam = c.V(c.o.gam);
    double* tinv = c.V(c.o.tinv);
    double* coef = c.V(c.o.rowv);
    int bad = 0;
    for (int k = tid; k < c.nc; k += T) {
        double g = 0.0, ti = 0.0;
        if (!isnan(dvec[k])) {
            if (lam[k] <= 0.0 || t[k] <= 0.0) bad = 1;
            ti = 1.0 / t[k];
            g = lam[k] * ti;
        }
        gam[k] = g;
        tinv[k] = ti;
    }
    if (__syncthreads_or(bad)) return 2;
    for (int r = tid; r < c.m; r += T) coef[r] = gam[r] + gam[r + c.m];
    __syncthreads();
    // Hred = H; Hred[idxb, idxb] += coef_box; Hred = (C' diag(coef_g) C) + Hred (add_reduced_hessian)
    double* L = c.V(c.o.L);
    for (int idx = tid; idx < nv * nv; idx += T) {
        const int i = idx / nv, j = idx - i * nv;
        double h = c.H(i, j);
        if (i == j)
            for (int r = 0; r < c.nb; ++r)
                if (c.p->idxb[r] == i) h += coef[r];
        if (c.ng) {
            double s = 0.0;
            for (int g = 0; g < c.ng; ++g) s = fma(c.Cg(g, i), coef[c.nb + g] * c.Cg(g, j), s);
            h = s + h;
        }
        if (i == j && reg != 0.0) h += reg;
        L[idx] = h;
    }
    if (c.ng) flops += 2ll * nv * nv * c.ng;
    __syncthreads();
    flops += (long long)nv * nv * nv / 3;
    if (c.p->method == 1 && ne) {
        // the null-space products use the assembled Hred (kkt_dense.py:154-156)
        double* Hc = c.V(c.o.Q);
        for (int idx = tid; idx < nv * nv; idx += T) Hc[idx] = L[idx];
        __syncthreads();
    }
    if (!tchol(L, nv, nv, c.flag)) return 1;
    if (!ne) return 0;
    if (c.p->method == 0) {
        // W = L^{-1} A' (solve_triangular, nv^2 ne flops), column i by warp (i mod warps)
        double* W = c.V(c.o.W);
        const int warp = tid >> 5, lane = tid & 31, nw = T >> 5;
        for (int i = warp; i < ne; i += nw) {
            for (int r = 0; r < nv; ++r) {
                double acc = 0.0;
                for (int k = lane; k < r; k += 32) acc = fma(L[r * nv + k], W[k * ne + i], acc);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(FULL, acc, o);
                if (lane == 0) W[r * ne + i] = (c.A(i, r) - acc) / L[r * nv + r];
                __syncwarp();
            }
        }
        flops += (long long)nv * nv * ne;
        __syncthreads();
        // M = W'W (+ reg_dual I), Lm = chol(M)
        double* M = c.V(c.o.M);
        for (int idx = tid; idx < ne * ne; idx += T) {
            const int i = idx / ne, j = idx - i * ne;
            double s = 0.0;
            for (int k = 0; k < nv; ++k) s = fma(W[k * ne + i], W[k * ne + j], s);
            if (i == j && reg_dual != 0.0) s += reg_dual;
            M[idx] = s;
        }
        flops += 2ll * ne * ne * nv;
        __syncthreads();
        flops += (long long)ne * ne * ne / 3;
        if (!tchol(M, ne, ne, c.flag)) return 1;
        return 0;
    }
    // ---- null space: Householder QR of A' (nv x ne): reflectors in W,
    // R in R, Z = last nv - ne columns of Q = H_1 .. H_ne in HZ ----
    const double* Hc = c.V(c.o.Q);
    double* Vr = c.V(c.o.W);
    double* Ra = c.V(c.o.R);
    // Vr <- A'
    for (int idx = tid; idx < nv * ne; idx += T) {
        const int r = idx / ne, i = idx - r * ne;
        Vr[idx] = c.A(i, r);
    }
    __syncthreads();
    double* tau = c.V(c.o.te1);
    for (int k = 0; k < ne; ++k) {
        // column k below the diagonal: x = Vr[k:, k]
        double s = 0.0;
        for (int r = k + tid; r < nv; r += T) s = fma(Vr[r * ne + k], Vr[r * ne + k], s);
        s = tsum(s, c.red);
        const double alpha = Vr[k * ne + k];
        const double nrm = sqrt(s);
        const double beta = alpha >= 0.0 ? -nrm : nrm;   // dlarfg sign convention
        const double v0 = alpha - beta;
        __syncthreads();
        if (tid == 0) {
            tau[k] = nrm > 0.0 ? (beta - alpha) / beta : 0.0;
            Ra[k * ne + k] = nrm > 0.0 ? beta : alpha;
        }
        for (int r = k + 1 + tid; r < nv; r += T) Vr[r * ne + k] = nrm > 0.0 ? Vr[r * ne + k] / v0 : 0.0;
        __syncthreads();
        if (tid == 0) Vr[k * ne + k] = 1.0;
        __syncthreads();
        // apply H_k = I - tau v v' to the remaining columns j > k
        for (int j = k + 1; j < ne; ++j) {
            double d = 0.0;
            for (int r = k + tid; r < nv; r += T) d = fma(Vr[r * ne + k], Vr[r * ne + j], d);
            d = tsum(d, c.red) * tau[k];
            for (int r = k + tid; r < nv; r += T) Vr[r * ne + j] = fma(-d, Vr[r * ne + k], Vr[r * ne + j]);
            __syncthreads();
            if (tid == 0) Ra[k * ne + j] = Vr[k * ne + j];
            __syncthreads();
        }
    }
    // rank check (kkt_dense.py:157-158)
    double amax = 0.0;
    for (int idx = tid; idx < ne * nv; idx += T) amax = fmax(amax, fabs(c.f[DA][idx]));
    amax = -tmin(-amax, c.red);
    int rank_bad = 0;
    if (tid == 0)
        for (int k = 0; k < ne; ++k)
            if (fabs(Ra[k * ne + k]) < 1e-14 * fmax(1.0, amax)) rank_bad = 1;
    if (__syncthreads_or(rank_bad)) return 1;
    // Hz = Z' (Hred Z) with Z the last nv - ne columns of Q = H_1 .. H_ne
    const int nz = nv - ne;
    double* HZ = c.V(c.o.HZ);        // Z (nv x nz)
    for (int idx = tid; idx < nv * nz; idx += T) {
        const int r = idx / nz, j = idx - r * nz;
        HZ[idx] = (r == ne + j) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int k = ne - 1; k >= 0; --k) {   // Z = H_1 (.. (H_ne [0; I]))
        for (int j = 0; j < nz; ++j) {
            double d = 0.0;
            for (int r = k + tid; r < nv; r += T) d = fma(Vr[r * ne + k], HZ[r * nz + j], d);
            d = tsum(d, c.red) * tau[k];
            for (int r = k + tid; r < nv; r += T) HZ[r * nz + j] = fma(-d, Vr[r * ne + k], HZ[r * nz + j]);
            __syncthreads();
        }
    }
    // Hz = Z' (Hred Z) (matmul_acc, 2 nz^2 nv counted; Hred Z inline)
    double* HRZ = c.V(c.o.HRZ);
    for (int idx = tid; idx < nv * nz; idx += T) {
        const int r = idx / nz, j = idx - r * nz;
        double s = 0.0;
        for (int k = 0; k < nv; ++k) s = fma(Hc[r * nv + k], HZ[k * nz + j], s);
        HRZ[idx] = s;
    }
    __syncthreads();
    double* Hz = c.V(c.o.Hz);
    for (int idx = tid; idx < nz * nz; idx += T) {
        const int i = idx / nz, j = idx - i * nz;
        double s = 0.0;
        for (int r = 0; r < nv; ++r) s = fma(HZ[r * nz + i], HRZ[r * nz + j], s);
        Hz[idx] = s;
    }
    flops += 2ll * nz * nz * nv;
    __syncthreads();
    flops += (long long)nz * nz * nz / 3;
    if (!tchol(Hz, nz, nz, c.flag)) return 1;
    return 0;
}

// RHS r_m per slot: ext, or (lam t - tau) + corr (solver.py:207-258)
struct Rm {
    double tau;
    const double* dla;
    const double* dta;
};

// solve (kkt_dense.py:200-231) + fold_rhs / recover_block (kkt_common.py:118-163)
__device__ int solve(C& c, const double* lam, const double* t, const Rm& rm, double* dv, double* dpi,
                     double* dlam, double* dt, long long& flops) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int nv = c.nv, ne = c.ne;
    const double* dvec = c.V(c.o.act);
    const double* gam = c.V(c.o.gam);
    const double* tinv = c.V(c.o.tinv);
    const double* rg = c.V(c.o.rg);
    const double* rb = c.V(c.o.rb);
    const double* rd = c.V(c.o.rd);
    double* wall = c.V(c.o.wall);
    double* rhat = c.V(c.o.rhat);
    double* crow = c.V(c.o.rowv);
    double* z = c.V(c.o.tv1);
    double* z2 = c.V(c.o.tv2);
    const double* L = c.V(c.o.L);
    for (int k = tid; k < c.nc; k += T) {
        double w = 0.0;
        if (!isnan(dvec[k])) {
            const double comp = lam[k] * t[k];
            double rmk = comp - rm.tau;
            if (rm.dla) rmk = rmk + rm.dla[k] * rm.dta[k];
            w = (lam[k] * rd[k] - rmk) * tinv[k];
        }
        wall[k] = w;
    }
    __syncthreads();
    for (int r = tid; r < c.m; r += T) crow[r] = wall[r] - wall[r + c.m];
    __syncthreads();
    for (int j = tid; j < nv; j += T) rhat[j] = rg[j] - rows_t(c, j, crow);
    __syncthreads();
    if (ne == 0) {
        for (int j = tid; j < nv; j += T) z[j] = rhat[j];
        __syncthreads();
        wtrsv(L, nv, nv, z, false);
        wtrsv(L, nv, nv, z, true);
        flops += 2ll * nv * nv;
        __syncthreads();
        for (int j = tid; j < nv; j += T) dv[j] = -z[j];
    } else if (c.p->method == 0) {
        const double* Lm = c.V(c.o.M);
        for (int j = tid; j < nv; j += T) z[j] = rhat[j];
        __syncthreads();
        wtrsv(L, nv, nv, z, false);
        wtrsv(L, nv, nv, z, true);
        flops += 2ll * nv * nv;
        __syncthreads();
        // rhs_pi = r_b + A z
        for (int i = tid; i < ne; i += T) {
            double s = 0.0;
            for (int k = 0; k < nv; ++k) s = fma(c.A(i, k), z[k], s);
            dpi[i] = rb[i] + s;
        }
        __syncthreads();
        wtrsv(Lm, ne, ne, dpi, false);
        wtrsv(Lm, ne, ne, dpi, true);
        flops += 2ll * ne * ne;
        __syncthreads();
        // dv = Hred^{-1} (A' dpi - rhat)
        for (int j = tid; j < nv; j += T) {
            double s = 0.0;
            for (int i = 0; i < ne; ++i) s = fma(c.A(i, j), dpi[i], s);
            z[j] = s - rhat[j];
        }
        __syncthreads();
        wtrsv(L, nv, nv, z, false);
        wtrsv(L, nv, nv, z, true);
        flops += 2ll * nv * nv;
        __syncthreads();
        for (int j = tid; j < nv; j += T) dv[j] = z[j];
    } else {
        const int nz = nv - ne;
        const double* Ra = c.V(c.o.R);
        const double* Vr = c.V(c.o.W);
        const double* tau = c.V(c.o.te1);
        const double* Hc = c.V(c.o.Q);
        const double* Zm = c.V(c.o.HZ);
        const double* Lz = c.V(c.o.Hz);
        // v_p = Q1 Ra^{-T} r_b = Q [Ra^{-T} r_b; 0]
        double* s = c.V(c.o.te2);
        for (int i = tid; i < ne; i += T) s[i] = rb[i];
        __syncthreads();
        wtrsv(Ra, ne, ne, s, true, true);
        flops += (long long)ne * ne;
        __syncthreads();
        for (int j = tid; j < nv; j += T) z[j] = j < ne ? s[j] : 0.0;
        __syncthreads();
        for (int k = ne - 1; k >= 0; --k) {   // Q x = H_1 (.. H_ne x)
            double d = 0.0;
            for (int r = k + tid; r < nv; r += T) d = fma(Vr[r * ne + k], z[r], d);
            d = tsum(d, c.red) * tau[k];
            for (int r = k + tid; r < nv; r += T) z[r] = fma(-d, Vr[r * ne + k], z[r]);
            __syncthreads();
        }
        // rhs_z = Z'(rhat + Hred v_p); q = -Hz^{-1} rhs_z
        for (int j = tid; j < nv; j += T) {
            double hv = 0.0;
            for (int k = 0; k < nv; ++k) hv = fma(Hc[j * nv + k], z[k], hv);
            z2[j] = rhat[j] + hv;
        }
        __syncthreads();
        // q = -Hz^{-1} Z' (rhat + Hred v_p), held in dv[0 .. nz)
        for (int i = tid; i < nz; i += T) {
            double a = 0.0;
            for (int r = 0; r < nv; ++r) a = fma(Zm[r * nz + i], z2[r], a);
            dv[i] = -a;
        }
        __syncthreads();
        wtrsv(Lz, nz, nz, dv, false);
        wtrsv(Lz, nz, nz, dv, true);
        flops += 2ll * nz * nz;
        __syncthreads();
        // dv = v_p + Z q  (q in dv[0..nz)): write into z2
        for (int j = tid; j < nv; j += T) {
            double a = 0.0;
            for (int i = 0; i < nz; ++i) a = fma(Zm[j * nz + i], dv[i], a);
            z2[j] = z[j] + a;
        }
        __syncthreads();
        for (int j = tid; j < nv; j += T) dv[j] = z2[j];
        __syncthreads();
        // dpi = Ra^{-1} Q1'(Hred dv + rhat): y = Q'(Hred dv + rhat), first ne entries
        for (int j = tid; j < nv; j += T) {
            double hv = 0.0;
            for (int k = 0; k < nv; ++k) hv = fma(Hc[j * nv + k], dv[k], hv);
            z[j] = hv + rhat[j];
        }
        __syncthreads();
        for (int k = 0; k < ne; ++k) {   // Q' x = H_ne (.. H_1 x)
            double d = 0.0;
            for (int r = k + tid; r < nv; r += T) d = fma(Vr[r * ne + k], z[r], d);
            d = tsum(d, c.red) * tau[k];
            for (int r = k + tid; r < nv; r += T) z[r] = fma(-d, Vr[r * ne + k], z[r]);
            __syncthreads();
        }
        for (int i = tid; i < ne; i += T) dpi[i] = z[i];
        __syncthreads();
        wtrsv(Ra, ne, ne, dpi, false, true);
        flops += (long long)ne * ne;
        __syncthreads();
    }
    __syncthreads();
    // recover_block: cy = Jc dv; dlam = w - gamma cy; dt = -r_d + cy (active slots)
    int nonfinite = 0;
    for (int r = tid; r < c.m; r += T) crow[r] = rowval(c, r, dv);
    __syncthreads();
    for (int k = tid; k < c.nc; k += T) {
        double dl = 0.0, dtt = 0.0;
        if (!isnan(dvec[k])) {
            const double cy = k < c.m ? crow[k] : -crow[k - c.m];
            dl = wall[k] - gam[k] * cy;
            dtt = -rd[k] + cy;
        }
        dlam[k] = dl;
        dt[k] = dtt;
        if (!isfinite(dl) || !isfinite(dtt)) nonfinite = 1;
    }
    for (int j = tid; j < nv; j += T)
        if (!isfinite(dv[j])) nonfinite = 1;
    for (int i = tid; i < ne; i += T)
        if (!isfinite(dpi[i])) nonfinite = 1;
    return __syncthreads_or(nonfinite);
}

__device__ double max_step(C& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double ftb) {
    const double* dvec = c.V(c.o.act);
    double a = INFINITY;
    for (int k = threadIdx.x; k < c.nc; k += blockDim.x) {
        if (!isnan(dvec[k])) {
            if (dlam[k] < 0.0) a = fmin(a, -lam[k] / dlam[k]);
            if (dt[k] < 0.0) a = fmin(a, -t[k] / dt[k]);
        }
    }
    a = tmin(a, c.red);
    return fmin(1.0, ftb * a);
}

__device__ double trial_mu(C& c, const double* lam, const double* t, const double* dlam,
                           const double* dt, double alpha) {
    const double* dvec = c.V(c.o.act);
    double s = 0.0;
    for (int k = threadIdx.x; k < c.nc; k += blockDim.x)
        if (!isnan(dvec[k])) s += (lam[k] + alpha * dlam[k]) * (t[k] + alpha * dt[k]);
    s = tsum(s, c.red);
    return c.n_act > 0.0 ? s / c.n_act : 0.0;
}

__global__ void __launch_bounds__(256) k_dense_ipm(DKParams p, SolveParams sp) {
    __shared__ double red[16];
    __shared__ int flag, qs;
    __shared__ double n_act_s;
    const int tid = threadIdx.x, T = blockDim.x;
    C c;
    c.p = &p;
    c.nv = p.nv; c.ne = p.ne; c.nb = p.nb; c.ng = p.ng; c.nc = p.nc; c.m = p.m;
    c.o = ws_layout(p.nv, p.ne, p.nc, p.m);
    c.w = p.ws + (long long)blockIdx.x * p.ws_slot;
    c.red = red;
    c.flag = &flag;
    const OcpIpmArgC& arg = sp.arg;
    while (true) {
        if (tid == 0) qs = atomicAdd(p.counter, 1);
        __syncthreads();
        const int q = qs;
        if (q >= p.B) break;
        for (int f = 0; f < 11; ++f) c.f[f] = p.f[f] + (long long)q * p.bs[f];
        setup(c);
        if (tid == 0) n_act_s = c.n_act;
        __syncthreads();
        c.n_act = n_act_s;
        double* v = c.V(c.o.v);
        double* pi = c.V(c.o.pi);
        double* lam = c.V(c.o.lam);
        double* t = c.V(c.o.t);
        double* dv = c.V(c.o.dv);
        double* dpi = c.V(c.o.dpi);
        double* dlam = c.V(c.o.dlam);
        double* dt = c.V(c.o.dt);
        double* alam = c.V(c.o.alam);
        double* at = c.V(c.o.at);
        const double* dvec = c.V(c.o.act);
        // cold start (solver.py:113-142): v = 0, pi = 0, t = max(-d, t0), lam = mu0 / t
        for (int j = tid; j < c.nv; j += T) v[j] = 0.0;
        for (int i = tid; i < c.ne; i += T) pi[i] = 0.0;
        for (int k = tid; k < c.nc; k += T) {
            double tv = 0.0, lv = 0.0;
            if (!isnan(dvec[k])) {
                tv = fmax(0.0 - dvec[k], arg.t0);
                lv = arg.mu0 / tv;
            }
            t[k] = tv;
            lam[k] = lv;
        }
        __syncthreads();
        double* trace = sp.trace ? sp.trace + (long long)q * arg.iter_max * 8 : nullptr;
        long long flops = 0;
        double alpha_last = 1.0;
        int it = 0, status = -1;
        Res res;
        const double reg2 = arg.reg_prim > 0.0 ? 2.0 * arg.reg_prim : 1e-8;
        while (true) {
            res = residuals(c, v, pi, lam, t);
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
            if (status >= 0) break;
            __syncthreads();
            int fs = factor(c, lam, t, arg.reg_prim, p.reg_dual, flops);
            if (fs == 1) {
                __syncthreads();
                fs = factor(c, lam, t, reg2, p.reg_dual, flops);
            }
            if (fs == 2) { status = OCPQP_STATUS_NONPOSITIVE_ITERATE; break; }
            if (fs == 1) { status = OCPQP_STATUS_FAILURE; break; }
            __syncthreads();
            int nf = solve(c, lam, t, Rm{0.0, nullptr, nullptr}, dv, dpi, alam, at, flops);
            if (nf) { status = OCPQP_STATUS_NAN; break; }
            const double alpha_aff = max_step(c, lam, t, alam, at, 1.0);
            const double mu_aff = trial_mu(c, lam, t, alam, at, alpha_aff);
            double sigma = 0.0;
            if (mu > 0.0) sigma = fmin(1.0, fmax(0.0, pow(mu_aff / mu, 3.0)));
            const double tau = sigma * mu;
            nf = solve(c, lam, t, Rm{tau, arg.pred_corr ? alam : nullptr, arg.pred_corr ? at : nullptr},
                       dv, dpi, dlam, dt, flops);
            if (arg.pred_corr && arg.cond_pred_corr) {
                const double a_t = max_step(c, lam, t, dlam, dt, 1.0);
                const double mu_t = trial_mu(c, lam, t, dlam, dt, a_t);
                if (!(mu_t <= arg.corr_ratio * mu_aff))
                    nf = solve(c, lam, t, Rm{tau, nullptr, nullptr}, dv, dpi, dlam, dt, flops);
            }
            if (nf) { status = OCPQP_STATUS_NAN; break; }
            const double alpha = max_step(c, lam, t, dlam, dt, arg.ftb);
            for (int j = tid; j < c.nv; j += T) v[j] += alpha * dv[j];
            for (int i = tid; i < c.ne; i += T) pi[i] += alpha * dpi[i];
            for (int k = tid; k < c.nc; k += T) {
                double lv = lam[k] + alpha * dlam[k];
                double tv = t[k] + alpha * dt[k];
                if (!isnan(dvec[k])) {
                    lv = fmax(lv, arg.lam_min);
                    tv = fmax(tv, arg.t_min);
                }
                lam[k] = lv;
                t[k] = tv;
            }
            if (trace && tid == 0 && it < arg.iter_max) {
                double* tr = trace + (long long)it * 8;
                tr[0] = alpha_aff; tr[1] = alpha; tr[2] = mu; tr[3] = sigma;
                tr[4] = res.g; tr[5] = res.b; tr[6] = res.d; tr[7] = res.m;
            }
            __syncthreads();
            alpha_last = alpha;
            ++it;
        }
        __syncthreads();
        double* gy = sp.y + (long long)q * c.nv;
        double* gpi = sp.pi + (long long)q * c.ne;
        double* glam = sp.lam + (long long)q * c.nc;
        double* gt = sp.t + (long long)q * c.nc;
        for (int j = tid; j < c.nv; j += T) gy[j] = v[j];
        for (int i = tid; i < c.ne; i += T) gpi[i] = pi[i];
        for (int k = tid; k < c.nc; k += T) { glam[k] = lam[k]; gt[k] = t[k]; }
        if (tid == 0) {
            sp.status[q] = status;
            sp.iters[q] = it;
            double* r = sp.res + (long long)q * 5;
            r[0] = res.g; r[1] = res.b; r[2] = res.d; r[3] = res.m; r[4] = res.mu;
            sp.flops[q] = flops;
        }
        __syncthreads();
    }
}

}  // namespace densek
}  // namespace ocpqp

// ---------------------------------------------------------------------------
// C ABI (include/ocpqp_b200.h: ocpqp_dense_*)
// ---------------------------------------------------------------------------
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

struct OcpDensePlan {
    int device = 0;
    int B = 0, nv = 0, ne = 0, nb = 0, ng = 0, method = 0;
    int slots = 0, threads = 128;
    long long ws_slot = 0;
    int* d_idxb = nullptr;
    int* d_counter = nullptr;
    double* d_ws = nullptr;
    double* d_defaults = nullptr;   // zeros | ones | -inf | +inf rows of length max_len
    long long max_len = 0;
};

namespace {
int dense_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    ocpqp::set_last_error(buf);
    return code;
}
}  // namespace

extern "C" int ocpqp_dense_plan_create(const OcpDenseDimC* dim, int32_t batch, int32_t method,
                                       OcpDensePlan** out) {
    using namespace ocpqp::densek;
    if (!dim || !out) return dense_fail(OCPQP_E_ARG, "NULL argument");
    *out = nullptr;
    if (batch < 0) return dense_fail(OCPQP_E_ARG, "batch must be >= 0");
    if (dim->nv < 0 || dim->ne < 0 || dim->nb < 0 || dim->ng < 0)
        return dense_fail(OCPQP_E_INVALID_DIM, "dense dims must be >= 0");
    if (dim->nb > dim->nv) return dense_fail(OCPQP_E_INVALID_DIM, "nb = %d exceeds nv = %d", dim->nb, dim->nv);
    if (dim->ns != 0) return dense_fail(OCPQP_E_UNSUPPORTED, "soft rows (ns > 0) with equality constraints are not provided");
    if (dim->ne > dim->nv) return dense_fail(OCPQP_E_INVALID_DIM, "ne = %d exceeds nv = %d", dim->ne, dim->nv);
    if (method != 0 && method != 1) return dense_fail(OCPQP_E_UNSUPPORTED, "kkt_method must be 0 (schur) or 1 (null_space)");
    for (int i = 0; i < dim->nb; ++i) {
        const int v = dim->idxb ? dim->idxb[i] : i;
        if (v < 0 || v >= dim->nv) return dense_fail(OCPQP_E_ARG, "idxb[%d] = %d outside 0..%d", i, v, dim->nv - 1);
        if (i && dim->idxb && v <= dim->idxb[i - 1]) return dense_fail(OCPQP_E_DIMENSION, "idxb entries must be strictly increasing");
    }
    OcpDensePlan* P = new OcpDensePlan();
    P->B = batch; P->nv = dim->nv; P->ne = dim->ne; P->nb = dim->nb; P->ng = dim->ng; P->method = method;
    cudaError_t e = cudaGetDevice(&P->device);
    int nsm = 148;
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, P->device);
    const int m = P->nb + P->ng, nc = 2 * m;
    const WS w = ws_layout(P->nv, P->ne, nc, m);
    P->ws_slot = std::max(2ll, (w.end + 1) & ~1ll);
    P->slots = std::max(1, std::min(std::max(1, batch), nsm * 4));
    P->max_len = std::max<long long>(1, std::max<long long>((long long)P->nv * P->nv,
                 std::max<long long>((long long)P->ne * P->nv, (long long)P->ng * P->nv)));
    P->max_len = std::max<long long>(P->max_len, m + 1);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_idxb, sizeof(int) * std::max(1, P->nb));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_counter, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_ws, sizeof(double) * (size_t)P->ws_slot * P->slots);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_defaults, sizeof(double) * 4 * P->max_len);
    if (e == cudaSuccess) {
        std::vector<int> ib(std::max(1, P->nb));
        for (int i = 0; i < P->nb; ++i) ib[i] = dim->idxb ? dim->idxb[i] : i;
        e = cudaMemcpy(P->d_idxb, ib.data(), sizeof(int) * ib.size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) {
        std::vector<double> d(4 * P->max_len);
        for (long long i = 0; i < P->max_len; ++i) {
            d[i] = 0.0; d[P->max_len + i] = 1.0; d[2 * P->max_len + i] = -INFINITY; d[3 * P->max_len + i] = INFINITY;
        }
        e = cudaMemcpy(P->d_defaults, d.data(), sizeof(double) * d.size(), cudaMemcpyHostToDevice);
    }
    if (e != cudaSuccess) {
        ocpqp_dense_plan_destroy(P);
        return dense_fail(OCPQP_E_CUDA, "dense plan allocation: %s", cudaGetErrorString(e));
    }
    *out = P;
    return OCPQP_OK;
}

extern "C" int ocpqp_dense_plan_destroy(OcpDensePlan* P) {
    if (!P) return OCPQP_OK;
    cudaFree(P->d_idxb); cudaFree(P->d_counter); cudaFree(P->d_ws); cudaFree(P->d_defaults);
    delete P;
    return OCPQP_OK;
}

extern "C" int ocpqp_dense_solve(OcpDensePlan* P, const OcpDenseDataC* data, const OcpIpmArgC* arg,
                                 double reg_dual, OcpIterC* iter, OcpStatsC* stats, void* stream) {
    using namespace ocpqp::densek;
    if (!P || !data || !arg || !iter || !stats) return dense_fail(OCPQP_E_ARG, "NULL argument");
    if (arg->itref_corr_max > 0 || arg->use_qr_fallback || arg->use_qr_always || arg->abs_form ||
        arg->warm_start != 0 || !arg->pred_corr)
        return dense_fail(OCPQP_E_UNSUPPORTED, "dense QPs with equality constraints run the speed-mode "
                                       "loop (no refinement, QR, absolute form or warm start)");
    if (P->B == 0) return OCPQP_OK;
    int prev = -1;
    cudaGetDevice(&prev);
    if (prev != P->device) cudaSetDevice(P->device);
    DKParams k;
    memset(&k, 0, sizeof(k));
    k.B = P->B; k.nv = P->nv; k.ne = P->ne; k.nb = P->nb; k.ng = P->ng;
    k.m = P->nb + P->ng; k.nc = 2 * k.m; k.method = P->method;
    k.idxb = P->d_idxb;
    const double* src[11] = {data->H, data->g, data->A, data->b, data->lb, data->ub, data->C,
                             data->lg, data->ug, data->maskl, data->masku};
    const int dflt[11] = {0, 0, 0, 0, 2, 3, 0, 2, 3, 1, 1};
    for (int f = 0; f < 11; ++f) {
        k.f[f] = src[f] ? src[f] : P->d_defaults + dflt[f] * P->max_len;
        k.bs[f] = src[f] ? data->batch_stride[f] : 0;
    }
    k.ws = P->d_ws; k.ws_slot = P->ws_slot; k.counter = P->d_counter;
    k.reg_dual = reg_dual;
    ocpqp::SolveParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.arg = *arg;
    sp.y = iter->y; sp.pi = iter->pi; sp.lam = iter->lam; sp.t = iter->t;
    sp.status = stats->status; sp.iters = stats->iterations; sp.res = stats->res;
    sp.flops = (long long*)stats->flops; sp.trace = stats->trace;
    cudaError_t e = cudaMemsetAsync(P->d_counter, 0, sizeof(int), (cudaStream_t)stream);
    if (e == cudaSuccess) {
        k_dense_ipm<<<P->slots, P->threads, 0, (cudaStream_t)stream>>>(k, sp);
        e = cudaGetLastError();
    }
    if (prev >= 0 && prev != P->device) cudaSetDevice(prev);
    if (e != cudaSuccess) return dense_fail(OCPQP_E_CUDA, "k_dense_ipm launch: %s", cudaGetErrorString(e));
    return OCPQP_OK;
}
