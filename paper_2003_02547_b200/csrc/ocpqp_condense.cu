// Batched partial and full condensing and expansion (reference
// condensing.py:451-619, condense :160-340, _cost_recursion :128-157 and
// expand_solution :343-429).  Full condensing is the one-block case over the
// whole horizon, terminal stage included, whose dense QP is emitted as a
// single-stage OCP-QP (N = 0, nx = 0, nu = nv) -- the form the IPM kernels
// solve identically to the reference's dense-QP backend when ne = 0.
//
// Host side (C++): the block structure and every row routing table are
// computed once per (dims, idxb, N1) -- they are identical for all QPs of a
// batch.  Device side: one CTA per (QP, block) work item runs the prediction
// recursion pred[i+1] = A pred[i] (+B), the backward cost recursion
// P/Y/beta, the condensed Hessian / gradient assembly and the constraint
// routing; expansion rolls the states forward, routes multipliers back and
// runs the costate recursion for pi.  All fp64.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "ocpqp_internal.h"

using namespace ocpqp;

namespace {

thread_local std::string pc_err;

int pc_fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    pc_err = buf;
    return code;
}

// canonical per-stage field sizes (include/ocpqp_b200.h)
long long fsize(int f, int nx, int nu, int nb, int ng, int ns, int nxn, bool last) {
    switch (f) {
        case OCPQP_F_A: return last ? 0 : (long long)nxn * nx;
        case OCPQP_F_B: return last ? 0 : (long long)nxn * nu;
        case OCPQP_F_b: return last ? 0 : nxn;
        case OCPQP_F_Q: return (long long)nx * nx;
        case OCPQP_F_S: return (long long)nu * nx;
        case OCPQP_F_R: return (long long)nu * nu;
        case OCPQP_F_q: return nx;
        case OCPQP_F_r: return nu;
        case OCPQP_F_lb: case OCPQP_F_ub: return nb;
        case OCPQP_F_C: return (long long)ng * nx;
        case OCPQP_F_D: return (long long)ng * nu;
        case OCPQP_F_lg: case OCPQP_F_ug: return ng;
        case OCPQP_F_maskl: case OCPQP_F_masku: return nb + ng;
        default: return ns;
    }
}

struct Dims {
    int N;
    std::vector<int> nx, nu, nb, ng, ns;
    std::vector<int> idxb;  // concatenated
    std::vector<int> idxs;  // concatenated
    std::vector<int> ib_off, is_off;
    std::vector<long long> foff;  // [(N+1) * NF]
    std::vector<long long> flen;  // [NF]
    // flat solution layout
    std::vector<int> u_off, x_off, pi_off, c_off, s_off;
    int ny = 0, ne = 0, nc = 0, nv = 0, ns_tot = 0;
    void finish() {
        const int S = N + 1;
        ib_off.assign(S, 0);
        is_off.assign(S, 0);
        for (int n = 1; n < S; ++n) {
            ib_off[n] = ib_off[n - 1] + nb[n - 1];
            is_off[n] = is_off[n - 1] + ns[n - 1];
        }
        foff.assign((size_t)S * OCPQP_NUM_FIELDS, 0);
        flen.assign(OCPQP_NUM_FIELDS, 0);
        for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
            long long o = 0;
            for (int n = 0; n < S; ++n) {
                foff[(size_t)n * OCPQP_NUM_FIELDS + f] = o;
                o += fsize(f, nx[n], nu[n], nb[n], ng[n], ns[n], n < N ? nx[n + 1] : 0, n == N);
            }
            flen[f] = o;
        }
        u_off.assign(S, 0); x_off.assign(S, 0); pi_off.assign(S, 0); c_off.assign(S, 0);
        s_off.assign(S, 0);
        int v = 0, p = 0, c = 0, sl = 0;
        for (int n = 0; n < S; ++n) {
            u_off[n] = v; x_off[n] = v + nu[n]; v += nu[n] + nx[n];
            pi_off[n] = p; if (n < N) p += nx[n + 1];
            c_off[n] = c; c += 2 * (nb[n] + ng[n]) + 2 * ns[n];
            s_off[n] = sl; sl += ns[n];
        }
        nv = v; ns_tot = sl; ny = v + 2 * sl; ne = p; nc = c;
    }
};

}  // namespace

// ---------------------------------------------------------------------------
// device tables
// ---------------------------------------------------------------------------
struct PcBlockDev {
    int n0, L, nx0, nv, nb_new, ng_new;   // block geometry; new stage k = block index
    int zx;        // x0 columns of z (nx0, or 0 when full condensing drops a fixed x0)
    int ox;        // leading z columns emitted as the new stage's x part (nx0; 0 for full)
    int row0;      // first entry of this block in the row tables
    int uoff0;     // first entry in the per-block-stage u offset table
    int s0, ns_new;  // the new stage's slacks: entries s0.. of the slack tables
};

struct PcParams {
    int B, nblk, N, N2;
    int full;               // full condensing: one block 0..N including the terminal stage
    int nfix; const int* fix_row; const int* fix_c;   // dropped stage-0 fixing rows (full, x0 dropped)
    int nxmax, nvmax, numax, Lmax;
    const PcBlockDev* blk;
    const int* uoff;        // z offset of u for each block stage (-1 when nu = 0)
    // routing of the new stage's rows (box rows first in new order, then general rows)
    const int* row_kind;    // 0 = box u-row, 1 = box x0-row, 2 = general from x-box, 3 = general row
    const int* row_stage;   // block-local stage i
    const int* row_src;     // original row index within the stage (0..m_i-1)
    const int* row_aux;     // z index (box rows) / state component c (kind 2) / general g (kind 3)
    // original and new stage dims / offsets
    const int* onx; const int* onu; const int* onb; const int* ong;
    const long long* ofoff;  // [(N+1) * NF]
    const long long* nfoff;  // [(N2+1) * NF]
    const int* o_u; const int* o_x; const int* o_pi; const int* o_c;   // original flat layout
    const int* n_u; const int* n_x; const int* n_pi; const int* n_c;   // condensed flat layout
    const int* o_ib;  const int* o_idxb;
    // soft rows: source (block-local stage, stage slack index) of each new slack,
    // slack offsets / counts of both layouts
    const int* slk_stage; const int* slk_j;
    const int* o_s; const int* n_s; const int* ons; const int* nns;
    int nv_s, nv_f, nst_s, nst_f;
    // data
    const double* fin[OCPQP_NUM_FIELDS]; long long bin[OCPQP_NUM_FIELDS];
    double* fout[OCPQP_NUM_FIELDS]; long long bout[OCPQP_NUM_FIELDS];
    // workspace
    double* ws; long long ws_slot; int* counter;
    // square-root cost recursion (condensing.py:134-146): per-slot extra workspace behind the
    // classical one; *fail = 1 + 4 q (chol(Q) not positive definite) or 2 + 4 q (rank-deficient stack)
    int sqrt_cost; int* fail;
    // solutions (expansion)
    const double* sy; const double* spi; const double* slam; const double* st;
    double* fy; double* fpi; double* flam; double* ft;
    int ny_s, ne_s, nc_s, ny_f, ne_f, nc_f;
};

namespace {

__device__ __forceinline__ const double* fin(const PcParams& p, int q, int f, int n) {
    return p.fin[f] + (long long)q * p.bin[f] + p.ofoff[(long long)n * OCPQP_NUM_FIELDS + f];
}
__device__ __forceinline__ double* fout(const PcParams& p, int q, int f, int k) {
    return p.fout[f] + (long long)q * p.bout[f] + p.nfoff[(long long)k * OCPQP_NUM_FIELDS + f];
}

// In-place lower Cholesky of the n x n matrix at L (row-major, only the lower
// triangle is read, as scipy.linalg.cholesky(lower=True) behind
// linalg.cholesky_factor, linalg.py:81-118); the upper triangle is zeroed.
// False on a pivot that is not > 0.
__device__ bool pc_team_chol(double* L, int n) {
    const int tid = threadIdx.x, T = blockDim.x;
    for (int k = 0; k < n; ++k) {
        const double d = L[k * n + k];
        if (!(d > 0.0)) {
            __syncthreads();
            return false;
        }
        const double dk = sqrt(d);
        __syncthreads();
        for (int i = k + tid; i < n; i += T) L[i * n + k] = i == k ? dk : L[i * n + k] / dk;
        __syncthreads();
        for (int e = tid; e < (n - k - 1) * (n - k - 1); e += T) {
            const int i = k + 1 + e / (n - k - 1), j = k + 1 + e % (n - k - 1);
            if (j <= i) L[i * n + j] -= L[i * n + k] * L[j * n + k];
        }
        __syncthreads();
    }
    for (int e = tid; e < n * n; e += T)
        if (e % n > e / n) L[e] = 0.0;
    __syncthreads();
    return true;
}

// Householder QR of the m x n (m >= n) row-major stack S in place (LAPACK
// dgeqr2 / dlarfg reflectors, the arithmetic of np.linalg.qr(mode="r")), then
// qr_cholesky's rank test and row-sign normalisation (linalg.py:152-187): the
// leading n x n block becomes R with a positive diagonal.  False when rank-deficient.
__device__ bool pc_team_qr(double* S, int m, int n, double* red) {
    const int tid = threadIdx.x, T = blockDim.x;
    const int lane = tid & 31, warp = tid >> 5, nwarp = (T + 31) >> 5;
    for (int k = 0; k < n; ++k) {
        double ss = 0.0;
        for (int i = k + 1 + tid; i < m; i += T) ss = fma(S[i * n + k], S[i * n + k], ss);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
        __syncthreads();
        if (lane == 0) red[warp] = ss;
        __syncthreads();
        ss = 0.0;
        for (int w = 0; w < nwarp; ++w) ss += red[w];
        if (ss == 0.0) continue;    // H = I (tau = 0)
        const double alpha = S[k * n + k];
        const double beta = -copysign(hypot(alpha, sqrt(ss)), alpha);
        const double tau = (beta - alpha) / beta;
        const double sc = 1.0 / (alpha - beta);
        __syncthreads();
        for (int i = k + 1 + tid; i < m; i += T) S[i * n + k] *= sc;
        __syncthreads();
        for (int j = k + 1 + warp; j < n; j += nwarp) {
            double w = 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) w = fma(S[i * n + k], S[i * n + j], w);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            w = (S[k * n + j] + w) * tau;
            for (int i = k + 1 + lane; i < m; i += 32) S[i * n + j] = fma(-w, S[i * n + k], S[i * n + j]);
            if (lane == 0) S[k * n + j] -= w;
        }
        if (tid == 0) S[k * n + k] = beta;
        __syncthreads();
    }
    double dmax = 0.0;
    for (int i = 0; i < n; ++i) dmax = fmax(dmax, fabs(S[i * n + i]));
    const double tol = (m > n ? m : n) * 2.220446049250313e-16 * dmax;
    int bad = 0;
    for (int i = 0; i < n; ++i)
        if (!(fabs(S[i * n + i]) > tol)) bad = 1;
    __syncthreads();
    if (bad) return false;
    for (int i = tid; i < n; i += T) {
        const double sg = S[i * n + i] < 0.0 ? -1.0 : 1.0;
        for (int j = 0; j < n; ++j) S[i * n + j] = j < i ? 0.0 : sg * S[i * n + j];
    }
    __syncthreads();
    return true;
}

// One (QP, block) condensing work item; team = CTA.
__device__ void condense_block(const PcParams& p, int q, int k, double* ws) {
    const int tid = threadIdx.x, T = blockDim.x;
    const PcBlockDev bk = p.blk[k];
    const int L = bk.L, n0 = bk.n0, nx0 = bk.nx0, nv = bk.nv;
    const int* uoff = p.uoff + bk.uoff0;
    const int XM = p.nxmax, VM = p.nvmax, UM = p.numax;
    // workspace carve-up
    double* P = ws;                                 // (L+1) * XM*XM
    double* Y = P + (long long)(p.Lmax + 1) * XM * XM;   // (L+1) * XM*UM
    double* gam = Y + (long long)(p.Lmax + 1) * XM * UM;     // (L+1) * XM
    double* bet = gam + (long long)(p.Lmax + 1) * XM;  // (L+1) * XM
    double* Hc = bet + (long long)(p.Lmax + 1) * XM;   // VM * VM
    double* gc = Hc + (long long)VM * VM;              // VM
    double* pr0 = gc + VM;                             // XM * VM
    double* pr1 = pr0 + (long long)XM * VM;            // XM * VM
    double* T1 = pr1 + (long long)XM * VM;             // XM * max(XM, UM)
    double* T2 = T1 + (long long)XM * (XM > UM ? XM : UM);  // XM * UM
    // square-root cost recursion only (behind the classical workspace)
    double* Uc = T2 + (long long)XM * UM + 64;         // XM * XM: U_{n+1} (upper triangular)
    double* Stk = Uc + (long long)XM * XM;             // 2 XM * XM: [chol(Q_n)'; U_{n+1} A], then R
    double* UBb = Stk + 2ll * XM * XM;                 // XM * UM: U_{n+1} B
    double* Lq = UBb + (long long)XM * UM;             // XM * XM: chol(Q_n)
    __shared__ double s_red[32];
    const bool sq = p.sqrt_cost != 0;
    // gamma forward: gamma[0] = 0, gamma[i+1] = A gamma[i] + b  (condensing.py:199-207)
    // (full condensing without x0: gamma[0] = x0hat from the fixing rows, :97-118, :197)
    for (int a = tid; a < nx0; a += T) gam[a] = 0.0;
    __syncthreads();
    if (tid == 0 && p.full && bk.zx == 0)
        for (int j = 0; j < p.nfix; ++j) gam[p.fix_c[j]] = fin(p, q, OCPQP_F_lb, 0)[p.fix_row[j]];
    __syncthreads();
    for (int i = 0; i < L; ++i) {
        const int n = n0 + i, nx = p.onx[n], nxn = p.onx[n + 1];
        const double* A = fin(p, q, OCPQP_F_A, n);
        const double* b = fin(p, q, OCPQP_F_b, n);
        for (int a = tid; a < nxn; a += T) {
            double s = 0.0;
            for (int c = 0; c < nx; ++c) s = fma(A[a * nx + c], gam[i * XM + c], s);
            gam[(i + 1) * XM + a] = s + b[a];
        }
        __syncthreads();
    }
    // zero Hc, gc
    for (int e = tid; e < nv * nv; e += T) Hc[e] = 0.0;
    for (int e = tid; e < nv; e += T) gc[e] = 0.0;
    __syncthreads();
    // backward cost recursion (condensing.py:148-157) with P[L] = 0, beta[L] = 0 (the
    // sub-QP's zero-cost terminal placeholder, condensing.py:432-448, 211); full
    // condensing starts from the real terminal stage: P[N] = sym(Q_N),
    // beta[N] = q_N + Q_N gamma_N, and its inputs (if any) enter with R_N, S_N'
    // (condensing.py:151, 209, 238-241)
    {
        const int nxL = p.onx[n0 + L];
        double* PL = P + (long long)L * XM * XM;
        if (p.full) {
            const int nuL = p.onu[n0 + L];
            const double* Q = fin(p, q, OCPQP_F_Q, n0 + L);
            const double* S = fin(p, q, OCPQP_F_S, n0 + L);
            const double* R = fin(p, q, OCPQP_F_R, n0 + L);
            const double* qv = fin(p, q, OCPQP_F_q, n0 + L);
            const double* rv = fin(p, q, OCPQP_F_r, n0 + L);
            if (sq) {
                // U_N = chol(Q_N)', P_N = U_N' U_N (condensing.py:135-137)
                for (int e = tid; e < nxL * nxL; e += T) Lq[e] = Q[e];
                __syncthreads();
                if (!pc_team_chol(Lq, nxL)) {
                    if (tid == 0) atomicCAS(p.fail, 0, 1 + 4 * q);
                    return;
                }
                for (int e = tid; e < nxL * nxL; e += T) {
                    const int a = e / nxL, c = e - a * nxL;
                    Uc[e] = Lq[c * nxL + a];
                    const int km = a < c ? a : c;
                    double v = 0.0;
                    for (int k2 = 0; k2 <= km; ++k2) v = fma(Lq[a * nxL + k2], Lq[c * nxL + k2], v);
                    PL[e] = v;
                }
            } else
            for (int e = tid; e < nxL * nxL; e += T) {
                const int a = e / nxL, c = e - a * nxL;
                PL[e] = 0.5 * (Q[e] + Q[c * nxL + a]);
            }
            for (int a = tid; a < nxL; a += T) {
                double qg = 0.0;
                for (int c = 0; c < nxL; ++c) qg = fma(Q[a * nxL + c], gam[L * XM + c], qg);
                bet[L * XM + a] = qv[a] + qg;
            }
            const int ou = uoff[L];
            if (nuL && ou >= 0) {
                double* YL = Y + (long long)L * XM * UM;
                for (int e = tid; e < nxL * nuL; e += T) {
                    const int a = e / nuL, c = e - a * nuL;
                    YL[e] = S[c * nxL + a];
                }
                for (int e = tid; e < nuL * nuL; e += T) {
                    const int a = e / nuL, c = e - a * nuL;
                    Hc[(ou + a) * nv + ou + c] = R[e];
                }
                for (int a = tid; a < nuL; a += T) {
                    double sg = 0.0;
                    for (int c = 0; c < nxL; ++c) sg = fma(S[a * nxL + c], gam[L * XM + c], sg);
                    gc[ou + a] = rv[a] + sg;
                }
            }
        } else {
            for (int e = tid; e < nxL * nxL; e += T) PL[e] = 0.0;
            for (int a = tid; a < nxL; a += T) bet[L * XM + a] = 0.0;
        }
    }
    __syncthreads();
    for (int i = L - 1; i >= 0; --i) {
        const int n = n0 + i, nx = p.onx[n], nu = p.onu[n], nxn = p.onx[n + 1];
        const double* A = fin(p, q, OCPQP_F_A, n);
        const double* Bm = fin(p, q, OCPQP_F_B, n);
        const double* Q = fin(p, q, OCPQP_F_Q, n);
        const double* S = fin(p, q, OCPQP_F_S, n);
        const double* R = fin(p, q, OCPQP_F_R, n);
        const double* qv = fin(p, q, OCPQP_F_q, n);
        const double* rv = fin(p, q, OCPQP_F_r, n);
        const double* Pn = P + (long long)(i + 1) * XM * XM;
        // PA = P_{n+1} A (nxn x nx) -> T1 ; PB = P_{n+1} B (nxn x nu) -> T2
        for (int e = tid; e < nxn * nx; e += T) {
            const int a = e / nx, c = e - a * nx;
            double s = 0.0;
            for (int k2 = 0; k2 < nxn; ++k2) s = fma(Pn[a * nxn + k2], A[k2 * nx + c], s);
            T1[e] = s;
        }
        for (int e = tid; e < nxn * nu; e += T) {
            const int a = e / nu, c = e - a * nu;
            double s = 0.0;
            for (int k2 = 0; k2 < nxn; ++k2) s = fma(Pn[a * nxn + k2], Bm[k2 * nu + c], s);
            T2[e] = s;
        }
        __syncthreads();
        // Y = A' PB + S'  (nx x nu) ; Pt = A' PA + Q (nx x nx) into P_i (unsymmetrised)
        double* Yi = Y + (long long)i * XM * UM;
        double* Pi = P + (long long)i * XM * XM;
        if (sq) {
            // UA = U_{n+1} A below chol(Q_n)' in the stack, UB = U_{n+1} B,
            // Y = UA' UB + S', U_n = qr_cholesky([Uq; UA]), P_n = U_n' U_n
            // (condensing.py:138-146)
            for (int e = tid; e < nxn * nx; e += T) {
                const int a = e / nx, c = e - a * nx;
                double v = 0.0;
                for (int k2 = a; k2 < nxn; ++k2) v = fma(Uc[a * nxn + k2], A[k2 * nx + c], v);
                Stk[(nx + a) * nx + c] = v;
            }
            for (int e = tid; e < nxn * nu; e += T) {
                const int a = e / nu, c = e - a * nu;
                double v = 0.0;
                for (int k2 = a; k2 < nxn; ++k2) v = fma(Uc[a * nxn + k2], Bm[k2 * nu + c], v);
                UBb[e] = v;
            }
            for (int e = tid; e < nx * nx; e += T) Lq[e] = Q[e];
            __syncthreads();
            for (int e = tid; e < nx * nu; e += T) {
                const int a = e / nu, c = e - a * nu;
                double v = 0.0;
                for (int k2 = 0; k2 < nxn; ++k2) v = fma(Stk[(nx + k2) * nx + a], UBb[k2 * nu + c], v);
                Yi[e] = v + S[c * nx + a];
            }
            if (!pc_team_chol(Lq, nx)) {
                if (tid == 0) atomicCAS(p.fail, 0, 1 + 4 * q);
                return;
            }
            for (int e = tid; e < nx * nx; e += T) {
                const int a = e / nx, c = e - a * nx;
                Stk[e] = Lq[c * nx + a];
            }
            __syncthreads();
            if (!pc_team_qr(Stk, nx + nxn, nx, s_red)) {
                if (tid == 0) atomicCAS(p.fail, 0, 2 + 4 * q);
                return;
            }
            for (int e = tid; e < nx * nx; e += T) {
                const int a = e / nx, c = e - a * nx;
                const int km = a < c ? a : c;
                double v = 0.0;
                for (int k2 = 0; k2 <= km; ++k2) v = fma(Stk[k2 * nx + a], Stk[k2 * nx + c], v);
                Pi[e] = v;
            }
        } else {
        for (int e = tid; e < nx * nu; e += T) {
            const int a = e / nu, c = e - a * nu;
            double s = 0.0;
            for (int k2 = 0; k2 < nxn; ++k2) s = fma(A[k2 * nx + a], T2[k2 * nu + c], s);
            Yi[e] = s + S[c * nx + a];
        }
        for (int e = tid; e < nx * nx; e += T) {
            const int a = e / nx, c = e - a * nx;
            double s = 0.0;
            for (int k2 = 0; k2 < nxn; ++k2) s = fma(A[k2 * nx + a], T1[k2 * nx + c], s);
            Pi[e] = s + Q[e];
        }
        }
        // condensed u_i block R + B' (P_{n+1} B) and gradient r + S gamma + B' beta
        // (condensing.py:229-237)
        const int ou = uoff[i];
        if (nu && ou >= 0) {
            for (int e = tid; e < nu * nu; e += T) {
                const int a = e / nu, c = e - a * nu;
                double s = 0.0;
                for (int k2 = 0; k2 < nxn; ++k2) s = fma(Bm[k2 * nu + a], T2[k2 * nu + c], s);
                Hc[(ou + a) * nv + ou + c] = R[e] + s;
            }
            for (int a = tid; a < nu; a += T) {
                double sg = 0.0, bb = 0.0;
                for (int c = 0; c < nx; ++c) sg = fma(S[a * nx + c], gam[i * XM + c], sg);
                for (int c = 0; c < nxn; ++c) bb = fma(Bm[c * nu + a], bet[(i + 1) * XM + c], bb);
                gc[ou + a] = (rv[a] + sg) + bb;
            }
        }
        // beta_i = q + Q gamma_i + A' beta_{i+1}  (condensing.py:213-217)
        for (int a = tid; a < nx; a += T) {
            double qg = 0.0, ab = 0.0;
            for (int c = 0; c < nx; ++c) qg = fma(Q[a * nx + c], gam[i * XM + c], qg);
            for (int c = 0; c < nxn; ++c) ab = fma(A[c * nx + a], bet[(i + 1) * XM + c], ab);
            bet[i * XM + a] = (qv[a] + qg) + ab;
        }
        __syncthreads();
        if (sq) {
            for (int e = tid; e < nx * nx; e += T) Uc[e] = Stk[e];
            __syncthreads();
            continue;
        }
        // symmetrise P_i in place (read pairs, then write)
        for (int e = tid; e < nx * nx; e += T) {
            const int a = e / nx, c = e - a * nx;
            if (c < a) {
                const double v = 0.5 * (Pi[e] + Pi[c * nx + a]);
                Pi[e] = v;
                Pi[c * nx + a] = v;
            } else if (c == a) {
                Pi[e] = 0.5 * (Pi[e] + Pi[e]);
            }
        }
        __syncthreads();
    }
    // x0 block and gradient (condensing.py:220-222), when x0 is a variable
    const int zx = bk.zx, ox = bk.ox;
    for (int e = tid; e < zx * zx; e += T) {
        const int a = e / zx, c = e - a * zx;
        Hc[a * nv + c] = P[e];
    }
    for (int a = tid; a < zx; a += T) gc[a] = bet[a];
    __syncthreads();
    // forward pass over the prediction operators (condensing.py:196-207, 242-245)
    double* pr = pr0;
    double* prn = pr1;
    for (int e = tid; e < nx0 * nv; e += T) {
        const int a = e / nv, c = e - a * nv;
        pr[e] = (c == a && c < zx) ? 1.0 : 0.0;
    }
    __syncthreads();
    for (int i = 0; i <= L; ++i) {
        const int n = n0 + i, nx = p.onx[n];
        if (i < L || p.full) {
            const int nu = p.onu[n], ou = uoff[i];
            if (nu && ou >= 0) {
                // cols = pred_i' Y_i (nv x nu); Hc[:, u_i] += cols; Hc[u_i, :] += cols'
                const double* Yi = Y + (long long)i * XM * UM;
                for (int e = tid; e < nv * nu; e += T) {
                    const int a = e / nu, c = e - a * nu;
                    double s = 0.0;
                    for (int k2 = 0; k2 < nx; ++k2) s = fma(pr[k2 * nv + a], Yi[k2 * nu + c], s);
                    T1[e] = s;  // reuse as cols (nv x nu <= XM*max(XM,UM) checked on host)
                }
                __syncthreads();
                for (int e = tid; e < nv * nu; e += T) {
                    const int a = e / nu, c = e - a * nu;
                    Hc[a * nv + ou + c] += T1[e];
                }
                __syncthreads();
                for (int e = tid; e < nv * nu; e += T) {
                    const int a = e / nu, c = e - a * nu;
                    Hc[(ou + c) * nv + a] += T1[e];
                }
                __syncthreads();
            }
        }
        // constraint rows that read pred_i: general rows of this stage, x-box rows (i > 0)
        for (int r = bk.nb_new; r < bk.nb_new + bk.ng_new; ++r) {
            const int ridx = bk.row0 + r;
            if (p.row_stage[ridx] != i) continue;
            const int kind = p.row_kind[ridx];
            const int g = r - bk.nb_new;
            double* Cz = fout(p, q, OCPQP_F_C, k) + (long long)g * ox;
            double* Dz = fout(p, q, OCPQP_F_D, k) + (long long)g * (nv - ox);
            if (kind == 2) {
                const int cc = p.row_aux[ridx];
                for (int e = tid; e < nv; e += T) {
                    const double v = pr[cc * nv + e];
                    if (e < ox) Cz[e] = v; else Dz[e - ox] = v;
                }
                if (tid == 0) {
                    const int src = p.row_src[ridx];
                    const double gsh = gam[i * XM + cc];
                    fout(p, q, OCPQP_F_lg, k)[g] = fin(p, q, OCPQP_F_lb, n)[src] - gsh;
                    fout(p, q, OCPQP_F_ug, k)[g] = fin(p, q, OCPQP_F_ub, n)[src] - gsh;
                }
            } else {
                const int gg = p.row_aux[ridx];
                const int nu = p.onu[n], ou = uoff[i];
                const double* Cg = fin(p, q, OCPQP_F_C, n) + (long long)gg * nx;
                const double* Dg = fin(p, q, OCPQP_F_D, n) + (long long)gg * nu;
                for (int e = tid; e < nv; e += T) {
                    double s = 0.0;
                    for (int c = 0; c < nx; ++c) s = fma(Cg[c], pr[c * nv + e], s);
                    double base = 0.0;
                    if (nu && ou >= 0 && e >= ou && e < ou + nu) base = Dg[e - ou];
                    const double v = base + s;
                    if (e < ox) Cz[e] = v; else Dz[e - ox] = v;
                }
                if (tid == 0) {
                    double sh = 0.0;
                    for (int c = 0; c < nx; ++c) sh = fma(Cg[c], gam[i * XM + c], sh);
                    fout(p, q, OCPQP_F_lg, k)[g] = fin(p, q, OCPQP_F_lg, n)[gg] - sh;
                    fout(p, q, OCPQP_F_ug, k)[g] = fin(p, q, OCPQP_F_ug, n)[gg] - sh;
                }
            }
        }
        __syncthreads();
        if (i == L) break;
        // pred_{i+1} = A pred_i (+ B at u_i)
        {
            const int nu = p.onu[n], ou = uoff[i], nxn = p.onx[n + 1];
            const double* A = fin(p, q, OCPQP_F_A, n);
            const double* Bm = fin(p, q, OCPQP_F_B, n);
            for (int e = tid; e < nxn * nv; e += T) {
                const int a = e / nv, c = e - a * nv;
                double s = 0.0;
                for (int k2 = 0; k2 < nx; ++k2) s = fma(A[a * nx + k2], pr[k2 * nv + c], s);
                if (nu && ou >= 0 && c >= ou && c < ou + nu) s += Bm[a * nu + (c - ou)];
                prn[e] = s;
            }
            __syncthreads();
            double* tmp = pr; pr = prn; prn = tmp;
        }
    }
    // new stage dynamics: A = pred_L[:, :nx0], B = pred_L[:, nx0:], b = gamma_L
    if (!p.full) {
        const int nxn = p.onx[n0 + L], nun = nv - nx0;
        double* Ao = fout(p, q, OCPQP_F_A, k);
        double* Bo = fout(p, q, OCPQP_F_B, k);
        double* bo = fout(p, q, OCPQP_F_b, k);
        for (int e = tid; e < nxn * nv; e += T) {
            const int a = e / nv, c = e - a * nv;
            if (c < nx0) Ao[a * nx0 + c] = pr[e]; else Bo[a * nun + (c - nx0)] = pr[e];
        }
        for (int a = tid; a < nxn; a += T) bo[a] = gam[L * XM + a];
    }
    __syncthreads();
    // Hc = 0.5 (Hc + Hc') and the new stage cost blocks (condensing.py:246, 504-509)
    {
        const int nun = nv - ox;
        double* Qo = fout(p, q, OCPQP_F_Q, k);
        double* So = fout(p, q, OCPQP_F_S, k);
        double* Ro = fout(p, q, OCPQP_F_R, k);
        double* qo = fout(p, q, OCPQP_F_q, k);
        double* ro = fout(p, q, OCPQP_F_r, k);
        for (int e = tid; e < nv * nv; e += T) {
            const int a = e / nv, c = e - a * nv;
            const double v = 0.5 * (Hc[e] + Hc[c * nv + a]);
            if (a < ox && c < ox) Qo[a * ox + c] = v;
            else if (a >= ox && c < ox) So[(a - ox) * ox + c] = v;
            else if (a >= ox && c >= ox) Ro[(a - ox) * nun + (c - ox)] = v;
        }
        for (int a = tid; a < nv; a += T) {
            if (a < ox) qo[a] = gc[a]; else ro[a - ox] = gc[a];
        }
    }
    // box rows of the new stage (bounds unshifted) and masks of every row
    for (int r = tid; r < bk.nb_new + bk.ng_new; r += T) {
        const int ridx = bk.row0 + r;
        const int i = p.row_stage[ridx], src = p.row_src[ridx];
        const int n = n0 + i;
        if (r < bk.nb_new) {
            fout(p, q, OCPQP_F_lb, k)[r] = fin(p, q, OCPQP_F_lb, n)[src];
            fout(p, q, OCPQP_F_ub, k)[r] = fin(p, q, OCPQP_F_ub, n)[src];
        }
        fout(p, q, OCPQP_F_maskl, k)[r] = fin(p, q, OCPQP_F_maskl, n)[src];
        fout(p, q, OCPQP_F_masku, k)[r] = fin(p, q, OCPQP_F_masku, n)[src];
    }
    // soft-row data travels with its row (condensing.py:289-334, 523-534)
    for (int jn = tid; jn < bk.ns_new; jn += T) {
        const int e = bk.s0 + jn;
        const int n = n0 + p.slk_stage[e], j = p.slk_j[e];
        const int sf[6] = {OCPQP_F_Zl, OCPQP_F_Zu, OCPQP_F_zl, OCPQP_F_zu, OCPQP_F_sl_lb, OCPQP_F_su_lb};
#pragma unroll
        for (int f = 0; f < 6; ++f) fout(p, q, sf[f], k)[jn] = fin(p, q, sf[f], n)[j];
    }
}

// copy the terminal stage verbatim (condensing.py:547-549)
__device__ void copy_terminal(const PcParams& p, int q) {
    const int tid = threadIdx.x, T = blockDim.x;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
        if (f == OCPQP_F_A || f == OCPQP_F_B || f == OCPQP_F_b) continue;
        const long long a0 = p.ofoff[(long long)p.N * OCPQP_NUM_FIELDS + f];
        const int nx = p.onx[p.N], nu = p.onu[p.N], nb = p.onb[p.N], ng = p.ong[p.N];
        long long sz;
        switch (f) {
            case OCPQP_F_Q: sz = (long long)nx * nx; break;
            case OCPQP_F_S: sz = (long long)nu * nx; break;
            case OCPQP_F_R: sz = (long long)nu * nu; break;
            case OCPQP_F_q: sz = nx; break;
            case OCPQP_F_r: sz = nu; break;
            case OCPQP_F_lb: case OCPQP_F_ub: sz = nb; break;
            case OCPQP_F_C: sz = (long long)ng * nx; break;
            case OCPQP_F_D: sz = (long long)ng * nu; break;
            case OCPQP_F_lg: case OCPQP_F_ug: sz = ng; break;
            case OCPQP_F_maskl: case OCPQP_F_masku: sz = nb + ng; break;
            default: sz = p.ons[p.N]; break;   // soft-row fields
        }
        const double* src = p.fin[f] + (long long)q * p.bin[f] + a0;
        double* dst = fout(p, q, f, p.N2);
        for (long long e = tid; e < sz; e += T) dst[e] = src[e];
    }
}

__global__ void __launch_bounds__(256) k_pc_condense(PcParams p) {
    __shared__ int s_item;
    double* ws = p.ws + (long long)blockIdx.x * p.ws_slot;
    const int per = p.nblk + (p.full ? 0 : 1);
    const int items = p.B * per;
    while (true) {
        if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1);
        __syncthreads();
        const int it = s_item;
        __syncthreads();
        if (it >= items) break;
        const int q = it / per, k = it - q * per;
        if (k < p.nblk) condense_block(p, q, k, ws);
        else copy_terminal(p, q);
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// expansion (condensing.py:553-619, 343-429)
// ---------------------------------------------------------------------------
__device__ void expand_block(const PcParams& p, int q, int k, double* ws) {
    const int tid = threadIdx.x, T = blockDim.x;
    const PcBlockDev bk = p.blk[k];
    const int L = bk.L, n0 = bk.n0, nx0 = bk.nx0;
    const int* uoff = p.uoff + bk.uoff0;
    const double* sy = p.sy + (long long)q * p.ny_s;
    const double* spi = p.spi + (long long)q * p.ne_s;
    const double* slam = p.slam + (long long)q * p.nc_s;
    const double* sts = p.st + (long long)q * p.nc_s;
    double* fy = p.fy + (long long)q * p.ny_f;
    double* fpi = p.fpi + (long long)q * p.ne_f;
    double* flam = p.flam + (long long)q * p.nc_f;
    double* ft = p.ft + (long long)q * p.nc_f;
    const double* xk = sy + p.n_x[k];
    const double* uk = sy + p.n_u[k];
    double* xs = ws;                           // (L+1) * XM
    double* ctx = xs + (long long)(p.Lmax + 1) * p.nxmax;   // XM
    double* pis = ctx + p.nxmax;               // XM
    double* gap = pis + p.nxmax;               // XM
    const int XM = p.nxmax;
    const int ox = bk.ox;
    // forward rollout (condensing.py:359-367); full condensing: x0 from z or x0hat
    if (!p.full) {
        for (int a = tid; a < nx0; a += T) xs[a] = xk[a];
    } else if (bk.zx) {
        for (int a = tid; a < nx0; a += T) xs[a] = uk[a];
    } else if (tid == 0) {
        for (int j = 0; j < p.nfix; ++j) xs[p.fix_c[j]] = fin(p, q, OCPQP_F_lb, 0)[p.fix_row[j]];
    }
    __syncthreads();
    for (int i = 0; i < L + (p.full ? 1 : 0); ++i) {
        const int n = n0 + i, nx = p.onx[n], nu = p.onu[n];
        const int ou = uoff[i];
        for (int a = tid; a < nu; a += T) fy[p.o_u[n] + a] = (ou >= 0) ? uk[ou - ox + a] : 0.0;
        for (int a = tid; a < nx; a += T) fy[p.o_x[n] + a] = xs[i * XM + a];
        if (i == L) break;
        const int nxn = p.onx[n + 1];
        const double* A = fin(p, q, OCPQP_F_A, n);
        const double* Bm = fin(p, q, OCPQP_F_B, n);
        const double* b = fin(p, q, OCPQP_F_b, n);
        for (int a = tid; a < nxn; a += T) {
            double ax = 0.0, bu = 0.0;
            for (int c = 0; c < nx; ++c) ax = fma(A[a * nx + c], xs[i * XM + c], ax);
            if (ou >= 0)
                for (int c = 0; c < nu; ++c) bu = fma(Bm[a * nu + c], uk[ou - ox + c], bu);
            xs[(i + 1) * XM + a] = (ax + bu) + b[a];
        }
        __syncthreads();
    }
    // route lam / t of the new stage back to the original rows (condensing.py:369-396, 572-591)
    const int mn = bk.nb_new + bk.ng_new;
    for (int r = tid; r < mn; r += T) {
        const int ridx = bk.row0 + r;
        const int i = p.row_stage[ridx], src = p.row_src[ridx];
        const int n = n0 + i;
        const int mo = p.onb[n] + p.ong[n];
        const int cs = p.n_c[k], cf = p.o_c[n];
        flam[cf + src] = slam[cs + r];
        flam[cf + mo + src] = slam[cs + mn + r];
        ft[cf + src] = sts[cs + r];
        ft[cf + mo + src] = sts[cs + mn + r];
    }
    // slacks and their multipliers (condensing.py:397-405, 592-601)
    for (int jn = tid; jn < bk.ns_new; jn += T) {
        const int e = bk.s0 + jn;
        const int n = n0 + p.slk_stage[e], j = p.slk_j[e];
        const int mo = p.onb[n] + p.ong[n], ons = p.ons[n], nns = p.nns[k];
        const int cs = p.n_c[k] + 2 * mn, cf = p.o_c[n] + 2 * mo;
        fy[p.nv_f + p.o_s[n] + j] = sy[p.nv_s + p.n_s[k] + jn];
        fy[p.nv_f + p.nst_f + p.o_s[n] + j] = sy[p.nv_s + p.nst_s + p.n_s[k] + jn];
        flam[cf + j] = slam[cs + jn];
        flam[cf + ons + j] = slam[cs + nns + jn];
        ft[cf + j] = sts[cs + jn];
        ft[cf + ons + j] = sts[cs + nns + jn];
    }
    __syncthreads();
    // costate recursion (condensing.py:397-412) seeded with the short-horizon pi_k;
    // full condensing runs it from the terminal stage (no seed) down to the
    // stage-0 stationarity gap of the dropped fixing rows (:414-428)
    if (!p.full) {
        for (int a = tid; a < p.onx[n0 + L]; a += T) pis[a] = spi[p.n_pi[k] + a];
        __syncthreads();
        if (L >= 1)
            for (int a = tid; a < p.onx[n0 + L]; a += T) fpi[p.o_pi[n0 + L - 1] + a] = pis[a];
    }
    const bool want_gap = p.full && bk.zx == 0 && p.nfix > 0;
    for (int m = p.full ? L : L - 1; m >= (want_gap ? 0 : 1); --m) {
        const int n = n0 + m, nx = p.onx[n], nu = p.onu[n];
        const int nxn = (p.full && m == L) ? 0 : p.onx[n + 1];
        const int nb = p.onb[n], ng = p.ong[n], mo = nb + ng;
        const int cf = p.o_c[n];
        // (C' lam)_x of stage n over the masked multipliers (view.py:145-153, 197-205)
        for (int a = tid; a < nx; a += T) {
            double out = 0.0;
            for (int r = 0; r < nb; ++r) {
                if (p.o_idxb[p.o_ib[n] + r] == nu + a) {
                    const double ll = (fin(p, q, OCPQP_F_maskl, n)[r] != 0.0 &&
                                       isfinite(fin(p, q, OCPQP_F_lb, n)[r])) ? flam[cf + r] : 0.0;
                    const double lu = (fin(p, q, OCPQP_F_masku, n)[r] != 0.0 &&
                                       isfinite(fin(p, q, OCPQP_F_ub, n)[r])) ? flam[cf + mo + r] : 0.0;
                    out += ll - lu;
                }
            }
            double g = 0.0;
            for (int r = 0; r < ng; ++r) {
                const double ll = (fin(p, q, OCPQP_F_maskl, n)[nb + r] != 0.0 &&
                                   isfinite(fin(p, q, OCPQP_F_lg, n)[r])) ? flam[cf + nb + r] : 0.0;
                const double lu = (fin(p, q, OCPQP_F_masku, n)[nb + r] != 0.0 &&
                                   isfinite(fin(p, q, OCPQP_F_ug, n)[r])) ? flam[cf + mo + nb + r] : 0.0;
                g = fma(fin(p, q, OCPQP_F_C, n)[r * nx + a], ll - lu, g);
            }
            ctx[a] = out + g;
        }
        __syncthreads();
        const double* Q = fin(p, q, OCPQP_F_Q, n);
        const double* S = fin(p, q, OCPQP_F_S, n);
        const double* qv = fin(p, q, OCPQP_F_q, n);
        const double* A = fin(p, q, OCPQP_F_A, n);
        const double* um = fy + p.o_u[n];
        for (int a = tid; a < nx; a += T) {
            double qx = 0.0, su = 0.0, ap = 0.0;
            for (int c = 0; c < nx; ++c) qx = fma(Q[a * nx + c], xs[m * XM + c], qx);
            for (int c = 0; c < nu; ++c) su = fma(S[c * nx + a], um[c], su);
            for (int c = 0; c < nxn; ++c) ap = fma(A[c * nx + a], pis[c], ap);
            const double v = (((qx + su) + qv[a]) - ctx[a]) + ap;
            if (m >= 1) fpi[p.o_pi[n - 1] + a] = v; else gap[a] = v;
        }
        __syncthreads();
        if (m >= 1)
            for (int a = tid; a < nx; a += T) pis[a] = fpi[p.o_pi[n - 1] + a];
        __syncthreads();
    }
    if (want_gap && tid == 0) {
        // net multiplier of each dropped fixing row, split by sign (condensing.py:414-428)
        const int mo = p.onb[0] + p.ong[0], cf = p.o_c[0];
        for (int j = 0; j < p.nfix; ++j) {
            const double g = gap[p.fix_c[j]];
            if (g >= 0.0) flam[cf + p.fix_row[j]] = g;
            else flam[cf + mo + p.fix_row[j]] = -g;
        }
    }
}

__device__ void expand_terminal(const PcParams& p, int q) {
    const int tid = threadIdx.x, T = blockDim.x;
    const double* sy = p.sy + (long long)q * p.ny_s;
    const double* slam = p.slam + (long long)q * p.nc_s;
    const double* sts = p.st + (long long)q * p.nc_s;
    double* fy = p.fy + (long long)q * p.ny_f;
    double* flam = p.flam + (long long)q * p.nc_f;
    double* ft = p.ft + (long long)q * p.nc_f;
    const int N = p.N, N2 = p.N2;
    const int ncN = 2 * (p.onb[N] + p.ong[N]) + 2 * p.ons[N];
    for (int e = tid; e < ncN; e += T) {
        flam[p.o_c[N] + e] = slam[p.n_c[N2] + e];
        ft[p.o_c[N] + e] = sts[p.n_c[N2] + e];
    }
    for (int j = tid; j < p.ons[N]; j += T) {
        fy[p.nv_f + p.o_s[N] + j] = sy[p.nv_s + p.n_s[N2] + j];
        fy[p.nv_f + p.nst_f + p.o_s[N] + j] = sy[p.nv_s + p.nst_s + p.n_s[N2] + j];
    }
    // boundary states come verbatim from the short-horizon solution (condensing.py:608-610)
    for (int k = 0; k <= N2; ++k) {
        const int n = (k < p.nblk) ? p.blk[k].n0 : N;
        const int nx = p.onx[n];
        for (int a = tid; a < nx; a += T) fy[p.o_x[n] + a] = sy[p.n_x[k] + a];
    }
    for (int a = tid; a < p.onu[N]; a += T) fy[p.o_u[N] + a] = sy[p.n_u[N2] + a];
}

__global__ void __launch_bounds__(256) k_pc_expand(PcParams p) {
    __shared__ int s_item;
    double* ws = p.ws + (long long)blockIdx.x * p.ws_slot;
    const int items = p.B * p.nblk;
    while (true) {
        if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1);
        __syncthreads();
        const int it = s_item;
        __syncthreads();
        if (it >= items) break;
        const int q = it / p.nblk, k = it - q * p.nblk;
        expand_block(p, q, k, ws);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(256) k_pc_expand_terminal(PcParams p) {
    for (int q = blockIdx.x; q < p.B; q += gridDim.x) expand_terminal(p, q);
}

}  // namespace

// ---------------------------------------------------------------------------
// host plan
// ---------------------------------------------------------------------------
struct OcpPcPlan {
    Dims od, nd;
    int N1 = 1, nblk = 0;
    int full = 0;
    std::vector<int> fix_row, fix_c;
    std::vector<int> slk_stage, slk_j;
    int *d_slk_stage = nullptr, *d_slk_j = nullptr, *d_os = nullptr, *d_ns = nullptr;
    int *d_ons = nullptr, *d_nns = nullptr;
    int* d_fix_row = nullptr;
    int* d_fix_c = nullptr;
    std::vector<PcBlockDev> blk;
    std::vector<int> uoff, row_kind, row_stage, row_src, row_aux;
    int nxmax = 1, nvmax = 1, numax = 1, Lmax = 1;
    long long ws_slot = 1;
    int sqrt_cost = 0;         // square-root cost recursion (full condensing)
    int* d_fail = nullptr;
    // device copies of the tables
    bool uploaded = false;
    PcBlockDev* d_blk = nullptr;
    int *d_uoff = nullptr, *d_kind = nullptr, *d_stage = nullptr, *d_src = nullptr, *d_aux = nullptr;
    int *d_onx = nullptr, *d_onu = nullptr, *d_onb = nullptr, *d_ong = nullptr;
    int *d_ou = nullptr, *d_ox = nullptr, *d_opi = nullptr, *d_oc = nullptr;
    int *d_nu = nullptr, *d_nx = nullptr, *d_npi = nullptr, *d_nc = nullptr;
    int *d_oib = nullptr, *d_oidxb = nullptr;
    long long *d_ofoff = nullptr, *d_nfoff = nullptr;
    int* d_counter = nullptr;
    double* d_ws = nullptr;
    int slots = 0;
};

namespace {

template <typename T>
int upload(T** dst, const std::vector<T>& v) {
    const size_t n = std::max<size_t>(1, v.size());
    if (cudaMalloc(dst, sizeof(T) * n) != cudaSuccess) return -1;
    if (!v.empty() && cudaMemcpy(*dst, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice) != cudaSuccess)
        return -1;
    return 0;
}

// Soft rows of one new stage: a row keeps its slack, and the new slacks are
// ordered by new row index (condense's slack_entries sorted by dense row,
// condensing.py:289-300, then partial_condense's idxs re-ordering through the
// box permutation, :523-534).  Fills b.s0 / b.ns_new and the new idxs.
void pc_slacks(OcpPcPlan* P, PcBlockDev& b) {
    const Dims& od = P->od;
    b.s0 = (int)P->slk_stage.size();
    b.ns_new = 0;
    for (int r = 0; r < b.nb_new + b.ng_new; ++r) {
        const int e = b.row0 + r;
        const int i = P->row_stage[e], src = P->row_src[e], n = b.n0 + i;
        for (int j = 0; j < od.ns[n]; ++j)
            if (od.idxs[od.is_off[n] + j] == src) {
                P->slk_stage.push_back(i);
                P->slk_j.push_back(j);
                P->nd.idxs.push_back(r);
                ++b.ns_new;
                break;
            }
    }
}

// workspace per CTA slot; T1 scratch doubles as the (nv x nu) cross-term buffer
void pc_size(OcpPcPlan* P) {
    const long long UM = P->numax, VM = P->nvmax;
    long long XM = P->nxmax;
    while (XM * std::max(XM, UM) < VM * UM) ++XM;
    P->nxmax = (int)XM;
    P->ws_slot = (P->Lmax + 1) * XM * XM + (long long)(P->Lmax + 1) * XM * UM + 2ll * (P->Lmax + 1) * XM +
                 VM * VM + VM + 2ll * XM * VM + XM * std::max(XM, UM) + XM * UM + 64;
    // square-root cost recursion: U, the QR stack, U B, chol(Q)
    if (P->sqrt_cost) P->ws_slot += 4ll * XM * XM + XM * UM + 64;
}

int pc_prepare(OcpPcPlan* P, int items) {
    if (!P->uploaded) {
        int rc = 0;
        rc |= upload(&P->d_blk, P->blk);
        rc |= upload(&P->d_uoff, P->uoff);
        rc |= upload(&P->d_kind, P->row_kind);
        rc |= upload(&P->d_stage, P->row_stage);
        rc |= upload(&P->d_src, P->row_src);
        rc |= upload(&P->d_aux, P->row_aux);
        rc |= upload(&P->d_onx, P->od.nx);
        rc |= upload(&P->d_onu, P->od.nu);
        rc |= upload(&P->d_onb, P->od.nb);
        rc |= upload(&P->d_ong, P->od.ng);
        rc |= upload(&P->d_ou, P->od.u_off);
        rc |= upload(&P->d_ox, P->od.x_off);
        rc |= upload(&P->d_opi, P->od.pi_off);
        rc |= upload(&P->d_oc, P->od.c_off);
        rc |= upload(&P->d_nu, P->nd.u_off);
        rc |= upload(&P->d_nx, P->nd.x_off);
        rc |= upload(&P->d_npi, P->nd.pi_off);
        rc |= upload(&P->d_nc, P->nd.c_off);
        rc |= upload(&P->d_oib, P->od.ib_off);
        rc |= upload(&P->d_oidxb, P->od.idxb);
        rc |= upload(&P->d_ofoff, P->od.foff);
        rc |= upload(&P->d_nfoff, P->nd.foff);
        rc |= upload(&P->d_slk_stage, P->slk_stage);
        rc |= upload(&P->d_slk_j, P->slk_j);
        rc |= upload(&P->d_os, P->od.s_off);
        rc |= upload(&P->d_ns, P->nd.s_off);
        rc |= upload(&P->d_ons, P->od.ns);
        rc |= upload(&P->d_nns, P->nd.ns);
        rc |= upload(&P->d_fix_row, P->fix_row);
        rc |= upload(&P->d_fix_c, P->fix_c);
        if (cudaMalloc(&P->d_counter, sizeof(int)) != cudaSuccess) rc = -1;
        if (rc) return pc_fail(OCPQP_E_CUDA, "partial condensing: table upload failed");
        P->uploaded = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int slots = std::max(1, std::min(items, sms * 4));
    if (slots > P->slots) {
        cudaFree(P->d_ws);
        P->d_ws = nullptr;
        if (cudaMalloc(&P->d_ws, sizeof(double) * P->ws_slot * slots) != cudaSuccess)
            return pc_fail(OCPQP_E_CUDA, "partial condensing: workspace allocation failed");
        P->slots = slots;
    }
    return OCPQP_OK;
}

void pc_fill(const OcpPcPlan* P, PcParams& k, int B) {
    memset(&k, 0, sizeof(k));
    k.B = B; k.nblk = P->nblk; k.N = P->od.N; k.N2 = P->nd.N;
    k.full = P->full; k.nfix = (int)P->fix_row.size();
    k.slk_stage = P->d_slk_stage; k.slk_j = P->d_slk_j;
    k.o_s = P->d_os; k.n_s = P->d_ns; k.ons = P->d_ons; k.nns = P->d_nns;
    k.nv_s = P->nd.nv; k.nv_f = P->od.nv; k.nst_s = P->nd.ns_tot; k.nst_f = P->od.ns_tot;
    k.fix_row = P->d_fix_row; k.fix_c = P->d_fix_c;
    k.nxmax = P->nxmax; k.nvmax = P->nvmax; k.numax = P->numax; k.Lmax = P->Lmax;
    k.blk = P->d_blk; k.uoff = P->d_uoff;
    k.row_kind = P->d_kind; k.row_stage = P->d_stage; k.row_src = P->d_src; k.row_aux = P->d_aux;
    k.onx = P->d_onx; k.onu = P->d_onu; k.onb = P->d_onb; k.ong = P->d_ong;
    k.ofoff = P->d_ofoff; k.nfoff = P->d_nfoff;
    k.o_u = P->d_ou; k.o_x = P->d_ox; k.o_pi = P->d_opi; k.o_c = P->d_oc;
    k.n_u = P->d_nu; k.n_x = P->d_nx; k.n_pi = P->d_npi; k.n_c = P->d_nc;
    k.o_ib = P->d_oib; k.o_idxb = P->d_oidxb;
    k.ws = P->d_ws; k.ws_slot = P->ws_slot; k.counter = P->d_counter;
    k.sqrt_cost = P->sqrt_cost; k.fail = P->d_fail;
    k.ny_s = P->nd.ny; k.ne_s = P->nd.ne; k.nc_s = P->nd.nc;
    k.ny_f = P->od.ny; k.ne_f = P->od.ne; k.nc_f = P->od.nc;
}

}  // namespace

extern "C" {

const char* ocpqp_pc_last_error(void) { return pc_err.c_str(); }

// Block structure of partial_condense(qp, N1) (condensing.py:451-550).  Soft
// rows are not supported by the batched path (OCPQP_E_UNSUPPORTED).
int ocpqp_pc_create(const OcpQpDimC* dim, int32_t N1, OcpPcPlan** out) {
    if (!dim || !out) return pc_fail(OCPQP_E_ARG, "NULL argument");
    *out = nullptr;
    if (N1 < 1) return pc_fail(OCPQP_E_INVALID_DIM, "block size must be >= 1");
    if (dim->N < 1) return pc_fail(OCPQP_E_INVALID_DIM, "horizon must be >= 1 for partial condensing");
    OcpPcPlan* P = new OcpPcPlan();
    Dims& od = P->od;
    od.N = dim->N;
    const int S = od.N + 1;
    od.nx.assign(dim->nx, dim->nx + S); od.nu.assign(dim->nu, dim->nu + S);
    od.nb.assign(dim->nb, dim->nb + S); od.ng.assign(dim->ng, dim->ng + S);
    od.ns.assign(dim->ns, dim->ns + S);
    long long snb = 0, sns = 0;
    for (int n = 0; n < S; ++n) { snb += od.nb[n]; sns += od.ns[n]; }
    od.idxb.assign(dim->idxb, dim->idxb + snb);
    if (sns) od.idxs.assign(dim->idxs, dim->idxs + sns);
    od.finish();
    P->N1 = N1;
    std::vector<int> starts;
    for (int n0 = 0; n0 < od.N; n0 += N1) starts.push_back(n0);
    P->nblk = (int)starts.size();
    Dims& nd = P->nd;
    nd.N = P->nblk;
    for (int k = 0; k < P->nblk; ++k) {
        const int n0 = starts[k], n1 = std::min(n0 + N1, od.N), L = n1 - n0;
        PcBlockDev b{};
        b.n0 = n0; b.L = L; b.nx0 = od.nx[n0];
        b.zx = b.ox = b.nx0;
        b.uoff0 = (int)P->uoff.size();
        int off = b.nx0;
        for (int i = 0; i < L; ++i) {
            const int nu = od.nu[n0 + i];
            P->uoff.push_back(nu ? off : -1);
            off += nu;
            P->nxmax = std::max(P->nxmax, od.nx[n0 + i + 1]);
            P->numax = std::max(P->numax, nu);
        }
        b.nv = off;
        P->nxmax = std::max(P->nxmax, b.nx0);
        P->nvmax = std::max(P->nvmax, b.nv);
        P->Lmax = std::max(P->Lmax, L);
        // condense(keep_x0=True) row routing (condensing.py:251-288): u-box rows and
        // the block's first-stage x-box rows are dense box rows keyed by z index;
        // later x-box rows and all general rows become dense general rows, in
        // stage order (x-box rows of a stage before its general rows)
        struct Box { int z, i, r; };
        struct Gen { int kind, i, r, aux; };
        std::vector<Box> box;
        std::vector<Gen> gen;
        for (int i = 0; i < L; ++i) {
            const int n = n0 + i, nu = od.nu[n];
            for (int r = 0; r < od.nb[n]; ++r) {
                const int kk = od.idxb[od.ib_off[n] + r];
                if (kk < nu) box.push_back({P->uoff[b.uoff0 + i] + kk, i, r});
                else if (i == 0) box.push_back({kk - nu, i, r});
                else gen.push_back({2, i, r, kk - nu});
            }
            for (int g = 0; g < od.ng[n]; ++g) gen.push_back({3, i, od.nb[n] + g, g});
        }
        std::stable_sort(box.begin(), box.end(), [](const Box& a, const Box& c) { return a.z < c.z; });
        // box rows permuted into (u', x') order: new index z < nx0 ? z + nu' : z - nx0
        // (condensing.py:477-480)
        const int nun = b.nv - b.nx0;
        std::vector<std::pair<int, int>> ni;
        for (int j = 0; j < (int)box.size(); ++j) {
            const int z = box[j].z;
            ni.push_back({z < b.nx0 ? z + nun : z - b.nx0, j});
        }
        std::stable_sort(ni.begin(), ni.end(),
                         [](const std::pair<int, int>& a, const std::pair<int, int>& c) { return a.first < c.first; });
        b.row0 = (int)P->row_kind.size();
        b.nb_new = (int)box.size();
        b.ng_new = (int)gen.size();
        for (auto& e : ni) {
            const Box& bx = box[e.second];
            P->row_kind.push_back(bx.z < b.nx0 ? 1 : 0);
            P->row_stage.push_back(bx.i);
            P->row_src.push_back(bx.r);
            P->row_aux.push_back(bx.z);
            nd.idxb.push_back(e.first);
        }
        for (auto& g : gen) {
            P->row_kind.push_back(g.kind);
            P->row_stage.push_back(g.i);
            P->row_src.push_back(g.r);
            P->row_aux.push_back(g.aux);
        }
        pc_slacks(P, b);
        P->blk.push_back(b);
        nd.nx.push_back(b.nx0); nd.nu.push_back(nun); nd.nb.push_back(b.nb_new);
        nd.ng.push_back(b.ng_new); nd.ns.push_back(b.ns_new);
    }
    // the old terminal stage is carried over verbatim
    nd.nx.push_back(od.nx[od.N]); nd.nu.push_back(od.nu[od.N]); nd.nb.push_back(od.nb[od.N]);
    nd.ng.push_back(od.ng[od.N]); nd.ns.push_back(od.ns[od.N]);
    for (int r = 0; r < od.nb[od.N]; ++r) nd.idxb.push_back(od.idxb[od.ib_off[od.N] + r]);
    for (int j = 0; j < od.ns[od.N]; ++j) nd.idxs.push_back(od.idxs[od.is_off[od.N] + j]);
    nd.finish();
    pc_size(P);
    *out = P;
    return OCPQP_OK;
}

// Full condensing, condense(qp, keep_x0) (condensing.py:160-340): one block over
// stages 0..N, terminal included.  With keep_x0 = 0 the stage-0 x rows are
// dropped and x0hat is read from the fixing rows (fix_row[j] fixes component
// fix_comp[j]; the caller detects them from the data, condensing.py:97-118).
// The dense QP comes out as a single-stage OCP-QP: nx = 0, nu = nv, box rows
// keyed and sorted by z, general rows in stage order.
int ocpqp_fc_create(const OcpQpDimC* dim, int32_t keep_x0, int32_t nfix, const int32_t* fix_row,
                    const int32_t* fix_comp, OcpPcPlan** out) {
    if (!dim || !out || (nfix > 0 && (!fix_row || !fix_comp))) return pc_fail(OCPQP_E_ARG, "NULL argument");
    *out = nullptr;
    if (dim->N < 0) return pc_fail(OCPQP_E_INVALID_DIM, "negative horizon");
    OcpPcPlan* P = new OcpPcPlan();
    P->full = 1;
    Dims& od = P->od;
    od.N = dim->N;
    const int N = od.N, S = N + 1;
    od.nx.assign(dim->nx, dim->nx + S); od.nu.assign(dim->nu, dim->nu + S);
    od.nb.assign(dim->nb, dim->nb + S); od.ng.assign(dim->ng, dim->ng + S);
    od.ns.assign(dim->ns, dim->ns + S);
    long long snb = 0, sns = 0;
    for (int n = 0; n < S; ++n) { snb += od.nb[n]; sns += od.ns[n]; }
    od.idxb.assign(dim->idxb, dim->idxb + snb);
    if (sns) od.idxs.assign(dim->idxs, dim->idxs + sns);
    od.finish();
    const int nx0 = od.nx[0];
    if (!keep_x0)
        for (int j = 0; j < od.ns[0]; ++j) {
            const int r = od.idxs[od.is_off[0] + j];
            if (r < od.nb[0] && od.idxb[od.ib_off[0] + r] >= od.nu[0]) {
                delete P;
                return pc_fail(OCPQP_E_CONDENSE, "soft initial-state fixing rows are not supported "
                                                  "with keep_x0=False");
            }
        }
    if (!keep_x0) {
        std::vector<int> seen(nx0, 0);
        for (int j = 0; j < nfix; ++j) {
            if (fix_comp[j] < 0 || fix_comp[j] >= nx0 || fix_row[j] < 0 || fix_row[j] >= od.nb[0]) {
                delete P;
                return pc_fail(OCPQP_E_ARG, "fixing row %d out of range", j);
            }
            seen[fix_comp[j]] = 1;
            P->fix_row.push_back(fix_row[j]);
            P->fix_c.push_back(fix_comp[j]);
        }
        for (int c = 0; c < nx0; ++c)
            if (!seen[c]) {
                delete P;
                return pc_fail(OCPQP_E_CONDENSE, "keep_x0=False requires every initial-state component "
                                                  "fixed by active equal-bound box rows");
            }
    }
    P->nblk = 1;
    PcBlockDev b{};
    b.n0 = 0; b.L = N; b.nx0 = nx0;
    b.zx = keep_x0 ? nx0 : 0;
    b.ox = 0;
    b.uoff0 = 0;
    int off = b.zx;
    for (int n = 0; n <= N; ++n) {
        const int nu = od.nu[n];
        P->uoff.push_back(nu ? off : -1);
        off += nu;
        P->nxmax = std::max(P->nxmax, od.nx[n]);
        P->numax = std::max(P->numax, nu);
    }
    b.nv = off;
    P->nvmax = std::max(1, b.nv);
    P->Lmax = std::max(1, N);
    // routing (condensing.py:251-297): u-box rows and kept-x0 rows are dense box
    // rows keyed by z; x-box rows past stage 0 and all general rows become dense
    // general rows in stage order; stage-0 x rows are dropped with x0
    struct Box { int z, i, r, kind; };
    struct Gen { int kind, i, r, aux; };
    std::vector<Box> box;
    std::vector<Gen> gen;
    for (int n = 0; n <= N; ++n) {
        const int nu = od.nu[n];
        for (int r = 0; r < od.nb[n]; ++r) {
            const int kk = od.idxb[od.ib_off[n] + r];
            if (kk < nu) box.push_back({P->uoff[n] + kk, n, r, 0});
            else if (n == 0 && keep_x0) box.push_back({kk - nu, n, r, 1});
            else if (n == 0) continue;
            else gen.push_back({2, n, r, kk - nu});
        }
        for (int g = 0; g < od.ng[n]; ++g) gen.push_back({3, n, od.nb[n] + g, g});
    }
    std::stable_sort(box.begin(), box.end(), [](const Box& a, const Box& c) { return a.z < c.z; });
    Dims& nd = P->nd;
    nd.N = 0;
    b.row0 = 0;
    b.nb_new = (int)box.size();
    b.ng_new = (int)gen.size();
    for (auto& e : box) {
        P->row_kind.push_back(e.kind);
        P->row_stage.push_back(e.i);
        P->row_src.push_back(e.r);
        P->row_aux.push_back(e.z);
        nd.idxb.push_back(e.z);
    }
    for (auto& g : gen) {
        P->row_kind.push_back(g.kind);
        P->row_stage.push_back(g.i);
        P->row_src.push_back(g.r);
        P->row_aux.push_back(g.aux);
    }
    pc_slacks(P, b);
    P->blk.push_back(b);
    nd.nx.push_back(0); nd.nu.push_back(b.nv); nd.nb.push_back(b.nb_new);
    nd.ng.push_back(b.ng_new); nd.ns.push_back(b.ns_new);
    nd.finish();
    pc_size(P);
    *out = P;
    return OCPQP_OK;
}

int ocpqp_pc_destroy(OcpPcPlan* P) {
    if (!P) return OCPQP_OK;
    cudaFree(P->d_blk); cudaFree(P->d_uoff); cudaFree(P->d_kind); cudaFree(P->d_stage);
    cudaFree(P->d_src); cudaFree(P->d_aux); cudaFree(P->d_onx); cudaFree(P->d_onu);
    cudaFree(P->d_onb); cudaFree(P->d_ong); cudaFree(P->d_ou); cudaFree(P->d_ox);
    cudaFree(P->d_opi); cudaFree(P->d_oc); cudaFree(P->d_nu); cudaFree(P->d_nx);
    cudaFree(P->d_npi); cudaFree(P->d_nc); cudaFree(P->d_oib); cudaFree(P->d_oidxb);
    cudaFree(P->d_ofoff); cudaFree(P->d_nfoff); cudaFree(P->d_counter); cudaFree(P->d_ws); cudaFree(P->d_fail);
    cudaFree(P->d_fix_row); cudaFree(P->d_fix_c);
    cudaFree(P->d_slk_stage); cudaFree(P->d_slk_j); cudaFree(P->d_os); cudaFree(P->d_ns);
    cudaFree(P->d_ons); cudaFree(P->d_nns);
    delete P;
    return OCPQP_OK;
}

// Dimensions of the condensed QP: returns N2 (number of blocks).  When the
// arrays are non-NULL, nx/nu/nb/ng receive N2+1 entries and idxb_out the
// concatenated new idxb (sum of nb).
int ocpqp_pc_dims(const OcpPcPlan* P, int32_t* nx, int32_t* nu, int32_t* nb, int32_t* ng,
                  int32_t* idxb_out) {
    if (!P) return pc_fail(OCPQP_E_ARG, "NULL plan");
    if (nx && nu && nb && ng) {
        for (int k = 0; k <= P->nd.N; ++k) {
            nx[k] = P->nd.nx[k]; nu[k] = P->nd.nu[k]; nb[k] = P->nd.nb[k]; ng[k] = P->nd.ng[k];
        }
    }
    if (idxb_out)
        for (size_t i = 0; i < P->nd.idxb.size(); ++i) idxb_out[i] = P->nd.idxb[i];
    return P->nd.N;
}

// Soft rows of the condensed QP: ns (N2+1 entries) and the concatenated new
// idxs (sum of ns) when non-NULL; returns sum(ns).
int ocpqp_pc_soft(const OcpPcPlan* P, int32_t* ns, int32_t* idxs_out) {
    if (!P) return pc_fail(OCPQP_E_ARG, "NULL plan");
    if (ns)
        for (int k = 0; k <= P->nd.N; ++k) ns[k] = P->nd.ns[k];
    if (idxs_out)
        for (size_t i = 0; i < P->nd.idxs.size(); ++i) idxs_out[i] = P->nd.idxs[i];
    return (int)P->nd.idxs.size();
}

// Batched partial_condense arithmetic: `in` is the packed batch of B QPs
// (device), `out` receives the condensed packed batch (device, every field
// per QP, batch stride = per-QP field length of the condensed layout).
int ocpqp_pc_condense(OcpPcPlan* P, int32_t B, const OcpQpDataC* in, OcpQpDataC* out, void* stream) {
    if (!P || !in || !out) return pc_fail(OCPQP_E_ARG, "NULL argument");
    if (B <= 0) return OCPQP_OK;
    const int items = B * (P->nblk + (P->full ? 0 : 1));
    int rc = pc_prepare(P, items);
    if (rc) return rc;
    PcParams k;
    pc_fill(P, k, B);
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
        k.fin[f] = in->ptr[f]; k.bin[f] = in->batch_stride[f];
        k.fout[f] = (double*)out->ptr[f]; k.bout[f] = out->batch_stride[f];
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(P->d_counter, 0, sizeof(int), st) != cudaSuccess)
        return pc_fail(OCPQP_E_CUDA, "memset");
    if (P->sqrt_cost && cudaMemsetAsync(P->d_fail, 0, sizeof(int), st) != cudaSuccess)
        return pc_fail(OCPQP_E_CUDA, "memset");
    k_pc_condense<<<std::min(P->slots, items), 256, 0, st>>>(k);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return pc_fail(OCPQP_E_CUDA, "k_pc_condense: %s", cudaGetErrorString(e));
    if (P->sqrt_cost) {
        // the square-root recursion can fail numerically (cholesky_factor / qr_cholesky raise
        // in the reference, linalg.py:110-113, 181-184): one word back per call
        int fail = 0;
        if (cudaMemcpyAsync(&fail, P->d_fail, sizeof(int), cudaMemcpyDeviceToHost, st) != cudaSuccess ||
            cudaStreamSynchronize(st) != cudaSuccess)
            return pc_fail(OCPQP_E_CUDA, "square-root condensing: status read failed");
        if (fail) {
            const int q = fail >> 2;
            if ((fail & 3) == 1)
                return pc_fail(OCPQP_E_NOT_PD, "NotPositiveDefinite: stage cost Q of QP %d is not positive definite", q);
            return pc_fail(OCPQP_E_RANK, "RankDeficient: stacked cost factor of QP %d", q);
        }
    }
    return OCPQP_OK;
}

// Cost recursion of full condensing (condense(variant=...), condensing.py:128-157):
// 0 classical, 1 square-root.  Partial plans keep the classical recursion.
int ocpqp_pc_set_variant(OcpPcPlan* P, int32_t square_root) {
    if (!P) return pc_fail(OCPQP_E_ARG, "NULL plan");
    if (square_root && !P->full)
        return pc_fail(OCPQP_E_UNSUPPORTED, "the square-root cost recursion belongs to full condensing");
    if ((square_root != 0) == (P->sqrt_cost != 0)) return OCPQP_OK;
    P->sqrt_cost = square_root ? 1 : 0;
    pc_size(P);
    cudaFree(P->d_ws);       // the slot size changed: reallocated by the next call
    P->d_ws = nullptr;
    P->slots = 0;
    if (P->sqrt_cost && !P->d_fail && cudaMalloc(&P->d_fail, sizeof(int)) != cudaSuccess)
        return pc_fail(OCPQP_E_CUDA, "square-root condensing: allocation failed");
    return OCPQP_OK;
}

// Batched partial_expand (condensing.py:553-619): `short_sol` is the solution
// of the condensed batch, `full_sol` receives the full-horizon solution.
int ocpqp_pc_expand(OcpPcPlan* P, int32_t B, const OcpQpDataC* in, const OcpIterC* short_sol,
                    OcpIterC* full_sol, void* stream) {
    if (!P || !in || !short_sol || !full_sol) return pc_fail(OCPQP_E_ARG, "NULL argument");
    if (B <= 0) return OCPQP_OK;
    const int items = B * P->nblk;
    int rc = pc_prepare(P, items);
    if (rc) return rc;
    PcParams k;
    pc_fill(P, k, B);
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) { k.fin[f] = in->ptr[f]; k.bin[f] = in->batch_stride[f]; }
    k.sy = short_sol->y; k.spi = short_sol->pi; k.slam = short_sol->lam; k.st = short_sol->t;
    k.fy = full_sol->y; k.fpi = full_sol->pi; k.flam = full_sol->lam; k.ft = full_sol->t;
    cudaStream_t st = (cudaStream_t)stream;
    if (cudaMemsetAsync(P->d_counter, 0, sizeof(int), st) != cudaSuccess)
        return pc_fail(OCPQP_E_CUDA, "memset");
    if (cudaMemsetAsync(full_sol->pi, 0, sizeof(double) * (size_t)B * P->od.ne, st) != cudaSuccess)
        return pc_fail(OCPQP_E_CUDA, "memset");
    if (P->full) {
        // dropped fixing rows are not routed: their lam / t start from zero
        if (cudaMemsetAsync(full_sol->lam, 0, sizeof(double) * (size_t)B * P->od.nc, st) != cudaSuccess ||
            cudaMemsetAsync(full_sol->t, 0, sizeof(double) * (size_t)B * P->od.nc, st) != cudaSuccess)
            return pc_fail(OCPQP_E_CUDA, "memset");
    }
    k_pc_expand<<<std::min(P->slots, items), 256, 0, st>>>(k);
    if (!P->full) k_pc_expand_terminal<<<std::min(B, 1024), 256, 0, st>>>(k);
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return pc_fail(OCPQP_E_CUDA, "k_pc_expand: %s", cudaGetErrorString(e));
    return OCPQP_OK;
}

}  // extern "C"
