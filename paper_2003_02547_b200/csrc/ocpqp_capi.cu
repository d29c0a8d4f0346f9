// C ABI of the batched OCP-QP solver (include/ocpqp_b200.h): plan creation,
// layout tables, workspace placement (shared memory vs per-slot global), and
// the device- and host-buffer solve entry points.
#include <cuda_runtime.h>
#include <math.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <string>
#include <vector>

#include "ocpqp_internal.h"

using namespace ocpqp;

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

int cuda_fail(cudaError_t e, const char* what) {
    return fail(OCPQP_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

#define CUDA_TRY(expr)                                   \
    do {                                                 \
        cudaError_t _e = (expr);                         \
        if (_e != cudaSuccess) return cuda_fail(_e, #expr); \
    } while (0)

// Host copy of the structure; everything derived from OcpQpDimC.
struct Layout {
    int N = 0;
    std::vector<int> nx, nu, nb, ng, ns, idxb, idxs;
    std::vector<StageInfo> st;
    int ny = 0, ne = 0, nc = 0, nv = 0, ns_tot = 0, msum = 0;
    int nw_max = 0, nx_max = 0, nu_max = 0, m_max = 0, nc_max = 0, ns_max = 0;
    long long flen[OCPQP_NUM_FIELDS] = {0};
    std::vector<int> var_box, row_slack;
    long long ws_size[WS_NUM] = {0};
    int box_ident = 1;        // every stage's idxb is 0, 1, ..., nb - 1
};

long long field_stage_size(int f, const Layout& L, int n) {
    const int nx = L.nx[n], nu = L.nu[n], nb = L.nb[n], ng = L.ng[n], ns = L.ns[n];
    const int nxn = n < L.N ? L.nx[n + 1] : 0;
    switch (f) {
        case OCPQP_F_A: return n < L.N ? (long long)nxn * nx : 0;
        case OCPQP_F_B: return n < L.N ? (long long)nxn * nu : 0;
        case OCPQP_F_b: return n < L.N ? nxn : 0;
        case OCPQP_F_Q: return (long long)nx * nx;
        case OCPQP_F_S: return (long long)nu * nx;
        case OCPQP_F_R: return (long long)nu * nu;
        case OCPQP_F_q: return nx;
        case OCPQP_F_r: return nu;
        case OCPQP_F_lb: case OCPQP_F_ub: return nb;
        case OCPQP_F_C: return (long long)ng * nx;
        case OCPQP_F_D: return (long long)ng * nu;
        case OCPQP_F_lg: case OCPQP_F_ug: return ng;
        case OCPQP_F_Zl: case OCPQP_F_Zu: case OCPQP_F_zl: case OCPQP_F_zu:
        case OCPQP_F_sl_lb: case OCPQP_F_su_lb: return ns;
        case OCPQP_F_maskl: case OCPQP_F_masku: return nb + ng;
    }
    return 0;
}

// Validation mirrors OcpQpDim.__init__ (qp_data.py:82-111) and the index-set
// checks of validate() (qp_data.py:528-533).
int build_layout(const OcpQpDimC* d, Layout& L) {
    if (!d) return fail(OCPQP_E_ARG, "dim is NULL");
    if (d->N < 0) return fail(OCPQP_E_INVALID_DIM, "horizon N must be >= 0");
    if (!d->nx || !d->nu || !d->nb || !d->ng || !d->ns)
        return fail(OCPQP_E_ARG, "dimension arrays must not be NULL");
    L.N = d->N;
    const int S = d->N + 1;
    L.nx.assign(d->nx, d->nx + S);
    L.nu.assign(d->nu, d->nu + S);
    L.nb.assign(d->nb, d->nb + S);
    L.ng.assign(d->ng, d->ng + S);
    L.ns.assign(d->ns, d->ns + S);
    long long sum_nb = 0, sum_ns = 0;
    for (int n = 0; n < S; ++n) {
        if (L.nx[n] < 0 || L.nu[n] < 0 || L.nb[n] < 0 || L.ng[n] < 0 || L.ns[n] < 0)
            return fail(OCPQP_E_INVALID_DIM, "stage %d: dimensions must be nonnegative", n);
        if (L.nb[n] > L.nu[n] + L.nx[n])
            return fail(OCPQP_E_INVALID_DIM, "stage %d: nb = %d exceeds nu + nx = %d", n, L.nb[n],
                        L.nu[n] + L.nx[n]);
        if (L.ns[n] > L.nb[n] + L.ng[n])
            return fail(OCPQP_E_INVALID_DIM, "stage %d: ns = %d exceeds nb + ng = %d", n, L.ns[n],
                        L.nb[n] + L.ng[n]);
        sum_nb += L.nb[n];
        sum_ns += L.ns[n];
    }
    if (sum_nb && !d->idxb) return fail(OCPQP_E_ARG, "idxb is NULL");
    if (sum_ns && !d->idxs) return fail(OCPQP_E_ARG, "idxs is NULL");
    L.idxb.assign(d->idxb ? d->idxb : nullptr, d->idxb ? d->idxb + sum_nb : nullptr);
    L.idxs.assign(d->idxs ? d->idxs : nullptr, d->idxs ? d->idxs + sum_ns : nullptr);
    L.st.resize(S);
    int v = 0, s = 0, c = 0, p = 0, ib = 0, is = 0, mo = 0;
    int Po = 0, Ko = 0, Lo = 0, pvo = 0, kfo = 0;
    long long foff[OCPQP_NUM_FIELDS] = {0};
    long long t1 = 0;
    for (int n = 0; n < S; ++n) {
        StageInfo& si = L.st[n];
        memset(&si, 0, sizeof(si));
        si.nx = L.nx[n]; si.nu = L.nu[n]; si.nb = L.nb[n]; si.ng = L.ng[n]; si.ns = L.ns[n];
        si.nxn = n < L.N ? L.nx[n + 1] : 0;
        si.nw = si.nu + si.nx;
        si.m = si.nb + si.ng;
        si.nc = 2 * si.m + 2 * si.ns;
        si.u_off = v; si.x_off = v + si.nu;
        si.pi_off = p;
        si.c_off = c; si.s_off = s; si.ib_off = ib; si.is_off = is; si.m_off = mo;
        for (int i = 0; i < si.nb; ++i) {
            const int k = L.idxb[ib + i];
            if (k < 0 || k >= si.nw)
                return fail(OCPQP_E_DIMENSION, "stage %d: idxb entries must lie in [0, %d)", n, si.nw);
            if (i > 0 && k <= L.idxb[ib + i - 1])
                return fail(OCPQP_E_DIMENSION, "stage %d: idxb entries must be strictly increasing", n);
        }
        for (int j = 0; j < si.ns; ++j) {
            const int k = L.idxs[is + j];
            if (k < 0 || k >= si.m)
                return fail(OCPQP_E_DIMENSION, "stage %d: idxs entries must lie in [0, %d)", n, si.m);
            if (j > 0 && k <= L.idxs[is + j - 1])
                return fail(OCPQP_E_DIMENSION, "stage %d: idxs entries must be strictly increasing", n);
        }
        for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
            si.foff[f] = (int)foff[f];
            foff[f] += field_stage_size(f, L, n);
        }
        si.P_off = Po; Po += si.nx * si.nx;
        si.K_off = Ko; Ko += si.nu * si.nx;
        si.L_off = Lo; Lo += si.nu * si.nu;
        si.pv_off = pvo; pvo += si.nx;
        si.kff_off = kfo; kfo += si.nu;
        v += si.nw; s += si.ns; c += si.nc; ib += si.nb; is += si.ns; mo += si.m;
        if (n < L.N) p += si.nxn;
        L.nw_max = std::max(L.nw_max, si.nw);
        L.nx_max = std::max(L.nx_max, si.nx);
        L.nu_max = std::max(L.nu_max, si.nu);
        L.m_max = std::max(L.m_max, si.m);
        L.nc_max = std::max(L.nc_max, si.nc);
        L.ns_max = std::max(L.ns_max, si.ns);
        t1 = std::max(t1, std::max((long long)si.nxn * si.nw, (long long)si.nx * si.nx));
    }
    L.nv = v; L.ns_tot = s; L.ny = v + 2 * s; L.ne = p; L.nc = c; L.msum = mo;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) L.flen[f] = foff[f];
    L.var_box.assign(std::max(1, L.nv), -1);
    L.row_slack.assign(std::max(1, L.msum), -1);
    for (int n = 0; n < S; ++n) {
        const StageInfo& si = L.st[n];
        for (int i = 0; i < si.nb; ++i) {
            L.var_box[si.u_off + L.idxb[si.ib_off + i]] = i;
            if (L.idxb[si.ib_off + i] != i) L.box_ident = 0;
        }
        for (int j = 0; j < si.ns; ++j) L.row_slack[si.m_off + L.idxs[si.is_off + j]] = j;
    }
    long long* w = L.ws_size;
    w[WS_RG] = L.ny; w[WS_RB] = L.ne; w[WS_RD] = L.nc; w[WS_DVEC] = L.nc; w[WS_ACT] = L.nc;
    w[WS_AFF_Y] = w[WS_DIR_Y] = L.ny;
    w[WS_AFF_PI] = w[WS_DIR_PI] = L.ne;
    w[WS_AFF_LAM] = w[WS_AFF_T] = w[WS_DIR_LAM] = w[WS_DIR_T] = L.nc;
    w[WS_GAM] = L.nc; w[WS_COEF] = L.msum; w[WS_DL] = w[WS_DU] = L.ns_tot;
    w[WS_WALL] = L.nc; w[WS_RTSL] = w[WS_RTSU] = L.ns_tot;
    w[WS_CROW] = L.msum; w[WS_ROWV] = L.msum; w[WS_RHAT] = L.nv;
    w[WS_P] = Po; w[WS_K] = Ko; w[WS_L] = Lo; w[WS_LP0] = (long long)L.nx[0] * L.nx[0];
    w[WS_PV] = pvo; w[WS_KFF] = kfo;
    w[WS_G] = (long long)L.nw_max * L.nw_max;
    w[WS_T1] = t1;
    w[WS_VEC] = L.nw_max + L.nx_max + std::max(L.nu_max, L.nx_max);
    w[WS_IY] = L.ny; w[WS_IPI] = L.ne; w[WS_ILAM] = L.nc; w[WS_IT] = L.nc;
    w[WS_RINV] = kfo + L.nx[0];   // sum nu + nx0
    w[WS_TINV] = L.nc;
    // extended workspace (modes beyond speed)
    w[WS_LPS] = Po; w[WS_HASLP] = S; w[WS_MST] = (long long)L.nw_max * L.nw_max;
    w[WS_QR] = (long long)(L.nw_max + L.nx_max) * L.nw_max + (long long)L.nx_max * L.nx_max;
    w[WS_RMD] = L.nc; w[WS_GF] = L.ny; w[WS_BF] = L.ne;
    w[WS_RFY] = w[WS_BY] = L.ny; w[WS_RFPI] = w[WS_BPI] = L.ne;
    w[WS_RFLAM] = w[WS_RFT] = w[WS_BLAM] = w[WS_BT] = L.nc;
    w[WS_ZT] = L.ne;
    w[WS_RHD] = L.nc;
    return OCPQP_OK;
}

inline long long align2(long long x) { return (x + 1) & ~1ll; }

}  // namespace

namespace ocpqp {
void set_last_error(const char* msg) { g_last_error = msg; }
}  // namespace ocpqp

struct OcpPlan {
    Layout L;
    int B = 0;
    int device = 0;
    int num_sms = 0;
    int threads = 32;
    int slots = 1;
    int grid = 1;
    int team_stride = 0;
    size_t smem_bytes = 0;
    unsigned long long smem_mask = 0;
    int smem_off[WS_NUM] = {0};
    // shaped fast path (ocpqp_fast.cu)
    bool fast = false;
    FastShape shape{0, 0, 0, 0};
    int NB = 0, NBN = 0, NGN = 0;
    int stage_smem = 0;          // offset (doubles) of the per-stage scratch
    double* d_defaults = nullptr;  // zeros | ones | -inf | +inf, each max_flen long
    long long* dbg = nullptr;      // optional phase counters (ocpqp_debug_phases)
    long long max_flen = 1;
    int ws_off[WS_NUM] = {0};
    long long ws_slot = 0;
    // device structure tables
    StageInfo* d_st = nullptr;
    int* d_idxb = nullptr;
    int* d_idxs = nullptr;
    int* d_var_box = nullptr;
    int* d_row_slack = nullptr;
    int* d_counter = nullptr;
    // dispatch hint (ocpqp_plan_dispatch_hint): previous iteration counts, the QP order
    // derived from them, list cursors + CTAs per SM
    int* d_prev_iters = nullptr;
    int* d_order = nullptr;
    int* d_hint_ctr = nullptr;
    bool hint_on = false, hint_valid = false;
    int* d_sinv = nullptr;       // stage-invariance mask of the broadcast fields (team kernel)
    double* d_ba = nullptr;      // packed [B A] of every stage (team kernel)
    int* d_esc = nullptr;        // [1 + B]: count, QPs the team kernel leaves to the generic one
    long long* d_esc_meta = nullptr;  // [B, 3]: where each escaped QP resumes
    // generic-kernel shared-memory placement for the modes beyond speed on a
    // shaped-kernel plan (computed on first use)
    bool gen_placed = false;
    unsigned long long gen_mask = 0;
    int gen_off[WS_NUM] = {0};
    size_t gen_bytes = 0;
    long long ba_cap = 0;        // doubles allocated at d_ba
    double* d_ws = nullptr;
    double* d_ws2 = nullptr;     // extended workspace (allocated on the first non-speed solve)
    long long ws2_slot = 0;
    // host-path device buffers (allocated on first use)
    double* h_field[OCPQP_NUM_FIELDS] = {nullptr};
    long long h_field_len[OCPQP_NUM_FIELDS] = {0};
    double *hy = nullptr, *hpi = nullptr, *hlam = nullptr, *ht = nullptr;
    int32_t *hstatus = nullptr, *hiters = nullptr;
    double* hres = nullptr;
    long long* hflops = nullptr;
    double* htrace = nullptr;
    int htrace_iters = 0;
};

namespace {

// Workspace placement: the hottest buffers go to shared memory up to a
// per-CTA budget chosen so that enough CTAs stay resident per SM.
void place_workspace(OcpPlan* P) {
    const Layout& L = P->L;
    const char* env = getenv("OCPQP_THREADS");
    int threads;
    if (env && atoi(env) > 0) {
        threads = atoi(env);
    } else if (L.nw_max <= 12) {
        threads = 32;
    } else if (L.nw_max <= 24) {
        threads = 64;
    } else if (L.nw_max <= 48) {
        threads = 128;
    } else {
        threads = 256;
    }
    threads = std::min(512, std::max(32, (threads + 31) / 32 * 32));
    P->threads = threads;
    long long off = 0;
    for (int b = 0; b < WS_EXT0; ++b) {
        P->ws_off[b] = (int)off;
        off += align2(L.ws_size[b]);
    }
    P->ws_slot = std::max(2ll, off);

    int tgt = std::max(1, 768 / threads);
    const int per_sm_need = (P->B + P->num_sms - 1) / std::max(1, P->num_sms);
    tgt = std::max(1, std::min(tgt, per_sm_need));
    const char* envs = getenv("OCPQP_SMEM_KB");
    long long budget;
    if (envs) {
        budget = (long long)atoi(envs) * 1024;
    } else {
        budget = (228ll * 1024) / tgt - 2048;
        budget = std::min(budget, 227ll * 1024 - 1024);
    }
    const int prio[] = {WS_T1, WS_G, WS_VEC, WS_ACT, WS_DVEC, WS_GAM, WS_WALL, WS_COEF,
                        WS_CROW, WS_ROWV, WS_RHAT, WS_P, WS_K, WS_L, WS_LP0, WS_PV, WS_KFF,
                        WS_RG, WS_RB, WS_RD, WS_DIR_LAM, WS_DIR_T, WS_AFF_LAM, WS_AFF_T,
                        WS_DIR_Y, WS_DIR_PI, WS_AFF_Y, WS_AFF_PI, WS_DL, WS_DU, WS_RTSL, WS_RTSU};
    long long used = 0;
    P->smem_mask = 0;
    for (int b : prio) {
        const long long sz = align2(L.ws_size[b]) * 8;
        if (sz == 0) continue;
        if (used + sz <= budget) {
            P->smem_mask |= 1ull << b;
            P->smem_off[b] = (int)(used / 8);
            used += sz;
        }
    }
    P->smem_bytes = (size_t)used;
}

void fill_kparams(const OcpPlan* P, KParams& k, const OcpQpDataC* data, bool use_smem) {
    const Layout& L = P->L;
    memset(&k, 0, sizeof(k));
    k.N = L.N; k.B = P->B;
    k.ny = L.ny; k.ne = L.ne; k.nc = L.nc; k.nv = L.nv; k.ns_tot = L.ns_tot; k.msum = L.msum;
    k.nw_max = L.nw_max; k.nx_max = L.nx_max; k.nu_max = L.nu_max; k.m_max = L.m_max;
    k.nc_max = L.nc_max; k.ns_max = L.ns_max;
    k.st = P->d_st; k.idxb = P->d_idxb; k.idxs = P->d_idxs;
    k.var_box = P->d_var_box; k.row_slack = P->d_row_slack;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
        const bool present = data && data->ptr[f] && L.flen[f] > 0;
        k.f[f] = present ? data->ptr[f] : nullptr;
        k.bs[f] = present ? data->batch_stride[f] : 0;
    }
    k.ws = P->d_ws; k.ws_slot = P->ws_slot;
    k.ws2 = P->d_ws2; k.ws2_slot = P->ws2_slot;
    for (int b = 0; b < WS_NUM; ++b) { k.ws_off[b] = P->ws_off[b]; k.smem_off[b] = P->smem_off[b]; }
    k.smem_mask = use_smem ? P->smem_mask : 0ull;
    k.counter = P->d_counter;
    k.NB = P->NB; k.NBN = P->NBN; k.NGN = P->NGN;
    k.box_ident = L.box_ident;
    k.stage_smem = P->stage_smem;
    k.team_stride = P->team_stride;
    k.dbg = P->dbg;
}

// The shaped kernel reads every field unconditionally: absent fields point at
// the plan's default rows (zeros, ones for masks, -inf / +inf for bounds).
void fill_defaults(const OcpPlan* P, KParams& k) {
    const long long L = P->max_flen;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
        if (k.f[f]) continue;
        int which = 0;
        if (f == OCPQP_F_maskl || f == OCPQP_F_masku) which = 1;
        else if (f == OCPQP_F_lb || f == OCPQP_F_lg) which = 2;
        else if (f == OCPQP_F_ub || f == OCPQP_F_ug) which = 3;
        k.f[f] = P->d_defaults + which * L;
        k.bs[f] = 0;
    }
}

// Shaped-kernel eligibility: uniform stages 0..N-1 (nx, nu >= 1, nb, ng),
// terminal stage with nu = 0, nx equal, nb <= nx, ng <= NG; no soft rows.
// Prefers the row kernel (NX <= 32, full box rows) over the team kernel.
// Environment overrides: OCPQP_GENERIC=1, OCPQP_KIND=0|1, OCPQP_TEAM, OCPQP_WPB.
bool detect_fast(OcpPlan* P) {
    const Layout& L = P->L;
    const char* gen = getenv("OCPQP_GENERIC");
    if (gen && atoi(gen)) return false;
    const int N = L.N;
    if (N < 1 || L.ns_tot != 0) return false;
    const int NX = L.nx[0], NU = L.nu[0], NB = L.nb[0], NG = L.ng[0];
    if (NU < 1 || NX < 1) return false;
    for (int n = 0; n < N; ++n)
        if (L.nx[n] != NX || L.nu[n] != NU || L.nb[n] != NB || L.ng[n] != NG) return false;
    if (L.nx[N] != NX || L.nu[N] != 0 || L.ng[N] > NG || L.nb[N] > NX) return false;
    const char* envk = getenv("OCPQP_KIND");
    const char* envt = getenv("OCPQP_TEAM");
    const char* envw = getenv("OCPQP_WPB");
    const int want_kind = envk ? atoi(envk) : -1;
    FastShape pick{-1, 0, 0, 0, 0, 0, 0};
    // row kernel: only on request (measured slower than the team kernel on configs 1-4)
    if (want_kind == 1 && L.box_ident) {   // the row kernel maps box row i to variable i
        const int gdef = (NX <= 8 && NU <= 8) ? 8 : (NX <= 16 && NU <= 16) ? 16 : 32;
        const int g = envt && want_kind == 1 ? atoi(envt) : gdef;
        const int wpbs[] = {envw ? atoi(envw) : 1, 1, 2, 4};
        for (int w : wpbs) {
            FastShape s{1, NX, NU, NG, NB, g, w};
            if (fast_supported(s)) { pick = s; break; }
        }
    }
    if (pick.kind < 0 && want_kind != 1) {
        int team = 0;
        if (envt && atoi(envt) > 0) {
            team = atoi(envt);
            if (!fast_supported(FastShape{0, NX, NU, NG, NB, team, 1})) team = 0;
        } else {
            const int cands[] = {32, 64, 128, 256};
            int pref = NX + NU <= 32 ? 64 : NX + NU <= 48 ? 128 : 256;
            if (fast_supported(FastShape{0, NX, NU, NG, NB, pref, 1})) team = pref;
            for (int c : cands)
                if (!team && fast_supported(FastShape{0, NX, NU, NG, NB, c, 1})) team = c;
        }
        if (team) {
            pick = FastShape{0, NX, NU, NG, NB, team, 1};
            // the variant with the factor store at fixed shared-memory offsets
            // (Shape<..., SM=1>) is used when instantiated and requested;
            // measured no faster than generic addressing on config 1
            FastShape sm = pick;
            sm.sm = 1;
            const char* envm = getenv("OCPQP_SM");
            if (envm && atoi(envm) == 1 && fast_supported(sm)) pick = sm;
        }
    }
    if (pick.kind < 0) return false;
    P->fast = true;
    P->shape = pick;
    P->NB = NB; P->NBN = L.nb[N]; P->NGN = L.ng[N];
    return true;
}

// Placement for the shaped kernels: each team (a CTA for kind 0) gets a
// shared-memory region = [hottest per-QP buffers while they fit | stage tile].
void place_fast(OcpPlan* P, long long budget_per_cta) {
    const Layout& L = P->L;
    const int teams = fast_teams_per_cta(P->shape);
    P->threads = P->shape.kind == 1 ? 32 * P->shape.wpb : P->shape.team;
    long long off = 0;
    for (int b = 0; b < WS_EXT0; ++b) {
        P->ws_off[b] = (int)off;
        off += align2(L.ws_size[b]);
    }
    P->ws_slot = std::max(2ll, off);
    const long long tile = align2(fast_stage_smem_doubles(P->shape)) * 8;
    long long budget = budget_per_cta / teams - tile;
    // team kernel: the factor store and the per-stage vectors read inside the
    // sequential sweeps first, then the slot vectors of the parallel passes
    static const int prio0[] = {WS_L, WS_RINV, WS_K, WS_KFF, WS_PV, WS_LP0, WS_P, WS_RB, WS_RHAT,
                                WS_DIR_Y, WS_DIR_PI, WS_ILAM, WS_IT, WS_DVEC, WS_TINV, WS_GAM,
                                WS_WALL, WS_RD, WS_DIR_LAM, WS_DIR_T, WS_AFF_LAM, WS_AFF_T, WS_IY,
                                WS_IPI, WS_CROW, WS_ROWV, WS_COEF, WS_RG};
    static const int prio1[] = {WS_DVEC, WS_ILAM, WS_IT, WS_GAM, WS_RD, WS_WALL, WS_DIR_LAM, WS_DIR_T,
                                WS_AFF_LAM, WS_AFF_T, WS_IY, WS_DIR_Y, WS_RG, WS_IPI, WS_DIR_PI, WS_RB,
                                WS_CROW, WS_COEF, WS_TINV, WS_RINV, WS_L, WS_K, WS_KFF, WS_PV, WS_LP0,
                                WS_P};
    const int* prio = P->shape.kind == 1 ? prio1 : prio0;
    const int np = P->shape.kind == 1 ? (int)(sizeof(prio1) / sizeof(int)) : (int)(sizeof(prio0) / sizeof(int));
    long long used = 0;
    P->smem_mask = 0;
    // experiments: OCPQP_NOSMEM = bitmask of workspace buffers kept in global memory
    const char* envx = getenv("OCPQP_NOSMEM");
    const unsigned long long nosmem = envx ? strtoull(envx, nullptr, 0) : 0ull;
    for (int i = 0; i < np; ++i) {
        const int b = prio[i];
        long long words = L.ws_size[b];
        // the team kernel stores P packed (lower triangle) in its first part
        if (b == WS_P && P->shape.kind == 0 && OCPQP_PPACK && P->shape.nx >= 16)
            words = (long long)(L.N + 1) * P->shape.nx * (P->shape.nx + 1) / 2;
        const long long bytes = align2(words) * 8;
        if (bytes == 0 || ((nosmem >> b) & 1ull)) continue;
        if (used + bytes <= budget) {
            P->smem_mask |= 1ull << b;
            P->smem_off[b] = (int)(used / 8);
            used += bytes;
        }
    }
    // A placement that holds only a small part of the per-QP workspace costs
    // more L1 capacity (the shared-memory carve-out) than it saves: measured on
    // configs 2 / 3 / 4 (5 % or less of the workspace placed) leaving everything
    // to the L1 is 5-9 % faster; config 1 (45 % placed) is 10 % slower that way.
    const char* envp = getenv("OCPQP_PLACE");
    const bool force = envp && atoi(envp) == 1, never = envp && atoi(envp) == 0;
    // BIG shapes stream their per-stage operands from global memory by TMA
    // (the copy engine reads global memory only): no placement
    if (never || fast_big(P->shape) || (!force && used * 5 < P->ws_slot * 8)) {
        P->smem_mask = 0;
        used = 0;
    }
    P->stage_smem = (int)(used / 8);
    P->team_stride = (int)((used + tile) / 8);
    P->smem_bytes = (size_t)(used + tile) * teams;
}

// Plan the shaped kernel: choose a shared-memory budget so that the CTAs the
// batch needs can be resident, check occupancy, and size the slot count.
bool plan_fast_once(OcpPlan* P, int* occ_out);

// Buffers the SM variant of the team kernel addresses at fixed shared offsets.
static const int kSmRequired[] = {WS_P, WS_K, WS_L, WS_LP0, WS_RINV, WS_PV, WS_KFF, WS_RB, WS_RHAT};

bool plan_fast(OcpPlan* P, int* occ_out) {
    if (P->shape.kind == 0 && P->shape.sm) {
        if (plan_fast_once(P, occ_out)) {
            bool ok = true;
            for (int b : kSmRequired)
                if (P->L.ws_size[b] > 0 && !((P->smem_mask >> b) & 1ull)) ok = false;
            if (ok) return true;
        }
        P->shape.sm = 0;
    }
    return plan_fast_once(P, occ_out);
}

bool plan_fast_once(OcpPlan* P, int* occ_out) {
    const int teams = fast_teams_per_cta(P->shape);
    const int ctas_needed = (P->B + teams - 1) / teams;
    int per_sm = std::max(1, (ctas_needed + P->num_sms - 1) / P->num_sms);
    // never plan for more CTAs per SM than registers / threads allow
    const int tile_bytes = (int)(align2(fast_stage_smem_doubles(P->shape)) * 8) * teams;
    const int occ_max = fast_occupancy(P->shape, (size_t)tile_bytes);
    if (occ_max > 0) per_sm = std::min(per_sm, occ_max);
    const char* envs = getenv("OCPQP_SMEM_KB");
    long long budget;
    if (envs) budget = (long long)atoi(envs) * 1024;
    else budget = std::min((228ll * 1024) / std::min(per_sm, 32) - 2048, 227ll * 1024 - 2048);
    budget = std::max(budget, 0ll);
    for (int attempt = 0; attempt < 8; ++attempt) {
        place_fast(P, budget);
        const int occ = fast_occupancy(P->shape, P->smem_bytes);
        if (occ > 0) { *occ_out = occ; return true; }
        budget /= 2;
    }
    return false;
}

int check_arg(const OcpIpmArgC* a) {
    if (!a) return fail(OCPQP_E_ARG, "arg is NULL");
    if (!(a->tol_stat > 0) || !(a->tol_eq > 0) || !(a->tol_ineq > 0) || !(a->tol_comp > 0))
        return fail(OCPQP_E_ARG, "tolerances must be > 0");
    if (!(a->alpha_min > 0.0 && a->alpha_min < 1.0))
        return fail(OCPQP_E_ARG, "alpha_min must lie in (0, 1)");
    if (a->lam_min < 0.0 || a->t_min < 0.0) return fail(OCPQP_E_ARG, "lam_min and t_min must be >= 0");
    if (a->warm_start < 0 || a->warm_start > 2) return fail(OCPQP_E_ARG, "unknown warm_start");
    if (a->iter_max < 0) return fail(OCPQP_E_ARG, "iter_max must be >= 0");
    if (a->riccati_variant != 0 && a->riccati_variant != 1)
        return fail(OCPQP_E_ARG, "unknown riccati_variant");
    if (a->itref_corr_max < 0 || a->itref_pred_max < 0)
        return fail(OCPQP_E_ARG, "refinement step counts must be >= 0");
    // the reference's loop reads res.r_g etc. without per-iteration residuals
    // unless the absolute formulation supplies the rhs (solver.py:191-216)
    if (!a->comp_res_pred && !a->abs_form)
        return fail(OCPQP_E_UNSUPPORTED, "comp_res_pred=False needs abs_form=True");
    return OCPQP_OK;
}

// Shared-memory placement of the generic kernel on a shaped-kernel plan (the
// plan's own placement belongs to the shaped kernel): the generic priority
// order, a budget that keeps the plan's slots resident, checked by occupancy.
void place_generic_on_fast(OcpPlan* P) {
    if (P->gen_placed) return;
    P->gen_placed = true;
    const Layout& L = P->L;
    const int per_sm = std::max(1, (P->slots + P->num_sms - 1) / std::max(1, P->num_sms));
    long long budget = std::min((228ll * 1024) / per_sm - 2048, 227ll * 1024 - 1024);
    const int prio[] = {WS_T1, WS_G, WS_VEC, WS_ACT, WS_DVEC, WS_GAM, WS_WALL, WS_COEF,
                        WS_CROW, WS_ROWV, WS_RHAT, WS_P, WS_K, WS_L, WS_LP0, WS_PV, WS_KFF,
                        WS_RG, WS_RB, WS_RD, WS_DIR_LAM, WS_DIR_T, WS_AFF_LAM, WS_AFF_T,
                        WS_DIR_Y, WS_DIR_PI, WS_AFF_Y, WS_AFF_PI, WS_DL, WS_DU, WS_RTSL, WS_RTSU};
    for (int attempt = 0; attempt < 6 && budget > 0; ++attempt, budget /= 2) {
        long long used = 0;
        unsigned long long mask = 0;
        int off[WS_NUM] = {0};
        for (int b : prio) {
            const long long sz = align2(L.ws_size[b]) * 8;
            if (sz == 0 || used + sz > budget) continue;
            mask |= 1ull << b;
            off[b] = (int)(used / 8);
            used += sz;
        }
        if (ipm_occupancy(P->threads, (size_t)used) >= per_sm || attempt == 5) {
            if (ipm_occupancy(P->threads, (size_t)used) == 0) return;  // keep global memory
            P->gen_mask = mask;
            memcpy(P->gen_off, off, sizeof(off));
            P->gen_bytes = (size_t)used;
            return;
        }
    }
}

// The team kernel runs the classical-Riccati delta-form loop with optional
// refinement of the combined direction (speed, balance); the QR rungs of the
// balance ladder are left to the generic kernel per QP (escape list).
bool team_supports(const OcpIpmArgC* a, int nw, int nx) {
    // delta form with residuals every iteration, or the speed_abs combination
    // (absolute form, residuals only at exit, no refinement / QR)
    const bool delta = !a->abs_form && a->comp_res_pred;
    const bool abs_speed = a->abs_form && !a->comp_res_pred && a->itref_corr_max <= 0 &&
                           !a->use_qr_fallback;
    // square-root variant: warp Cholesky of the whole stage block (nw <= 32)
    const bool variant_ok = a->riccati_variant == 0 || (a->riccati_variant == 1 && nw <= 32);
    // robust mode's QR stage: the stacked factor (nw + nx rows) by one warp; soft-iterate
    // refinement of the ladder as in balance
    const bool qr_ok = !a->use_qr_always || (delta && nw + nx <= 32 && a->riccati_variant == 0);
    return (delta || abs_speed) && qr_ok && variant_ok && a->itref_pred_max <= 0;
}

// modes beyond the classical speed loop need the extended workspace
bool needs_ext(const OcpIpmArgC* a) {
    return a->itref_corr_max > 0 || a->itref_pred_max > 0 || a->use_qr_fallback ||
           a->use_qr_always || a->riccati_variant != 0 || a->abs_form || !a->comp_res_pred;
}

int ensure_ext(OcpPlan* P) {
    if (P->d_ws2) return OCPQP_OK;
    long long off = 0;
    for (int b = WS_EXT0; b < WS_NUM; ++b) {
        P->ws_off[b] = (int)off;
        off += align2(P->L.ws_size[b]);
    }
    P->ws2_slot = std::max(2ll, off);
    CUDA_TRY(cudaMalloc(&P->d_ws2, sizeof(double) * (size_t)P->ws2_slot * P->slots));
    return OCPQP_OK;
}

template <typename T>
int ensure(T** p, long long n) {
    if (*p) return OCPQP_OK;
    CUDA_TRY(cudaMalloc((void**)p, sizeof(T) * (size_t)std::max(1ll, n)));
    return OCPQP_OK;
}

}  // namespace

extern "C" {

int ocpqp_abi_version(void) { return OCPQP_ABI_VERSION; }

const char* ocpqp_last_error(void) { return g_last_error.c_str(); }

int ocpqp_layout(const OcpQpDimC* dim, int64_t* out, int32_t out_len) {
    Layout L;
    int rc = build_layout(dim, L);
    if (rc) return rc;
    if (!out || out_len < 6 + OCPQP_NUM_FIELDS) return fail(OCPQP_E_ARG, "out too short");
    out[0] = L.ny; out[1] = L.ne; out[2] = L.nc; out[3] = L.nv; out[4] = L.ns_tot; out[5] = L.nc;
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) out[6 + f] = L.flen[f];
    return OCPQP_OK;
}

int ocpqp_plan_dispatch_hint(OcpPlan* P, int32_t on);

int ocpqp_plan_create(const OcpQpDimC* dim, int32_t batch, OcpPlan** out) {
    if (!out) return fail(OCPQP_E_ARG, "out is NULL");
    *out = nullptr;
    if (batch < 0) return fail(OCPQP_E_ARG, "batch must be >= 0");
    OcpPlan* P = new OcpPlan();
    int rc = build_layout(dim, P->L);
    if (rc) { delete P; return rc; }
    P->B = batch;
    cudaError_t e = cudaGetDevice(&P->device);
    if (e == cudaSuccess) e = cudaDeviceGetAttribute(&P->num_sms, cudaDevAttrMultiProcessorCount, P->device);
    if (e != cudaSuccess) { delete P; return cuda_fail(e, "no CUDA device"); }
    int occ = 0;
    if (detect_fast(P)) {
        if (!plan_fast(P, &occ)) P->fast = false;
    }
    if (!P->fast) {
        place_workspace(P);
        occ = ipm_occupancy(P->threads, P->smem_bytes);
        while (occ == 0 && P->smem_bytes > 0) {
            // shrink the shared-memory share until one CTA fits
            P->smem_mask = 0; P->smem_bytes = 0;
            occ = ipm_occupancy(P->threads, 0);
        }
    }
    if (occ == 0) { delete P; return fail(OCPQP_E_CUDA, "kernel does not fit on an SM"); }
    // experiments: cap the resident CTAs per SM (working set vs latency hiding)
    if (const char* envc = getenv("OCPQP_CTAS_PER_SM")) occ = std::max(1, std::min(occ, atoi(envc)));
    if (P->fast) {
        const int teams = fast_teams_per_cta(P->shape);
        const int ctas = std::max(1, std::min((std::max(1, batch) + teams - 1) / teams, occ * P->num_sms));
        P->grid = ctas;
        P->slots = ctas * teams;
    } else {
        P->slots = std::max(1, std::min(std::max(1, batch), occ * P->num_sms));
        P->grid = P->slots;
    }
    const Layout& L = P->L;
    const size_t S = L.st.size();
    e = cudaMalloc(&P->d_st, sizeof(StageInfo) * S);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_idxb, sizeof(int) * std::max<size_t>(1, L.idxb.size()));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_idxs, sizeof(int) * std::max<size_t>(1, L.idxs.size()));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_var_box, sizeof(int) * L.var_box.size());
    if (e == cudaSuccess) e = cudaMalloc(&P->d_row_slack, sizeof(int) * L.row_slack.size());
    if (e == cudaSuccess) e = cudaMalloc(&P->d_counter, sizeof(int));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_sinv, sizeof(int));
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) P->max_flen = std::max(P->max_flen, L.flen[f]);
    if (e == cudaSuccess) e = cudaMalloc(&P->d_defaults, sizeof(double) * 4 * P->max_flen);
    if (e == cudaSuccess) {
        std::vector<double> dflt(4 * P->max_flen);
        for (long long i = 0; i < P->max_flen; ++i) {
            dflt[i] = 0.0;
            dflt[P->max_flen + i] = 1.0;
            dflt[2 * P->max_flen + i] = -INFINITY;
            dflt[3 * P->max_flen + i] = INFINITY;
        }
        e = cudaMemcpy(P->d_defaults, dflt.data(), sizeof(double) * dflt.size(), cudaMemcpyHostToDevice);
    }
    if (e == cudaSuccess) e = cudaMalloc(&P->d_ws, sizeof(double) * (size_t)P->ws_slot * P->slots);
    // per-solve buffers sized for the worst case here, so that a solve never
    // allocates (the extended workspace of the non-speed modes excepted, see
    // the header): the escape list of balance mode and the packed [B A]
    if (e == cudaSuccess) e = cudaMalloc(&P->d_esc, sizeof(int) * (1 + (size_t)std::max(1, P->B)));
    if (e == cudaSuccess) e = cudaMalloc(&P->d_esc_meta, sizeof(long long) * 3 * (size_t)std::max(1, P->B));
    if (e == cudaSuccess && P->fast && P->shape.kind == 0) {
        const long long need = std::max(1ll, (long long)L.N * P->shape.nx * (P->shape.nx + P->shape.nu) *
                                                  std::max(1, P->B));
        e = cudaMalloc(&P->d_ba, sizeof(double) * need);
        if (e == cudaSuccess) P->ba_cap = need;
    }
    if (e == cudaSuccess) e = cudaMemcpy(P->d_st, L.st.data(), sizeof(StageInfo) * S, cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !L.idxb.empty())
        e = cudaMemcpy(P->d_idxb, L.idxb.data(), sizeof(int) * L.idxb.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess && !L.idxs.empty())
        e = cudaMemcpy(P->d_idxs, L.idxs.data(), sizeof(int) * L.idxs.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(P->d_var_box, L.var_box.data(), sizeof(int) * L.var_box.size(), cudaMemcpyHostToDevice);
    if (e == cudaSuccess)
        e = cudaMemcpy(P->d_row_slack, L.row_slack.data(), sizeof(int) * L.row_slack.size(),
                       cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
        ocpqp_plan_destroy(P);
        return cuda_fail(e, "plan allocation");
    }
    const char* envh = getenv("OCPQP_DISPATCH_HINT");
    if (envh && atoi(envh) == 1 && P->fast && P->shape.kind == 0) ocpqp_plan_dispatch_hint(P, 1);
    *out = P;
    return OCPQP_OK;
}

int ocpqp_plan_destroy(OcpPlan* P) {
    if (!P) return OCPQP_OK;
    cudaFree(P->d_st); cudaFree(P->d_idxb); cudaFree(P->d_idxs); cudaFree(P->d_var_box);
    cudaFree(P->d_row_slack); cudaFree(P->d_counter); cudaFree(P->d_prev_iters); cudaFree(P->d_order); cudaFree(P->d_hint_ctr); cudaFree(P->d_ws); cudaFree(P->d_defaults);
    cudaFree(P->d_sinv);
    cudaFree(P->d_ba);
    cudaFree(P->d_esc);
    cudaFree(P->d_esc_meta);
    cudaFree(P->d_ws2);
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) cudaFree(P->h_field[f]);
    cudaFree(P->hy); cudaFree(P->hpi); cudaFree(P->hlam); cudaFree(P->ht);
    cudaFree(P->hstatus); cudaFree(P->hiters); cudaFree(P->hres); cudaFree(P->hflops);
    cudaFree(P->htrace);
    delete P;
    return OCPQP_OK;
}

// Plan introspection for the host bindings: threads, slots, smem bytes,
// smem mask, workspace doubles per slot.
// Internal diagnostics (not in the public header): make the shaped kernels
// accumulate clock64 cycles per IPM phase into dev_buf [B, 8] (nullptr = off).
int ocpqp_debug_phases(OcpPlan* P, int64_t* dev_buf) {
    if (!P) return fail(OCPQP_E_ARG, "plan is NULL");
    P->dbg = (long long*)dev_buf;
    return OCPQP_OK;
}

int ocpqp_plan_info(const OcpPlan* P, int64_t* out, int32_t out_len) {
    if (!P || !out || out_len < 8) return fail(OCPQP_E_ARG, "bad arguments");
    out[0] = P->threads; out[1] = P->slots; out[2] = (int64_t)P->smem_bytes;
    out[3] = (int64_t)P->smem_mask; out[4] = P->ws_slot;
    out[5] = P->fast ? 1 + P->shape.kind : 0;   /* 0 generic, 1 team kernel, 2 row kernel */
    out[6] = P->fast ? P->shape.team : P->threads;
    out[7] = P->grid;
    if (out_len >= 9) out[8] = P->fast && P->shape.kind == 0 ? P->shape.sm : 0;
    return OCPQP_OK;
}

// Runs a plan's work on the device it was created on (restoring the caller's
// current device afterwards): a plan's buffers live on that device.
struct DeviceGuard {
    int prev = -1, dev;
    explicit DeviceGuard(int d) : dev(d) {
        if (cudaGetDevice(&prev) == cudaSuccess && prev != dev) cudaSetDevice(dev);
    }
    ~DeviceGuard() {
        if (prev >= 0 && prev != dev) cudaSetDevice(prev);
    }
};

// order[rank] = q, ranked by the previous solve's iteration count (descending; ties by index)
__global__ void k_order_hint(const int* it, int B, int* order) {
    for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < B; q += gridDim.x * blockDim.x) {
        const int v = it[q];
        int r = 0;
        for (int j = 0; j < B; ++j) {
            const int w = it[j];
            r += (w > v) || (w == v && j < q);
        }
        order[r] = q;
    }
}
constexpr int kHintSms = 1024;   // per-SM counters behind the two list cursors

// Dispatch hint of the team kernel (opt-in; also OCPQP_DISPATCH_HINT=1 at plan creation):
// a solve hands out its QPs in the order of the plan's previous solve's iteration counts,
// slowest first, and the CTAs that find themselves alone on their SM take the slowest ones
// (a QP alone on an SM runs ~20 % faster per iteration, and a launch ends with its slowest
// QP).  For repeated solves of similar batches (closed-loop MPC); results do not change.
int ocpqp_plan_dispatch_hint(OcpPlan* P, int32_t on) {
    if (!P) return fail(OCPQP_E_ARG, "plan is NULL");
    DeviceGuard dg(P->device);
    if (on && !(P->fast && P->shape.kind == 0))
        return fail(OCPQP_E_UNSUPPORTED, "the dispatch hint belongs to the team kernel");
    if (on && !P->d_prev_iters) {
        const size_t nb = sizeof(int) * (size_t)std::max(1, P->B);
        if (cudaMalloc(&P->d_prev_iters, nb) != cudaSuccess || cudaMalloc(&P->d_order, nb) != cudaSuccess ||
            cudaMalloc(&P->d_hint_ctr, sizeof(int) * (2 + kHintSms)) != cudaSuccess)
            return fail(OCPQP_E_CUDA, "dispatch hint: allocation failed");
    }
    P->hint_on = on != 0;
    P->hint_valid = false;
    return OCPQP_OK;
}

// The BIG shapes read stage data by TMA bulk copies: 16-byte aligned blocks.
static int check_tma_alignment(const OcpPlan* P, const OcpQpDataC* data) {
    if (!(P->fast && P->shape.kind == 0 && fast_big(P->shape)) || !data) return OCPQP_OK;
    static const int fs[] = {OCPQP_F_Q, OCPQP_F_S, OCPQP_F_R, OCPQP_F_q, OCPQP_F_r, OCPQP_F_b};
    for (int f : fs) {
        if (!data->ptr[f] || P->L.flen[f] == 0) continue;
        if (((uintptr_t)data->ptr[f] & 15u) || (data->batch_stride[f] & 1))
            return fail(OCPQP_E_ARG, "this stage shape streams Q, S, R, q, r, b by TMA: their device "
                                     "pointers must be 16-byte aligned and batch strides even");
    }
    return OCPQP_OK;
}

int ocpqp_solve(OcpPlan* P, const OcpQpDataC* data, const OcpIpmArgC* arg, OcpIterC* iter,
                OcpStatsC* stats, void* stream) {
    if (!P) return fail(OCPQP_E_ARG, "plan is NULL");
    int rc = check_arg(arg);
    if (rc) return rc;
    if ((rc = check_tma_alignment(P, data))) return rc;
    DeviceGuard dg(P->device);
    // zero-length vectors (e.g. nc = 0 for an unconstrained QP) may be NULL
    const Layout& Ly = P->L;
    if (!iter || !stats || (Ly.ny && !iter->y) || (Ly.ne && !iter->pi) || (Ly.nc && !iter->lam) ||
        (Ly.nc && !iter->t) || !stats->status || !stats->iterations || !stats->res || !stats->flops)
        return fail(OCPQP_E_ARG, "iterate / stats buffers must not be NULL");
    if (P->B == 0) return OCPQP_OK;
    const bool ext = needs_ext(arg);
    if (ext && (rc = ensure_ext(P))) return rc;
    const bool team = P->fast && P->shape.kind == 0 &&
                      team_supports(arg, P->shape.nx + P->shape.nu, P->shape.nx) && !getenv("OCPQP_EXT_GENERIC");
    KParams k;
    fill_kparams(P, k, data, !(ext && P->fast) || team);
    size_t gen_smem = P->smem_bytes;
    if (ext && P->fast && !team && getenv("OCPQP_GEN_SMEM")) {
        // the generic kernel on a shaped-kernel plan keeps its workspace in
        // global memory by default: measured faster (the full L1 caches it)
        // than a shared-memory placement that shrinks the L1 (cfg 1 balance
        // 6.5 vs 8.9 ms); OCPQP_GEN_SMEM=1 selects the placement
        place_generic_on_fast(P);
        k.smem_mask = P->gen_mask;
        for (int b = 0; b < WS_EXT0; ++b) k.smem_off[b] = P->gen_off[b];
        gen_smem = P->gen_bytes;
    }
    SolveParams sp;
    memset(&sp, 0, sizeof(sp));
    sp.arg = *arg;
    sp.y = iter->y; sp.pi = iter->pi; sp.lam = iter->lam; sp.t = iter->t;
    sp.status = stats->status; sp.iters = stats->iterations; sp.res = stats->res;
    sp.flops = (long long*)stats->flops; sp.trace = stats->trace;
    fill_defaults(P, k);   // no null field pointers in any kernel
    cudaError_t e;
    if (P->fast && (!ext || team)) {
        if (ext && arg->use_qr_fallback) {
            CUDA_TRY(cudaMemsetAsync(P->d_esc, 0, sizeof(int), (cudaStream_t)stream));
            k.esc_count = P->d_esc;
            k.esc_list = P->d_esc + 1;
            k.esc_meta = P->d_esc_meta;
        }
        fill_defaults(P, k);
        if (P->shape.kind == 0) {
            if (!getenv("OCPQP_NO_SINV")) {
                e = launch_stage_invariant(k.f, k.bs, P->L.N, P->shape.nx, P->shape.nu, P->d_sinv,
                                           (cudaStream_t)stream);
                if (e != cudaSuccess) return cuda_fail(e, "k_stage_invariant launch");
                k.sinv = P->d_sinv;
            }
            // [B A] packed per stage: one copy when A and B are broadcast
            const int nx = P->shape.nx, nu = P->shape.nu;
            const long long per_qp = (long long)P->L.N * nx * (nx + nu);
            const bool shared = k.bs[OCPQP_F_A] == 0 && k.bs[OCPQP_F_B] == 0;
            const long long need = std::max(1ll, per_qp * (shared ? 1 : P->B));
            if (P->ba_cap < need) return fail(OCPQP_E_CUDA, "packed [B A] buffer smaller than the batch");
            k.ba = P->d_ba;
            k.ba_bs = shared ? 0 : per_qp;
            // OCPQP_BA_STAGE_MAJOR=1: batch-interleaved [N][B][stage] packing
            // (layout experiment; QP-major is the default, profiles/r02_layout_*)
            const char* envl = getenv("OCPQP_BA_STAGE_MAJOR");
            const int smaj = (!shared && envl && atoi(envl) == 1) ? 1 : 0;
            if (smaj) {
                k.ba_bs = (long long)nx * (nx + nu);
                k.ba_ns = (long long)P->B * nx * (nx + nu);
            }
            e = launch_pack_ba(k.f[OCPQP_F_A], k.bs[OCPQP_F_A], k.f[OCPQP_F_B], k.bs[OCPQP_F_B], P->B,
                               P->L.N, nx, nu, P->d_ba, shared ? 0 : per_qp, (cudaStream_t)stream,
                               fast_big(P->shape), smaj);
            if (e != cudaSuccess) return cuda_fail(e, "k_pack_ba launch");
        }
        if (P->hint_on && P->shape.kind == 0 && P->num_sms <= kHintSms) {
            k.prev_iters = P->d_prev_iters;
            if (P->hint_valid) {
                k_order_hint<<<std::min(64, (P->B + 255) / 256), 256, 0, (cudaStream_t)stream>>>(
                    P->d_prev_iters, P->B, P->d_order);
                CUDA_TRY(cudaMemsetAsync(P->d_hint_ctr, 0, sizeof(int) * (2 + kHintSms), (cudaStream_t)stream));
                // CTAs that stay alone on their SM when every CTA is resident at two per SM
                const int occ = fast_occupancy(P->shape, P->smem_bytes);
                const int alone = (occ == 2 && P->grid > P->num_sms && P->grid <= 2 * P->num_sms)
                                      ? 2 * P->num_sms - P->grid : 0;
                k.order = P->d_order;
                k.n_first = std::min(alone, P->B);
                k.hint_ctr = P->d_hint_ctr;
            }
        }
        e = launch_fast_solve(P->shape, k, sp, P->grid, P->smem_bytes, (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "k_fast_solve launch");
        if (k.prev_iters) P->hint_valid = true;
        if (k.esc_list) {
            // the QPs the team kernel escaped, re-solved from their start by the
            // generic kernel (workspace in global memory, list on the device)
            KParams g;
            fill_kparams(P, g, data, false);
            fill_defaults(P, g);
            g.esc_count = k.esc_count;
            g.esc_list = k.esc_list;
            g.esc_meta = k.esc_meta;
            // escapes are rare: widest CTAs (the per-QP latency sets their cost)
            e = launch_ipm_solve(g, sp, P->slots, 512, 0, (cudaStream_t)stream);
            if (e != cudaSuccess) return cuda_fail(e, "k_ipm_solve (escapes) launch");
            if (getenv("OCPQP_ESC_STATS")) {  // diagnostics: escaped QPs of this solve
                int cnt = 0;
                cudaMemcpyAsync(&cnt, k.esc_count, sizeof(int), cudaMemcpyDeviceToHost,
                                (cudaStream_t)stream);
                cudaStreamSynchronize((cudaStream_t)stream);
                fprintf(stderr, "ocpqp: %d of %d QPs escaped to the generic kernel\n", cnt, P->B);
            }
        }
    } else {
        e = launch_ipm_solve(k, sp, P->slots, P->threads, gen_smem, (cudaStream_t)stream);
        if (e != cudaSuccess) return cuda_fail(e, "k_ipm_solve launch");
    }
    return OCPQP_OK;
}

// Device-side address of a page-locked (pinned or registered) host buffer,
// nullptr for pageable / device / NULL pointers.
static void* mapped_host(void* p) {
    if (!p) return nullptr;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
        cudaGetLastError();
        return nullptr;
    }
    if (at.type != cudaMemoryTypeHost || !at.devicePointer) return nullptr;
    return at.devicePointer;
}

int ocpqp_solve_host(OcpPlan* P, const OcpQpDataC* hd, const OcpIpmArgC* arg, OcpIterC* hit,
                     OcpStatsC* hst, void* stream_) {
    if (!P || !hd || !hit || !hst) return fail(OCPQP_E_ARG, "NULL argument");
    DeviceGuard dg(P->device);
    int rc = check_arg(arg);
    if (rc) return rc;
    cudaStream_t stream = (cudaStream_t)stream_;
    const Layout& L = P->L;
    const long long B = P->B;
    OcpQpDataC dd;
    memset(&dd, 0, sizeof(dd));
    for (int f = 0; f < OCPQP_NUM_FIELDS; ++f) {
        if (!hd->ptr[f] || L.flen[f] == 0) continue;
        const long long copies = hd->batch_stride[f] == 0 ? 1 : B;
        if (hd->batch_stride[f] != 0 && hd->batch_stride[f] != L.flen[f])
            return fail(OCPQP_E_DIMENSION, "host field %d: batch stride must be 0 or %lld", f, L.flen[f]);
        const long long n = copies * L.flen[f];
        if (P->h_field_len[f] < n) {
            cudaFree(P->h_field[f]);
            P->h_field[f] = nullptr;
            CUDA_TRY(cudaMalloc(&P->h_field[f], sizeof(double) * n));
            P->h_field_len[f] = n;
        }
        CUDA_TRY(cudaMemcpyAsync(P->h_field[f], hd->ptr[f], sizeof(double) * n, cudaMemcpyHostToDevice, stream));
        dd.ptr[f] = P->h_field[f];
        dd.batch_stride[f] = hd->batch_stride[f];
    }
    if ((rc = ensure(&P->hy, B * L.ny)) || (rc = ensure(&P->hpi, B * L.ne)) ||
        (rc = ensure(&P->hlam, B * L.nc)) || (rc = ensure(&P->ht, B * L.nc)) ||
        (rc = ensure(&P->hstatus, B)) || (rc = ensure(&P->hiters, B)) ||
        (rc = ensure(&P->hres, B * 5)) || (rc = ensure(&P->hflops, B)))
        return rc;
    if (hst->trace) {
        if (P->htrace_iters < arg->iter_max) {
            cudaFree(P->htrace);
            P->htrace = nullptr;
            CUDA_TRY(cudaMalloc(&P->htrace, sizeof(double) * std::max(1ll, B * arg->iter_max * 8)));
            P->htrace_iters = arg->iter_max;
        }
    }
    if (arg->warm_start != 0) {
        CUDA_TRY(cudaMemcpyAsync(P->hy, hit->y, sizeof(double) * B * L.ny, cudaMemcpyHostToDevice, stream));
        if (arg->warm_start == 2) {
            CUDA_TRY(cudaMemcpyAsync(P->hpi, hit->pi, sizeof(double) * B * L.ne, cudaMemcpyHostToDevice, stream));
            CUDA_TRY(cudaMemcpyAsync(P->hlam, hit->lam, sizeof(double) * B * L.nc, cudaMemcpyHostToDevice, stream));
        }
    }
    OcpIterC di{P->hy, P->hpi, P->hlam, P->ht};
    OcpStatsC ds{P->hstatus, P->hiters, P->hres, (int64_t*)P->hflops, hst->trace ? P->htrace : nullptr};
    // Page-locked result buffers are written by the kernel directly (mapped
    // host memory): each QP stores its solution and statistics when it
    // finishes, overlapping the transfer with the QPs still iterating instead
    // of a device->host copy after the slowest one.
    void* my = mapped_host(hit->y);
    void* mpi = mapped_host(hit->pi);
    void* mlam = mapped_host(hit->lam);
    void* mt = mapped_host(hit->t);
    void* mst = mapped_host(hst->status);
    void* mit = mapped_host(hst->iterations);
    void* mres = mapped_host(hst->res);
    void* mfl = mapped_host(hst->flops);
    // only the shaped kernels keep their iterate on chip; the generic kernel
    // iterates in the output buffers, which must then be device memory
    const bool direct = my && mpi && mlam && mt && mst && mit && mres && mfl && !hst->trace &&
                        arg->warm_start == 0 && P->fast && !needs_ext(arg) &&
                        !getenv("OCPQP_NO_MAPPED");
    if (direct) {
        di = OcpIterC{(double*)my, (double*)mpi, (double*)mlam, (double*)mt};
        ds = OcpStatsC{(int32_t*)mst, (int32_t*)mit, (double*)mres, (int64_t*)mfl, nullptr};
    }
    rc = ocpqp_solve(P, &dd, arg, &di, &ds, stream);
    if (rc) return rc;
    if (direct) {
        CUDA_TRY(cudaStreamSynchronize(stream));
        return OCPQP_OK;
    }
    if (hit->y) CUDA_TRY(cudaMemcpyAsync(hit->y, P->hy, sizeof(double) * B * L.ny, cudaMemcpyDeviceToHost, stream));
    if (hit->pi) CUDA_TRY(cudaMemcpyAsync(hit->pi, P->hpi, sizeof(double) * B * L.ne, cudaMemcpyDeviceToHost, stream));
    if (hit->lam) CUDA_TRY(cudaMemcpyAsync(hit->lam, P->hlam, sizeof(double) * B * L.nc, cudaMemcpyDeviceToHost, stream));
    if (hit->t) CUDA_TRY(cudaMemcpyAsync(hit->t, P->ht, sizeof(double) * B * L.nc, cudaMemcpyDeviceToHost, stream));
    if (hst->status) CUDA_TRY(cudaMemcpyAsync(hst->status, P->hstatus, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, stream));
    if (hst->iterations) CUDA_TRY(cudaMemcpyAsync(hst->iterations, P->hiters, sizeof(int32_t) * B, cudaMemcpyDeviceToHost, stream));
    if (hst->res) CUDA_TRY(cudaMemcpyAsync(hst->res, P->hres, sizeof(double) * B * 5, cudaMemcpyDeviceToHost, stream));
    if (hst->flops) CUDA_TRY(cudaMemcpyAsync(hst->flops, P->hflops, sizeof(int64_t) * B, cudaMemcpyDeviceToHost, stream));
    if (hst->trace) CUDA_TRY(cudaMemcpyAsync(hst->trace, P->htrace, sizeof(double) * B * arg->iter_max * 8, cudaMemcpyDeviceToHost, stream));
    CUDA_TRY(cudaStreamSynchronize(stream));
    return OCPQP_OK;
}

int ocpqp_residuals(OcpPlan* P, const OcpQpDataC* data, const OcpIterC* pt, double* r_g,
                    double* r_b, double* r_d, double* r_m, double* norms, void* stream) {
    if (!P || !pt || !norms) return fail(OCPQP_E_ARG, "NULL argument");
    DeviceGuard dg(P->device);
    if (P->B == 0) return OCPQP_OK;
    KParams k;
    fill_kparams(P, k, data, false);
    fill_defaults(P, k);
    cudaError_t e = launch_residuals(k, pt->y, pt->pi, pt->lam, pt->t, r_g, r_b, r_d, r_m, norms,
                                     P->slots, P->threads, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "k_residuals launch");
    return OCPQP_OK;
}

int ocpqp_newton_step(OcpPlan* P, const OcpQpDataC* data, double reg, const OcpIterC* it,
                      const double* r_g, const double* r_b, const double* r_d, const double* r_m,
                      OcpIterC* step, int32_t* fail_stage, void* stream) {
    if (!P || !it || !step || !r_g || !r_b || !r_d || !r_m || !fail_stage)
        return fail(OCPQP_E_ARG, "NULL argument");
    DeviceGuard dg(P->device);
    if (P->B == 0) return OCPQP_OK;
    KParams k;
    fill_kparams(P, k, data, false);
    fill_defaults(P, k);
    cudaError_t e = launch_newton_step(k, reg, it->lam, it->t, r_g, r_b, r_d, r_m, step->y,
                                       step->pi, step->lam, step->t, fail_stage, P->slots,
                                       P->threads, (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "k_newton_step launch");
    return OCPQP_OK;
}

int ocpqp_shift_guess(OcpPlan* P, const OcpQpDataC* data, const OcpIterC* sol, OcpIterC* guess,
                      void* stream) {
    if (!P || !sol || !guess) return fail(OCPQP_E_ARG, "NULL argument");
    DeviceGuard dg(P->device);
    const Layout& L = P->L;
    if ((L.ny && (!sol->y || !guess->y)) || (L.ne && (!sol->pi || !guess->pi)) ||
        (L.nc && (!sol->lam || !sol->t || !guess->lam || !guess->t)))
        return fail(OCPQP_E_ARG, "solution / guess buffers must not be NULL");
    if (sol->y == guess->y) return fail(OCPQP_E_ARG, "guess must not alias the solution");
    for (int n = 0; n < L.N; ++n)
        if (L.nx[n] != L.nx[n + 1])
            return fail(OCPQP_E_DIMENSION, "shift needs equal state dimensions (stage %d)", n);
    if (P->B == 0) return OCPQP_OK;
    KParams k;
    fill_kparams(P, k, data, false);
    fill_defaults(P, k);
    cudaError_t e = launch_shift_guess(k, sol->y, sol->pi, sol->lam, sol->t, guess->y, guess->pi,
                                       guess->lam, guess->t, P->slots, P->threads,
                                       (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "k_shift_guess launch");
    return OCPQP_OK;
}

int ocpqp_factor_export(OcpPlan* P, int32_t qp, double* P_out, double* K_out) {
    if (!P || qp < 0 || qp >= P->B) return fail(OCPQP_E_ARG, "bad plan or qp index");
    DeviceGuard dg(P->device);
    if (P->B > P->slots)
        return fail(OCPQP_E_UNSUPPORTED, "factor export needs batch <= slots (%d)", P->slots);
    const double* slot = P->d_ws + (long long)qp * P->ws_slot;
    if (P_out)
        CUDA_TRY(cudaMemcpy(P_out, slot + P->ws_off[WS_P], sizeof(double) * P->L.ws_size[WS_P],
                            cudaMemcpyDeviceToHost));
    if (K_out)
        CUDA_TRY(cudaMemcpy(K_out, slot + P->ws_off[WS_K], sizeof(double) * P->L.ws_size[WS_K],
                            cudaMemcpyDeviceToHost));
    return OCPQP_OK;
}

}  // extern "C"
