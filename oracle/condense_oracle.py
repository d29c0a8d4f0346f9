"""CPU restatement of partial condensing / expansion (TEST INFRASTRUCTURE ONLY).

numpy restatement of the reference's partial_condense / partial_expand
(/root/reference/pkg/src/mpcqp/condensing.py:451-619, with condense(keep_x0=True)
:160-340, _cost_recursion (classical) :128-157, expand_solution :343-429), for
QPs without soft rows.  Pinned to the reference by tests/test_condense_oracle.py
against tests/golden/pcond.npz; used by the GPU parity tests as the checker of
csrc/ocpqp_condense.cu.  Operates on this package's OcpQp / QpSolution objects.
"""

from __future__ import annotations

import numpy as np


def _blocks(N, N1):
    starts = list(range(0, N, N1))
    return [(n0, min(n0 + N1, N)) for n0 in starts]


def _condense_block(qp, n0, n1):
    """Condensed data of stages n0..n1-1 (sub-QP with zero-cost terminal at n1)."""
    d = qp.dim
    L = n1 - n0
    st = [qp._stages[n] for n in range(n0, n1)]
    dy = [qp._dyn[n] for n in range(n0, n1)]
    nx0 = int(d.nx[n0])
    u_off, off = [], nx0
    for i in range(L):
        nu = int(d.nu[n0 + i])
        u_off.append(off if nu else None)
        off += nu
    nv = off
    # predictions (condensing.py:196-207)
    pred = [np.zeros((int(d.nx[n0 + i]), nv)) for i in range(L + 1)]
    pred[0][:, :nx0] = np.eye(nx0)
    gamma = [np.zeros(nx0)]
    for i in range(L):
        A, B, b = dy[i]["A"], dy[i]["B"], dy[i]["b"]
        pred[i + 1] = A @ pred[i]
        if u_off[i] is not None:
            pred[i + 1][:, u_off[i]: u_off[i] + B.shape[1]] += B
        gamma.append(A @ gamma[i] + b)
    # cost recursion with a zero-cost terminal placeholder (condensing.py:148-157)
    nxL = int(d.nx[n1])
    P = [None] * (L + 1)
    Y = [None] * L
    P[L] = np.zeros((nxL, nxL))
    for i in range(L - 1, -1, -1):
        A, B = dy[i]["A"], dy[i]["B"]
        PA = P[i + 1] @ A
        PB = P[i + 1] @ B
        Y[i] = A.T @ PB + st[i]["S"].T
        Pn = A.T @ PA + st[i]["Q"]
        P[i] = 0.5 * (Pn + Pn.T)
    beta = [None] * (L + 1)
    beta[L] = np.zeros(nxL)
    for i in range(L - 1, -1, -1):
        beta[i] = st[i]["q"] + st[i]["Q"] @ gamma[i] + dy[i]["A"].T @ beta[i + 1]
    Hc = np.zeros((nv, nv))
    gc = np.zeros(nv)
    Hc[:nx0, :nx0] = P[0]
    gc[:nx0] = beta[0]
    for j in range(L):
        nu = int(d.nu[n0 + j])
        if not nu:
            continue
        o = u_off[j]
        Bj = dy[j]["B"]
        Hc[o: o + nu, o: o + nu] = st[j]["R"] + Bj.T @ (P[j + 1] @ Bj)
        gc[o: o + nu] = st[j]["r"] + st[j]["S"] @ gamma[j] + Bj.T @ beta[j + 1]
        cols = pred[j].T @ Y[j]
        Hc[:, o: o + nu] += cols
        Hc[o: o + nu, :] += cols.T
    Hc = 0.5 * (Hc + Hc.T)
    # constraint routing (condensing.py:251-288)
    box, gen = [], []
    for i in range(L):
        n = n0 + i
        nu = int(d.nu[n])
        s = st[i]
        for r, k in enumerate(s["idxb"]):
            if k < nu:
                box.append((u_off[i] + int(k), i, r))
            elif i == 0:
                box.append((int(k) - nu, i, r))
            else:
                c = int(k) - nu
                gen.append((pred[i][c].copy(), s["lb"][r] - gamma[i][c], s["ub"][r] - gamma[i][c],
                            i, r))
        for g in range(int(d.ng[n])):
            row = np.zeros(nv)
            if nu:
                row[u_off[i]: u_off[i] + nu] = s["D"][g]
            row += s["C"][g] @ pred[i]
            sh = float(s["C"][g] @ gamma[i])
            gen.append((row, s["lg"][g] - sh, s["ug"][g] - sh, i, int(d.nb[n]) + g))
    box.sort(key=lambda e: e[0])
    return dict(nx0=nx0, nv=nv, u_off=u_off, pred=pred, gamma=gamma, Hc=Hc, gc=gc, box=box,
                gen=gen, L=L, n0=n0)


def partial_condense(qp, N1):
    """(fields per new stage, blocks) of the condensed QP; fields as dicts."""
    d = qp.dim
    out = []
    blocks = []
    for n0, n1 in _blocks(d.N, N1):
        c = _condense_block(qp, n0, n1)
        nx0, nv = c["nx0"], c["nv"]
        nun = nv - nx0
        zidx = np.array([e[0] for e in c["box"]], dtype=int)
        new_idx = np.where(zidx < nx0, zidx + nun, zidx - nx0)
        perm = np.argsort(new_idx, kind="stable")
        st = {}
        H, g = c["Hc"], c["gc"]
        st["Q"], st["S"], st["R"] = H[:nx0, :nx0], H[nx0:, :nx0], H[nx0:, nx0:]
        st["q"], st["r"] = g[:nx0], g[nx0:]
        pL = c["pred"][-1]
        st["A"], st["B"], st["b"] = pL[:, :nx0], pL[:, nx0:], c["gamma"][-1]
        src = [(e[1], e[2]) for e in c["box"]]
        st["idxb"] = new_idx[perm]
        st["lb"] = np.array([qp._stages[n0 + src[j][0]]["lb"][src[j][1]] for j in perm])
        st["ub"] = np.array([qp._stages[n0 + src[j][0]]["ub"][src[j][1]] for j in perm])
        Cz = np.array([e[0] for e in c["gen"]]).reshape(len(c["gen"]), nv)
        st["C"], st["D"] = Cz[:, :nx0], Cz[:, nx0:]
        st["lg"] = np.array([e[1] for e in c["gen"]])
        st["ug"] = np.array([e[2] for e in c["gen"]])
        rows = [src[j] for j in perm] + [(e[3], e[4]) for e in c["gen"]]
        st["maskl"] = np.array([qp._stages[n0 + i]["maskl"][r] for i, r in rows])
        st["masku"] = np.array([qp._stages[n0 + i]["masku"][r] for i, r in rows])
        out.append(st)
        blocks.append(dict(n0=n0, n1=n1, cond=c, rows=rows, m=len(rows)))
    return out, blocks


def partial_expand(qp, blocks, short):
    """Full-horizon (y, pi, lam, t) from the condensed solution arrays.

    ``short`` holds y/pi/lam/t of the condensed QP plus its layout offsets
    (u_off, x_off, pi_off, c_off lists); ``qp`` provides the full layout.
    """
    from paper_2003_02547_b200.layout import OcpLayout

    d = qp.dim
    lay = OcpLayout(d)
    y = np.zeros(lay.ny)
    pi = np.zeros(lay.ne)
    lam = np.zeros(lay.nc)
    t = np.zeros(lay.nc)
    sl = short["layout"]
    for k, blk in enumerate(blocks):
        c = blk["cond"]
        n0, L, nx0 = blk["n0"], c["L"], c["nx0"]
        xk = short["y"][sl.x_off[k]: sl.x_off[k] + nx0]
        uk = short["y"][sl.u_off[k]: sl.u_off[k] + c["nv"] - nx0]
        xs = [xk.copy()]
        for i in range(L):
            n = n0 + i
            nu = int(d.nu[n])
            u = uk[c["u_off"][i] - nx0: c["u_off"][i] - nx0 + nu] if nu else np.zeros(0)
            y[lay.u_off[n]: lay.u_off[n] + nu] = u
            y[lay.x_off[n]: lay.x_off[n] + int(d.nx[n])] = xs[i]
            dyn = qp._dyn[n]
            xs.append(dyn["A"] @ xs[i] + dyn["B"] @ u + dyn["b"])
        m = blk["m"]
        cs = sl.c_off[k]
        for r, (i, src) in enumerate(blk["rows"]):
            n = n0 + i
            mo = int(d.nb[n] + d.ng[n])
            lam[lay.c_off[n] + src] = short["lam"][cs + r]
            lam[lay.c_off[n] + mo + src] = short["lam"][cs + m + r]
            t[lay.c_off[n] + src] = short["t"][cs + r]
            t[lay.c_off[n] + mo + src] = short["t"][cs + m + r]
        # costate recursion (condensing.py:397-412)
        pim = short["pi"][sl.pi_off[k]: sl.pi_off[k] + int(d.nx[n0 + L])]
        pi[lay.pi_off[n0 + L - 1]: lay.pi_off[n0 + L - 1] + pim.size] = pim
        for mm in range(L - 1, 0, -1):
            n = n0 + mm
            s = qp._stages[n]
            nu = int(d.nu[n])
            lm = lam[lay.c_off[n]: lay.c_off[n] + 2 * int(d.nb[n] + d.ng[n])]
            mo = int(d.nb[n] + d.ng[n])
            lo = np.concatenate([s["lb"], s["lg"]])
            up = np.concatenate([s["ub"], s["ug"]])
            al = (s["maskl"] != 0) & np.isfinite(lo)
            au = (s["masku"] != 0) & np.isfinite(up)
            coef = np.where(al, lm[:mo], 0.0) - np.where(au, lm[mo:], 0.0)
            ct = np.zeros(nu + int(d.nx[n]))
            np.add.at(ct, s["idxb"], coef[: int(d.nb[n])])
            if int(d.ng[n]):
                ct += np.hstack([s["D"], s["C"]]).T @ coef[int(d.nb[n]):]
            u = y[lay.u_off[n]: lay.u_off[n] + nu]
            val = s["Q"] @ xs[mm] + s["S"].T @ u + s["q"] - ct[nu:]
            val = val + qp._dyn[n]["A"].T @ pim
            pi[lay.pi_off[n - 1]: lay.pi_off[n - 1] + val.size] = val
            pim = val
    N = d.N
    Np = len(blocks)
    for k in range(Np + 1):
        n = blocks[k]["n0"] if k < Np else N
        y[lay.x_off[n]: lay.x_off[n] + int(d.nx[n])] = short["y"][sl.x_off[k]: sl.x_off[k] + int(d.nx[n])]
    ncN = lay.stage_nc(N)
    lam[lay.c_off[N]: lay.c_off[N] + ncN] = short["lam"][sl.c_off[Np]: sl.c_off[Np] + ncN]
    t[lay.c_off[N]: lay.c_off[N] + ncN] = short["t"][sl.c_off[Np]: sl.c_off[Np] + ncN]
    return y, pi, lam, t


# ---------------------------------------------------------------------------
# full condensing (condensing.py:160-340) and expand_solution (:343-429)
# ---------------------------------------------------------------------------

def detect_fixed_x0(qp):
    """(all_fixed, x0hat, fix_rows) from stage-0 equal-bound rows (condensing.py:97-118)."""
    s = qp._stages[0]
    nu0, nx0 = int(qp.dim.nu[0]), int(qp.dim.nx[0])
    x0hat = np.full(nx0, np.nan)
    fix = []
    for i, k in enumerate(s["idxb"]):
        if k < nu0:
            continue
        c = int(k) - nu0
        lo, up = s["lb"][i], s["ub"][i]
        if lo == up and np.isfinite(lo) and s["maskl"][i] != 0.0 and s["masku"][i] != 0.0:
            x0hat[c] = lo
            fix.append((i, c))
    return (not np.any(np.isnan(x0hat))) if nx0 else True, x0hat, fix


def _qr_cholesky(stack):
    """R with R'R = stack'stack, nonnegative diagonal (linalg.py:152-187)."""
    m, n = stack.shape
    R = np.linalg.qr(stack, mode="r")
    d = np.diag(R).copy()
    tol = max(m, n) * np.finfo(float).eps * (np.max(np.abs(d)) if n else 0.0)
    if np.any(np.abs(d) <= tol):
        raise ArithmeticError("RankDeficient")
    return np.where(d[:, None] < 0.0, -R, R)


def full_condense(qp, keep_x0=None, variant="classical"):
    """Dense QP fields (H, g, idxb, lb, ub, C, lg, ug, maskl, masku) + map.

    Classical cost recursion (condensing.py:148-157) with P[N] = sym(Q_N), or
    the square-root recursion (condensing.py:134-146: U_n = qr_cholesky of
    [chol(Q_n)'; U_{n+1} A], P_n = U_n' U_n, Y_n = (U A)'(U B) + S';
    np.linalg.LinAlgError where the reference raises NotPositiveDefinite);
    z = [x0 (kept) | u_0 | ... | u_N]; x-box rows past stage 0 and all general
    rows become dense general rows in stage order; box rows sorted by z.
    """
    d = qp.dim
    N = int(d.N)
    all_fixed, x0hat, fix = detect_fixed_x0(qp)
    if keep_x0 is None:
        keep_x0 = not all_fixed
    if not keep_x0 and not all_fixed:
        raise ValueError("keep_x0=False requires every initial-state component fixed")
    nx0 = int(d.nx[0])
    zx = nx0 if keep_x0 else 0
    u_off, off = [], zx
    for n in range(N + 1):
        nu = int(d.nu[n])
        u_off.append(off if nu else None)
        off += nu
    nv = off
    pred = [np.zeros((int(d.nx[n]), nv)) for n in range(N + 1)]
    gamma = [np.zeros(nx0) if keep_x0 else x0hat.copy()]
    if keep_x0:
        pred[0][:, :nx0] = np.eye(nx0)
    for n in range(N):
        A, B, b = qp._dyn[n]["A"], qp._dyn[n]["B"], qp._dyn[n]["b"]
        pred[n + 1] = A @ pred[n]
        if u_off[n] is not None:
            pred[n + 1][:, u_off[n]: u_off[n] + B.shape[1]] += B
        gamma.append(A @ gamma[n] + b)
    st = qp._stages
    P = [None] * (N + 1)
    Y = [None] * N
    if variant == "square_root":
        def chol_lower(Q):   # scipy.linalg.cholesky(lower=True) reads the lower triangle
            return np.linalg.cholesky(np.tril(Q) + np.tril(Q, -1).T)
        U = chol_lower(st[N]["Q"]).T
        P[N] = U.T @ U
        for n in range(N - 1, -1, -1):
            A, B = qp._dyn[n]["A"], qp._dyn[n]["B"]
            UA, UB = U @ A, U @ B
            Y[n] = UA.T @ UB + st[n]["S"].T
            U = _qr_cholesky(np.vstack([chol_lower(st[n]["Q"]).T, UA]))
            P[n] = U.T @ U
    else:
        P[N] = 0.5 * (st[N]["Q"] + st[N]["Q"].T)
        for n in range(N - 1, -1, -1):
            A, B = qp._dyn[n]["A"], qp._dyn[n]["B"]
            Y[n] = A.T @ (P[n + 1] @ B) + st[n]["S"].T
            Pn = A.T @ (P[n + 1] @ A) + st[n]["Q"]
            P[n] = 0.5 * (Pn + Pn.T)
    beta = [None] * (N + 1)
    beta[N] = st[N]["q"] + st[N]["Q"] @ gamma[N]
    for n in range(N - 1, -1, -1):
        beta[n] = st[n]["q"] + st[n]["Q"] @ gamma[n] + qp._dyn[n]["A"].T @ beta[n + 1]
    H = np.zeros((nv, nv))
    g = np.zeros(nv)
    if keep_x0:
        H[:nx0, :nx0] = P[0]
        g[:nx0] = beta[0]
    for j in range(N + 1):
        nu = int(d.nu[j])
        if not nu:
            continue
        o = u_off[j]
        if j < N:
            Bj = qp._dyn[j]["B"]
            H[o: o + nu, o: o + nu] = st[j]["R"] + Bj.T @ (P[j + 1] @ Bj)
            cross = Y[j]
            g[o: o + nu] = st[j]["r"] + st[j]["S"] @ gamma[j] + Bj.T @ beta[j + 1]
        else:
            H[o: o + nu, o: o + nu] = st[j]["R"]
            cross = st[j]["S"].T
            g[o: o + nu] = st[j]["r"] + st[j]["S"] @ gamma[j]
        cols = pred[j].T @ cross
        H[:, o: o + nu] += cols
        H[o: o + nu, :] += cols.T
    H = 0.5 * (H + H.T)
    box, gen = [], []
    for n in range(N + 1):
        s = st[n]
        nu = int(d.nu[n])
        for r, k in enumerate(s["idxb"]):
            if k < nu:
                box.append((u_off[n] + int(k), n, r))
            elif n == 0 and keep_x0:
                box.append((int(k) - nu, n, r))
            elif n == 0:
                continue
            else:
                c = int(k) - nu
                gen.append((pred[n][c].copy(), s["lb"][r] - gamma[n][c], s["ub"][r] - gamma[n][c],
                            n, r))
        for gi in range(int(d.ng[n])):
            row = np.zeros(nv)
            if nu:
                row[u_off[n]: u_off[n] + nu] = s["D"][gi]
            row += s["C"][gi] @ pred[n]
            sh = float(s["C"][gi] @ gamma[n])
            gen.append((row, s["lg"][gi] - sh, s["ug"][gi] - sh, n, int(d.nb[n]) + gi))
    box.sort(key=lambda e: e[0])
    rows = [(e[1], e[2]) for e in box] + [(e[3], e[4]) for e in gen]
    dense = dict(
        H=H, g=g, idxb=np.array([e[0] for e in box], dtype=int),
        lb=np.array([st[e[1]]["lb"][e[2]] for e in box]),
        ub=np.array([st[e[1]]["ub"][e[2]] for e in box]),
        C=np.array([e[0] for e in gen]).reshape(len(gen), nv),
        lg=np.array([e[1] for e in gen]), ug=np.array([e[2] for e in gen]),
        maskl=np.array([st[n]["maskl"][r] for n, r in rows]),
        masku=np.array([st[n]["masku"][r] for n, r in rows]))
    cmap = dict(keep_x0=keep_x0, x0hat=None if keep_x0 else x0hat, nx0=nx0, u_off=u_off, nv=nv,
                rows=rows, nb=len(box), fix=[] if keep_x0 else fix)
    return dense, cmap


def _ctlam_x(qp, lam, lay, n):
    """(C' lam)_x of stage n over active multipliers (view.py:145-153, 197-205)."""
    d = qp.dim
    s = qp._stages[n]
    nu, nb, ng = int(d.nu[n]), int(d.nb[n]), int(d.ng[n])
    mo = nb + ng
    lm = lam[lay.c_off[n]: lay.c_off[n] + 2 * mo]
    lo = np.concatenate([s["lb"], s["lg"]])
    up = np.concatenate([s["ub"], s["ug"]])
    al = (s["maskl"] != 0) & np.isfinite(lo)
    au = (s["masku"] != 0) & np.isfinite(up)
    coef = np.where(al, lm[:mo], 0.0) - np.where(au, lm[mo:], 0.0)
    ct = np.zeros(nu + int(d.nx[n]))
    np.add.at(ct, s["idxb"], coef[:nb])
    if ng:
        ct += np.hstack([s["D"], s["C"]]).T @ coef[nb:]
    return ct[nu:]


def full_expand(qp, cmap, v, dlam, dt):
    """Full OCP (y, pi, lam, t) from the dense solution (condensing.py:343-429)."""
    from paper_2003_02547_b200.layout import OcpLayout

    d = qp.dim
    N = int(d.N)
    lay = OcpLayout(d)
    y = np.zeros(lay.ny)
    pi = np.zeros(lay.ne)
    lam = np.zeros(lay.nc)
    t = np.zeros(lay.nc)
    x = cmap["x0hat"].copy() if not cmap["keep_x0"] else v[: cmap["nx0"]].copy()
    xs = [x]
    for n in range(N + 1):
        nu = int(d.nu[n])
        u = v[cmap["u_off"][n]: cmap["u_off"][n] + nu] if nu else np.zeros(0)
        y[lay.u_off[n]: lay.u_off[n] + nu] = u
        y[lay.x_off[n]: lay.x_off[n] + int(d.nx[n])] = xs[n]
        if n < N:
            dyn = qp._dyn[n]
            xs.append(dyn["A"] @ xs[n] + dyn["B"] @ u + dyn["b"])
    mc = len(cmap["rows"])
    for r, (n, src) in enumerate(cmap["rows"]):
        mo = int(d.nb[n] + d.ng[n])
        c0 = lay.c_off[n]
        lam[c0 + src], lam[c0 + mo + src] = dlam[r], dlam[mc + r]
        t[c0 + src], t[c0 + mo + src] = dt[r], dt[mc + r]
    ctx = [_ctlam_x(qp, lam, lay, n) for n in range(N + 1)]
    for m in range(N, 0, -1):
        s = qp._stages[m]
        nu = int(d.nu[m])
        val = s["Q"] @ xs[m] + s["S"].T @ y[lay.u_off[m]: lay.u_off[m] + nu] + s["q"] - ctx[m]
        if m < N:
            val = val + qp._dyn[m]["A"].T @ pi[lay.pi_off[m]: lay.pi_off[m] + int(d.nx[m + 1])]
        pi[lay.pi_off[m - 1]: lay.pi_off[m - 1] + val.size] = val
    if cmap["fix"]:
        s = qp._stages[0]
        nu = int(d.nu[0])
        gap = s["Q"] @ xs[0] + s["S"].T @ y[lay.u_off[0]: lay.u_off[0] + nu] + s["q"] - ctx[0]
        if N >= 1:
            gap = gap + qp._dyn[0]["A"].T @ pi[lay.pi_off[0]: lay.pi_off[0] + int(d.nx[1])]
        mo = int(d.nb[0] + d.ng[0])
        for i, c in cmap["fix"]:
            if gap[c] >= 0.0:
                lam[lay.c_off[0] + i] = gap[c]
            else:
                lam[lay.c_off[0] + mo + i] = -gap[c]
    return y, pi, lam, t


def partial_condensed_qp(qp, N1):
    """(condensed OcpQp, blocks): partial_condense's stages assembled into an
    OcpQp of horizon N2 with the source terminal stage copied verbatim
    (condensing.py:530-550), ready for the C oracle's solve."""
    from paper_2003_02547_b200.qp_data import OcpQp, OcpQpDim

    stages, blocks = partial_condense(qp, N1)
    d = qp.dim
    N2 = len(stages)
    term = qp._stages[d.N]
    nx = [st["Q"].shape[0] for st in stages] + [int(d.nx[d.N])]
    nu = [st["R"].shape[0] for st in stages] + [0]
    nb = [len(st["idxb"]) for st in stages] + [int(d.nb[d.N])]
    ng = [st["C"].shape[0] for st in stages] + [int(d.ng[d.N])]
    q2 = OcpQp(OcpQpDim(N2, nx, nu, nb, ng))
    for k, st in enumerate(stages + [term]):
        for f in ("Q", "S", "R", "q", "r", "idxb", "lb", "ub", "C", "D", "lg", "ug",
                  "maskl", "masku"):
            q2.set_field(f, k, st[f])
        if k < N2:
            for f in ("A", "B", "b"):
                q2.set_field(f, k, st[f])
    return q2, blocks
