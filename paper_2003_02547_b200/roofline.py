"""Algorithmic work per QP-iteration for roofline reporting.

* ``factor_flops``: exactly the reference's nominal count of one classical
  ``riccati_factor`` (linalg.py:41-78 rules: potrf n^3//3, trsm n^2 m, gemm
  2mnk; kkt_ocp.py:142-251), e.g. 58,385 for config 0.
* ``solve_flops``: analytic count of one Riccati solve (kkt_ocp.py:254-320),
  sum_{n<N} (4 nx'^2 + 4 nx' nw + 2 nu^2 + 4 nu nx + 4 ng nw) + 2 nx0^2.
* ``residual_flops``: sum_n (2 nw^2 + 4 nx' nw + 4 ng nw).
* ``riccati_flops``: F_fac + 2 F_sol, the survey's recommended unit.
* ``stream_bytes``: data + 3 x factor workspace + 2 x iterate, the survey's
  streaming model of bytes per QP-iteration.
"""

from __future__ import annotations


def _stage(dim, n):
    nx = int(dim.nx[n]); nu = int(dim.nu[n]); ng = int(dim.ng[n]); nb = int(dim.nb[n])
    nxn = int(dim.nx[n + 1]) if n < dim.N else 0
    return nx, nu, ng, nb, nxn, nu + nx


def factor_flops(dim):
    f = 0
    for n in range(dim.N + 1):
        nx, nu, ng, nb, nxn, nw = _stage(dim, n)
        if ng:
            f += 2 * nw * nw * ng
        if n < dim.N:
            f += 2 * nxn * nw * nxn + 2 * nw * nw * nxn
        if nu:
            f += nu ** 3 // 3 + 2 * nu * nu * nx + 2 * nx * nx * nu
    nx0 = int(dim.nx[0])
    f += nx0 ** 3 // 3
    return f


def solve_flops(dim):
    f = 0
    for n in range(dim.N):
        nx, nu, ng, nb, nxn, nw = _stage(dim, n)
        f += 4 * nxn * nxn + 4 * nxn * nw + 2 * nu * nu + 4 * nu * nx + 4 * ng * nw
    f += 2 * int(dim.nx[0]) ** 2
    return f


def residual_flops(dim):
    f = 0
    for n in range(dim.N + 1):
        nx, nu, ng, nb, nxn, nw = _stage(dim, n)
        f += 2 * nw * nw + 4 * nxn * nw + 4 * ng * nw
    return f


def riccati_flops(dim):
    return factor_flops(dim) + 2 * solve_flops(dim)


def stream_bytes(dim, layout):
    data = sum(layout.field_len.values()) * 8
    work = 0
    for n in range(dim.N + 1):
        nx, nu, ng, nb, nxn, nw = _stage(dim, n)
        work += (nx * nx + nu * nx + nu * nu) * 8
    it = (layout.ny + layout.ne + 2 * layout.nc) * 8
    return data + 3 * work + 2 * it
