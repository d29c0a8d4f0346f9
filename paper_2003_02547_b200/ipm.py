"""Solver configuration and outcome records of the drop-in API.

``IpmArg``, ``mode_preset``, ``Status``, ``IterRecord`` and ``SolverStats``
carry the same fields, defaults and preset values as the reference
(mpcqp/ipm_core.py:56-168, :171-198), so an ``arg`` built for the reference
means the same thing here.  The GPU path implements every preset's loop:
``speed`` (classical or square-root Riccati), ``balance`` / ``robust``
(per-stage and whole-factor QR array algorithm, regularised retry, iterative
refinement of the combined direction) and ``speed_abs`` (absolute
formulation, duality-measure exit).  ``speed`` with the classical variant runs
on the shaped kernels; the other settings on the generic kernel.
:func:`supported_reason` rejects only what the reference itself cannot run
(``comp_res_pred=False`` without the absolute formulation).
"""

from __future__ import annotations

import enum
from dataclasses import dataclass, field, replace

import numpy as np

__all__ = ["IpmArg", "Status", "SolverStats", "IterRecord", "mode_preset",
           "STATUS_CODES"]


class Status(enum.Enum):
    """Terminal state of a solve; numerical trouble is a status, not a raise."""

    Success = "Success"
    MaxIter = "MaxIter"
    MinStep = "MinStep"
    NaNDetected = "NaNDetected"
    Failure = "Failure"


# C ABI status words (include/ocpqp_b200.h) -> Status
STATUS_CODES = {0: Status.Success, 1: Status.MaxIter, 2: Status.MinStep,
                3: Status.NaNDetected, 4: Status.Failure}


@dataclass
class IpmArg:
    """Full algorithmic configuration of one solve (ipm_core.py:66-128)."""

    mode: str = "balance"
    iter_max: int = 30
    alpha_min: float = 1e-8
    mu0: float = 1e2
    tol_stat: float = 1e-8
    tol_eq: float = 1e-8
    tol_ineq: float = 1e-8
    tol_comp: float = 1e-8
    reg_prim: float = 0.0
    reg_dual: float = 0.0
    lam_min: float = 1e-16
    t_min: float = 1e-16
    t0: float = 1.0
    warm_start: str = "none"          # none | primal | primal_dual
    pred_corr: bool = True
    cond_pred_corr: bool = True
    corr_ratio: float = 1.5
    itref_corr_max: int = 0
    itref_pred_max: int = 0
    itref_stop_ratio: float = 1e-12
    qr_fallback_ratio: float = 1e-6
    use_qr_fallback: bool = False
    use_qr_always: bool = False
    comp_res_pred: bool = True
    abs_form: bool = False
    ftb: float = 0.995
    kkt_method: str = "schur"
    riccati_variant: str = "classical"

    def with_tol(self, tol):
        """Copy with all four exit tolerances set to ``tol``."""
        return replace(self, tol_stat=tol, tol_eq=tol, tol_ineq=tol, tol_comp=tol)

    def validate(self):
        for name in ("tol_stat", "tol_eq", "tol_ineq", "tol_comp"):
            if getattr(self, name) <= 0.0:
                raise ValueError(f"{name} must be > 0")
        if not 0.0 < self.alpha_min < 1.0:
            raise ValueError("alpha_min must lie in (0, 1)")
        if self.lam_min < 0.0 or self.t_min < 0.0:
            raise ValueError("lam_min and t_min must be >= 0")
        if self.warm_start not in ("none", "primal", "primal_dual"):
            raise ValueError(f"unknown warm_start '{self.warm_start}'")
        return self


# preset overrides (ipm_core.py:131-157)
_PRESETS = {
    "speed_abs": dict(abs_form=True, comp_res_pred=False, itref_corr_max=0,
                      itref_pred_max=0, use_qr_fallback=False, use_qr_always=False,
                      lam_min=1e-16, t_min=1e-16),
    "speed": dict(abs_form=False, comp_res_pred=True, itref_corr_max=0,
                  itref_pred_max=0, use_qr_fallback=False, use_qr_always=False,
                  lam_min=1e-16, t_min=1e-16),
    "balance": dict(abs_form=False, comp_res_pred=True, itref_corr_max=2,
                    itref_pred_max=0, use_qr_fallback=True, use_qr_always=False,
                    lam_min=1e-10, t_min=1e-10),
    "robust": dict(abs_form=False, comp_res_pred=True, itref_corr_max=4,
                   itref_pred_max=0, use_qr_fallback=True, use_qr_always=True,
                   lam_min=1e-10, t_min=1e-10),
}


def mode_preset(mode):
    """Pre-defined argument set for one of the four solver modes."""
    try:
        overrides = _PRESETS[mode]
    except KeyError:
        raise ValueError(
            f"unknown mode '{mode}'; expected one of {sorted(_PRESETS)}") from None
    return IpmArg(mode=mode, **overrides)


@dataclass
class IterRecord:
    """One row of the per-iteration trace (ipm_core.py:171-184)."""

    it: int
    alpha_aff: float
    alpha: float
    mu: float
    sigma: float
    res_g: float
    res_b: float
    res_d: float
    res_m: float


@dataclass
class SolverStats:
    """Outcome summary of one solve (ipm_core.py:186-198)."""

    status: Status
    iterations: int
    res_g: float = np.nan
    res_b: float = np.nan
    res_d: float = np.nan
    res_m: float = np.nan
    mu: float = np.nan
    flops: int = 0
    trace: list = field(default_factory=list)


def supported_reason(arg):
    """None when the GPU loop implements ``arg``; otherwise why not."""
    if not arg.comp_res_pred and not arg.abs_form:
        # the reference's loop reads res.r_g of a skipped residual evaluation
        # (solver.py:191-216) and fails
        return "comp_res_pred=False without the absolute formulation"
    if arg.riccati_variant not in ("classical", "square_root"):
        return f"riccati_variant '{arg.riccati_variant}'"
    return None


def is_speed_classical(arg):
    """The setting the shaped (compile-time stage shape) kernels implement."""
    return (not arg.abs_form and arg.comp_res_pred and arg.itref_corr_max <= 0
            and arg.itref_pred_max <= 0 and not arg.use_qr_always and not arg.use_qr_fallback
            and arg.riccati_variant == "classical")


def team_supports(arg, nw=None, nx=None):
    """The settings the shaped team kernel runs (ocpqp_capi.cu team_supports):
    the delta form with per-iteration residuals (speed, balance -- QR rungs
    escape per QP to the generic kernel; robust where the stacked factor of
    nw + nx rows fits one warp) or the speed_abs combination."""
    delta = not arg.abs_form and arg.comp_res_pred
    abs_speed = (arg.abs_form and not arg.comp_res_pred and arg.itref_corr_max <= 0
                 and not arg.use_qr_fallback)
    variant_ok = arg.riccati_variant == "classical" or (
        arg.riccati_variant == "square_root" and nw is not None and nw <= 32)
    qr_ok = (not arg.use_qr_always) or (
        delta and nw is not None and nx is not None and nw + nx <= 32
        and arg.riccati_variant == "classical")
    return ((delta or abs_speed) and qr_ok and variant_ok
            and arg.itref_pred_max <= 0)
