"""B200-native batched OCP-QP interior-point solver (HPIPM-paper path).

Drop-in for the reference package's optimal-control QP solve
(mpcqp.solve_ocp_qp, solver.py:103-105): the same ``OcpQpDim`` / ``OcpQp`` /
``IpmArg`` / ``QpSolution`` / ``SolveReport`` objects, solved by a fused
sm_100a fp64 kernel (residuals, Riccati factor/solve and the IPM vector
steps of every QP in one launch).  See DESIGN.md.
"""

from .batch import OcpQpBatch
from .condensing import (
    CondensingMap,
    PartialCondensingMap,
    condense,
    condense_batch,
    expand_batch,
    expand_solution,
    partial_condense,
    partial_condense_batch,
    partial_expand,
    partial_expand_batch,
)
from .errors import (
    ClosedLoopFailed,
    CondenseError,
    DimensionMismatch,
    FactorizationFailed,
    IndexOutOfRange,
    InvalidBlockSize,
    InvalidConfig,
    InvalidDim,
    MpcQpError,
    NativeLibraryError,
    NonPositiveIterate,
    NotPositiveDefinite,
    RankDeficient,
    SingularFactor,
    SingularSlackBlock,
    UnknownField,
)
from .dense import DenseQp, dense_to_ocp, ocp_to_dense, solve_dense_qp
from .ipm import IpmArg, IterRecord, SolverStats, Status, mode_preset
from .mpc import (
    ClosedLoopResult,
    MassSpringConfig,
    default_x0,
    gen_mass_spring,
    mass_spring_dynamics,
    run_closed_loop,
    run_closed_loop_batch,
    shift_guess,
)
from .layout import OcpLayout, QpResiduals, QpSolution
from .qp_data import OcpQp, OcpQpDim, Violation, validate
from .solver import (
    BatchReport,
    SolveReport,
    compute_residuals,
    newton_step,
    solve_ocp_qp,
    solve_ocp_qp_batch,
    solve_ocp_qp_host,
)

__version__ = "0.1.0"

__all__ = [
    "OcpQpBatch", "ClosedLoopFailed", "CondenseError", "DimensionMismatch", "FactorizationFailed",
    "IndexOutOfRange", "InvalidBlockSize", "InvalidConfig", "InvalidDim", "MpcQpError",
    "NativeLibraryError", "NonPositiveIterate", "NotPositiveDefinite", "RankDeficient",
    "SingularFactor", "SingularSlackBlock", "UnknownField", "IpmArg", "IterRecord",
    "SolverStats", "Status", "mode_preset", "OcpLayout", "QpResiduals", "QpSolution",
    "OcpQp", "OcpQpDim", "Violation", "validate", "BatchReport", "SolveReport",
    "compute_residuals", "newton_step", "solve_ocp_qp", "solve_ocp_qp_batch",
    "solve_ocp_qp_host", "PartialCondensingMap", "partial_condense", "partial_condense_batch",
    "partial_expand", "partial_expand_batch", "ClosedLoopResult", "MassSpringConfig",
    "default_x0", "gen_mass_spring", "mass_spring_dynamics", "run_closed_loop",
    "run_closed_loop_batch", "shift_guess", "CondensingMap", "condense", "condense_batch",
    "expand_batch", "expand_solution", "DenseQp", "dense_to_ocp", "ocp_to_dense", "solve_dense_qp",
    "__version__",
]
