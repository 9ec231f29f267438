"""B200-native generalized DWD solver (inexact sGS-ADMM, arXiv 2305.12019).

Drop-in for the reference package ``gdwd`` on its hot path: the same
``sgs_admm_solve(data, config, meta=None, callback=None)`` entry point and
records, with every iteration running in ``libgdwd_b200.so`` (hand-written
sm_100a CUDA behind the C ABI in include/gdwd_b200.h).  There is no CPU
fallback.
"""

from .model import FeatureMeta, ModelFile, identity_meta
from .solver import (
    Backend,
    DegenerateSchurError,
    DeviceProblem,
    IndefiniteMatrixError,
    KKTResiduals,
    LanczosConvergenceError,
    ProblemData,
    SingleClassError,
    SolveResult,
    SolverConfig,
    SolverKind,
    SolverState,
    as_problem,
    compute_weights,
    device_problem,
    dual_objective,
    kkt_residuals,
    matvec,
    primal_objective,
    newton_r,
    newton_r_sweep,
    scale_problem,
    select_solver,
    sgs_admm_solve,
    update_sigma,
)
from .sparse import SparseFormatError, SparseMatrixCSC, csc_from_dense, csc_from_triplets
from .scoring import decision_values, predict, train_error
from .penalty import compute_penalty_C
from .ingest import ModelFormatError, ParseError, RawDataset, parse_libsvm, preprocess, read_model, write_model

__version__ = "0.1.0"

__all__ = [
    "Backend", "DegenerateSchurError", "DeviceProblem", "FeatureMeta", "IndefiniteMatrixError", "KKTResiduals",
    "LanczosConvergenceError", "ModelFile", "ProblemData", "SingleClassError", "SolveResult", "SolverConfig",
    "SolverKind", "SolverState", "SparseFormatError", "as_problem", "SparseMatrixCSC", "compute_weights", "csc_from_dense",
    "csc_from_triplets", "device_problem", "identity_meta", "matvec", "newton_r", "newton_r_sweep",
    "scale_problem", "select_solver", "sgs_admm_solve", "update_sigma", "decision_values", "predict",
    "train_error", "compute_penalty_C", "kkt_residuals", "primal_objective", "dual_objective", "ModelFormatError",
    "ParseError", "RawDataset", "parse_libsvm", "preprocess", "read_model", "write_model",
]
