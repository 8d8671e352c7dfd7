"""B200-native sparse Gauss-Newton (SGN) search-direction path -- drop-in for sgnopt.

Re-exports the reference package's solver-path names (reference
pkg/src/sgnopt/__init__.py:9-93, hot-path subset) with identical signatures and
error behaviour; the numerics run in hand-written sm_100a CUDA (``_sgnb200.so``).
"""
from .errors import (CapabilityMissing, DeviceError, DimensionMismatch, ForwardSimFailure,
                     InfeasiblePoint, LineSearchFailure, MeritLineSearchFailure,
                     NegativeCurvature, NoConvergence, NonSquareParamJacobian,
                     NotPositiveDefinite, NumericalBlowup, SingularConstraintJacobian,
                     SingularMatrix, ToolkitError, TripletIndexError)
from .linear_solvers import (SolveReport, SparseFactorization, StabilizationConfig,
                             factor_sparse, solve_kkt_stabilized, stabilized_matrix)
from .sparse import (CscMatrix, TripletMatrix, csc_from_triplets, read_matrix_market, spmv,
                     spmv_transpose, stack_kkt_blocks, write_matrix_market)
from .sensitivity import (EquilibriumProblem, GnBlocks, KktSystem, adjoint_gradient, assemble_sgn,
                          gn_blocks, kkt_from_blocks, solve_block_gn)
from .optimize import (CSV_HEADER, METHODS, IterationRecord, OptimizerConfig, OptimizerRun,
                       SearchDirection, direction_bgn, direction_cg_gn, direction_dgn, direction_gd, direction_lbfgs,
                       direction_sgn, minimize,
                       project_direction_bounds)

__version__ = "0.1.0"
