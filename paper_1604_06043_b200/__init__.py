"""B200-native M(s,l)stab / IDR(s)stab(l) solve loop (arXiv 1604.06043), drop-in for the
reference's proj/core solver path. See DESIGN.md and INTEGRATION.md."""
from .mstab import (  # noqa: F401
    BREAKDOWN, CONVERGED, MAXMV, BreakdownError, ConfigError, Context, CsrMatrix, CsrOperator, CudaError,
    DimensionMismatch, Error, FetchPolicy, FingerprintMismatch, HistoryPoint, IoError, NotReal, ParseError,
    RankDeficient, RecycleData, SingularProjection, SolveReport, SolveResult, SolverConfig, StaleData,
    TorchHostComm, ValidationReport, arnoldi_init, default_context, fetch, idrstab_solve, least_squares_tall, load,
    make_cut_space, mstab_solve, save, solve_small, validate, PrecondKind, SplitPreconditioner,
    PreconditionedOperator, ZeroPivot, build_ilu0, build_jacobi, build_none, preconditioned_rhs,
    unpreconditioned_solution, MissingOmegas, sridr_solve, bicg_solve, bicgstab_solve, gmres_solve,
    IterationState, PolyOut, arnoldi_init_draws, distributed_fingerprint, local_col_span, bicg_projection, level_iteration, poly_combination)
from ._capi import Lib, PRODUCT_LIB  # noqa: F401
