"""B200-native IHS-BIN ridge regularization path (arXiv 2210.12212).

The compute lives in ``libridgepath_b200.so`` (hand-written sm_100a CUDA +
C++ host orchestration behind the C ABI in include/ridgepath_b200.h);
``paper_2210_12212_b200.ridgepath`` mirrors the reference's ``ridgepath::``
API on top of it.
"""
from . import ridgepath  # noqa: F401
from .ridgepath import (  # noqa: F401
    BasisDivergedError,
    BinomialBasis,
    Context,
    Csr,
    FactorizationError,
    PathConfig,
    Preconditioner,
    RhoBounds,
    SketchSpec,
    SolverError,
    apply,
    apply_transpose,
    dual_path,
    gram_apply,
    ihs_basis,
    ihs_basis_matrix,
    ihs_bin_path,
    ihs_bin_path_matrix,
    ihs_compose,
    ihs_compose_matrix,
    interval_split,
    log_grid,
    sketch_apply,
    tune_interval,
)
