"""B200-native structure-aware irregular-blocking sparse LU (arXiv 2512.04389).

Drop-in for the reference package ``lublock`` (pkg/src/lublock/__init__.py):
same public names.  The numerical factorization (``factorize``) runs as
hand-written sm_100a CUDA behind the C-ABI in include/lbk.h; the structure
path (symbolic, partition, dependency levels) runs natively on the host and
is bit-identical to the reference.
"""

from .blocking import (
    PANGULU_SIZES,
    BlockingPlan,
    irregular_plan,
    pangulu_size_select,
    regular_plan,
)
from .errors import (
    BadParams,
    DegenerateCurve,
    DegenerateMatrix,
    DeviceError,
    DimensionMismatch,
    EmptyMatrix,
    IndexOutOfRange,
    LuBlockError,
    MalformedEntry,
    MissingDiagonal,
    NonSquare,
    NotSymmetric,
    SupportViolation,
    UnsupportedField,
    ZeroPivot,
)
from .features import (
    DiagBlockPointer,
    PercentCurve,
    classify_curve,
    diag_block_pointer,
    percentage_curve,
)
from .grid import (
    GESSM,
    GETRF,
    SSSSM,
    TSTRF,
    BlockGrid,
    DependencyTree,
    SparseBlock,
    TaskView,
    dependency_levels,
    partition,
)
from .matrix_io import (
    CscMatrix,
    Triplet,
    csc_from_triplets,
    generate,
    read_matrix_market,
    write_curve_csv,
    write_plan_json,
    write_report_csv,
)
from .metrics import BalanceReport, block_nnz_stats, level_work_stats, makespan_model
from .numeric import (
    LUFactors,
    factor_diagonal,
    factor_l_panel,
    factor_u_panel,
    factorize,
    residual,
    schur_update,
    solve,
)
from .symbolic import FilledPattern, fill_ratio, symbolic_factorize, symmetrize_pattern

__version__ = "0.1.0"
