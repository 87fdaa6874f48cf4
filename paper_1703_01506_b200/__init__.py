"""B200-native max-null permutation testing (NaivePT / RapidPT hot path).

Drop-in for the reference package ``rapidmaxnull`` 0.1.0's engine entry
points: same names, signatures, return types and error contract, computed by
hand-written sm_100a CUDA kernels (librmx.so, include/rmx.h) instead of numpy.
PyTorch is used only for device memory and streams; there is no CPU fallback.
"""

__version__ = "0.1.0"

from .domain import (  # noqa: F401
    Basis,
    DataMatrix,
    MaxNull,
    ObservedColumn,
    PermutationPlan,
    RunConfig,
    StatMatrix,
    SubspaceModel,
    min_sample_rate,
    permute_columns,
    relabel,
)
from .exceptions import (  # noqa: F401
    DataFormatError,
    DegenerateVoxelError,
    EngineUnavailableError,
    IllConditionedBasisError,
    NumericalError,
    UsageError,
)
from .matfiles import (  # noqa: F401
    load_matrix,
    read_array,
    read_matrix,
    read_matrix_csv,
    write_array,
    write_matrix,
    write_matrix_csv,
)
from .naive_engine import (  # noqa: F401
    NaiveJob,
    NaiveResult,
    dump_statistic_matrix,
    run_naive,
    run_naive_ex,
    run_naive_mat0,
)
from .rapid_engine import (  # noqa: F401
    complete_column,
    fit_coefficients,
    init_basis,
    recover,
    run_rapid,
    solve_block,
    track_update,
    train,
    train_basis,
)
from .metrics import (  # noqa: F401
    HistogramPair,
    RiskResult,
    ThresholdRow,
    build_histogram_pair,
    kl_divergence,
    resampling_risk,
    threshold_table,
)
from .stats import (  # noqa: F401
    StatColumn,
    column_max,
    pvalue,
    reject_set,
    stat_map,
    threshold_at,
    tstat_full,
    tstat_subset,
)

__all__ = [
    "__version__", "Basis", "DataMatrix", "MaxNull", "ObservedColumn", "PermutationPlan",
    "RunConfig", "StatMatrix", "SubspaceModel", "min_sample_rate", "permute_columns", "relabel",
    "DataFormatError", "DegenerateVoxelError", "EngineUnavailableError",
    "IllConditionedBasisError", "NumericalError", "UsageError", "NaiveJob", "NaiveResult",
    "run_naive", "run_naive_ex", "run_naive_mat0", "dump_statistic_matrix", "column_max", "pvalue", "reject_set", "stat_map",
    "threshold_at", "tstat_full", "tstat_subset", "complete_column", "fit_coefficients",
    "init_basis", "recover", "run_rapid", "solve_block", "train", "train_basis",
    "track_update", "StatColumn", "HistogramPair", "RiskResult", "ThresholdRow",
    "build_histogram_pair", "kl_divergence", "resampling_risk", "threshold_table",
    "load_matrix", "read_array", "read_matrix", "read_matrix_csv", "write_array", "write_matrix",
    "write_matrix_csv",
]
