"""B200-native D-NGD step (arXiv 2505.21404) behind the reference `dngd` API.

Drop-in for the hot path of the reference package: the step solvers
(`dense_dual_solve`, `pcg_step`, `assemble_gramian`, `kvp`, `nystrom_build`,
`precond_apply`), the residual-map plugin (`ResidualMap`, `PinnResidualMap`,
`LinearResidualMap`, `RegressionResidualMap`), the outer loop
(`OptimizerConfig`, `dngd_run`, `dngd_minimize`, `line_search`, `lm_damping`)
and the problem plugins.  All numerics run in libdngd_b200.so (hand-written
sm_100a CUDA behind the C ABI in include/dngd_b200.h); there is no CPU
fallback.  Importing this package does not touch the GPU; the first numeric
call does.
"""

from .errors import (
    ConfigError,
    DimensionError,
    DngdError,
    DomainError,
    FactorizationError,
    NonFiniteError,
)
from .model import MlpSpec, OutputTransform, init_params, point_columns, xavier_normal_params
from .optimizer import (
    LineSearchResult,
    OptimizerConfig,
    TraceRow,
    TrainTrace,
    device_line_search,
    dngd_minimize,
    dngd_run,
    line_search,
    lm_damping,
    network_values,
    primal_ga_correction,
    primal_gn_solve,
    relative_l2_error,
    timing_sweep,
)
from .params import ParameterLayout, ParameterVector
from .problems import (
    PROBLEMS,
    AllenCahn,
    Heat,
    Heat1d,
    PdeProblem,
    Poisson2d,
    Poisson10d,
    PoissonBallStde,
    PoissonSin,
    build_map,
    eval_residuals,
    make_problem,
    sample_collocation,
)
from .residuals import (
    BOUNDARY,
    INITIAL,
    INTERIOR,
    CollocationClass,
    CollocationSet,
    IcShiftResidualMap,
    LinearResidualMap,
    PinnResidualMap,
    RegressionResidualMap,
    ResidualBatch,
    ResidualMap,
)
from .solver import (
    GA_NORM_GUARD,
    GA_RATIO_MAX,
    GRAMIAN_MEMORY_BUDGET,
    DualOperator,
    GramianMatrix,
    NystromPreconditioner,
    StepResult,
    assemble_gramian,
    dense_dual_solve,
    kernel_entry,
    kvp,
    nystrom_build,
    pcg_step,
    precond_apply,
)

__version__ = "0.1.0"
