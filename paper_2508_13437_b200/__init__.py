"""B200-native AMVM inner loop for the Discrete Min-Max Violation problem.

A drop-in for the ``solve()`` path of the reference ``dmmv`` package
(arXiv 2508.13437): the same problem construction, ``solve()``, seed and
iteration controls, and the same returned assignment, objective and trace —
with every ALNS iteration running on the GPU through libamvm.so
(include/amvm.h).  See DESIGN.md.
"""

__version__ = "0.1.0"

from .controller import (  # noqa: F401
    ACCEPT_TIE_TOL,
    LOCAL_SEARCH_MAX_ROUNDS,
    N_SEGMENT,
    ONE_OPT_MAX_SWEEPS,
    PAIRS,
    WEIGHT_FLOOR,
    OUTCOME_ACCEPTED,
    OUTCOME_IMPROVED,
    OUTCOME_NEW_BEST,
    OUTCOME_REJECTED,
    DestroySet,
    FilterConfig,
    OperatorBank,
    ImpactScores,
    SolveReport,
    SolverConfig,
    SwapCandidate,
    TraceEntry,
    accept,
    best_swap,
    find_candidates,
    greedy_repair,
    impact_scores,
    initial_solution,
    local_search,
    one_opt,
    random_destroy,
    random_repair,
    removal_count,
    select_operators,
    solve,
    update_weights,
    worst_remove_destroy,
)
from .exact import (  # noqa: F401
    DEFAULT_BUDGET,
    MAX_SWAP_CHECK_N,
    BudgetExceededError,
    OracleResult,
    SwapCheckReport,
    brute_force,
    exhaustive_swap_check,
    is_improving,
)
from .scoring import MoveScores, score_moves  # noqa: F401
from .formats import (  # noqa: F401
    InstanceParseError,
    RunArtifacts,
    export_lp,
    format_values,
    instance_to_text,
    read_instance,
    write_instance,
    write_run_artifacts,
    write_solution,
)
from .core import (  # noqa: F401
    REFRESH_PERIOD,
    Instance,
    RowScreen,
    Solution,
    ValueSet,
    apply_shift,
    apply_swap,
    compute_residual,
    round_to_nearest,
    row_screen,
    two_nearest,
)

__all__ = [
    "__version__", "Instance", "RowScreen", "Solution", "ValueSet", "compute_residual",
    "round_to_nearest", "row_screen", "two_nearest", "DestroySet", "ImpactScores", "FilterConfig",
    "SwapCandidate", "SolveReport", "SolverConfig", "TraceEntry", "best_swap", "find_candidates",
    "greedy_repair", "impact_scores", "initial_solution", "local_search", "one_opt",
    "random_destroy", "random_repair", "removal_count", "solve", "worst_remove_destroy",
    "DEFAULT_BUDGET", "BudgetExceededError", "OracleResult", "brute_force", "MAX_SWAP_CHECK_N",
    "SwapCheckReport", "exhaustive_swap_check", "is_improving",
    "InstanceParseError", "RunArtifacts", "export_lp", "format_values", "instance_to_text",
    "read_instance", "write_instance", "write_run_artifacts", "write_solution",
    "MoveScores", "score_moves", "apply_shift", "apply_swap", "OperatorBank", "select_operators",
    "update_weights", "accept", "OUTCOME_NEW_BEST", "OUTCOME_IMPROVED", "OUTCOME_ACCEPTED", "OUTCOME_REJECTED",
]
