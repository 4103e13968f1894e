"""Drop-in for the reference's `swarmplan` Python package
(/root/reference/proj/python/swarmplan/__init__.py:6-33): same names, backed
by this framework's C++ planning core. The GPU averaging round is
`swarmplan.AveragingRound` (paper_2106_10207_b200.round)."""
from paper_2106_10207_b200._swarmplan import (  # noqa: F401
    SpecParseError,
    __version__,
    assignment_json,
    build_plan,
    compare_strategies,
    expected_iterations,
    optimal_group_size,
    part_offsets,
    plan_parts,
    run_plan,
    simulate_averaging,
    solve_strategy,
    validate_spec,
)
from paper_2106_10207_b200.groups import run_plan_gpu  # noqa: F401
from paper_2106_10207_b200.round import AveragingRound  # noqa: F401


def run_training(scenario_json: str, hours: float = 0.0):
    """Out of scope: the churn simulator models whole training runs, not the
    averaging round."""
    raise NotImplementedError("run_training (churn simulation) is not part of this framework")


def check_bound(*args, **kwargs):
    """Out of scope: the SGD convergence harness."""
    raise NotImplementedError("check_bound (SGD harness) is not part of this framework")


__all__ = [
    "SpecParseError", "__version__", "assignment_json", "build_plan", "check_bound",
    "compare_strategies", "expected_iterations", "optimal_group_size", "run_training",
    "simulate_averaging", "solve_strategy", "validate_spec", "part_offsets", "plan_parts",
    "run_plan", "AveragingRound",
]
