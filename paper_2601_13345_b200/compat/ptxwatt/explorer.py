"""ptxwatt.explorer (pkg/src/ptxwatt/explorer.py) -> K2 + K3 + K4.  adaptive_power_cap (scalar feedback
formula, explorer.py:215-227) is out of scope for this path and not provided."""
from paper_2601_13345_b200.api import (  # noqa: F401
    evaluate_configs, generate_valid_configs, pareto_explore, pareto_explore_sweep, pareto_front, pareto_front_bruteforce,
    predict_energy,
)
from paper_2601_13345_b200.model_types import ParetoSet, Prediction  # noqa: F401


def adaptive_power_cap(p_hat: float, dp_history: float, a_coef: float, b_coef: float, p_tdp: float,
                       p_cap_min: float = 0.0) -> float:
    """explorer.py:215-227.  A scalar feedback rule (three flops per call, nothing data-parallel, SURVEY §2
    row 14): it lives in this import-path shim only, on the host, so that code importing it from
    ``ptxwatt`` keeps working.  Not part of the accelerated path and not counted by bench.py."""
    if p_hat < 0:
        raise ValueError(f"predicted power must be >= 0, got {p_hat}")
    wanted = a_coef * p_hat + b_coef * dp_history
    return max(p_cap_min, min(p_tdp, wanted))
