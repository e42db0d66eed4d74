"""ptxwatt.power_model (pkg/src/ptxwatt/power_model.py) -> K3."""
from paper_2601_13345_b200.api import (  # noqa: F401
    activity_rate, compute_intensity, dvfs_frequency, dynamic_power, estimate_active_sms, memory_power, shape_power,
    sm_concurrency_power, transient_correction,
)
from paper_2601_13345_b200.model_types import PowerBreakdown  # noqa: F401
