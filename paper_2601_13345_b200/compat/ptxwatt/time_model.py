"""ptxwatt.time_model (pkg/src/ptxwatt/time_model.py) -> K3."""
from paper_2601_13345_b200.api import cwp, execution_time, mwp, wave_count  # noqa: F401
from paper_2601_13345_b200.model_types import TimeBreakdown  # noqa: F401
