"""ptxwatt.launch (pkg/src/ptxwatt/launch.py)."""
from paper_2601_13345_b200.api import RESOURCE_RULES, compute_input_resources  # noqa: F401
from paper_2601_13345_b200.model_types import InputResources, LaunchConfig  # noqa: F401
