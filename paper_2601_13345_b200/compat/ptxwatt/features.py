"""ptxwatt.features (pkg/src/ptxwatt/features.py) -> K1b + K2."""
from paper_2601_13345_b200.api import coalescing_efficiency, dynamic_instruction_counts, extract_features  # noqa: F401
from paper_2601_13345_b200.model_types import KernelFeatures  # noqa: F401
