"""ptxwatt.alignment (pkg/src/ptxwatt/alignment.py) -> K1b."""
from paper_2601_13345_b200.api import analyze_memory_alignment  # noqa: F401
