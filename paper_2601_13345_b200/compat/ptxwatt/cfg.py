"""ptxwatt.cfg (pkg/src/ptxwatt/cfg.py) -> K1b."""
from paper_2601_13345_b200.api import build_cfg, estimate_trip_counts  # noqa: F401
from paper_2601_13345_b200.model_types import ControlFlowGraph, Loop  # noqa: F401
