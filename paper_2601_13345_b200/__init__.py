"""B200-native implementation of FlipFlop's data-parallel analysis path (arXiv 2601.13345).

Drop-in names of the reference package ``ptxwatt`` are re-exported from ``api`` as they
come online; the tensor-level batched entry points live in ``engine`` / ``corpus``.
"""
from . import errors, model_types, specs  # noqa: F401
from .errors import *  # noqa: F401,F403
from .model_types import (  # noqa: F401
    ArchitectureSpec, CalibrationProfile, ControlFlowGraph, InputResources, Instruction,
    KernelFeatures, LaunchConfig, Loop, ParetoSet, PowerBreakdown, Prediction, PtxModule, TimeBreakdown,
)
from .specs import default_architecture, default_calibration, load_profile, save_profile  # noqa: F401

__version__ = "0.1.0"
