"""B200-native implementation of FlipFlop's data-parallel analysis path (arXiv 2601.13345).

Drop-in names of the reference package ``ptxwatt`` (pkg/src/ptxwatt/__init__.py:4-55) for the
analysis path, computed by hand-written sm_100a kernels behind a C-ABI (include/ffb.h);
the batched tensor-level entry points live in ``engine`` (grid, skyline) and ``corpus``
(lexer, dataflow).  There is no CPU path: without libffb.so and a CUDA device every entry
point raises ``NativeLibraryMissing``.
"""
from . import errors, model_types, specs  # noqa: F401
from .errors import *  # noqa: F401,F403
from .model_types import (  # noqa: F401
    OPCODE_CLASSES, STATE_SPACES, ArchitectureSpec, CalibrationProfile, ControlFlowGraph, InputResources,
    Instruction, KernelFeatures, LaunchConfig, Loop, ParetoSet, PowerBreakdown, Prediction, PtxModule, TimeBreakdown,
)
from .specs import (  # noqa: F401
    default_architecture, default_calibration, load_architecture, load_profile, save_profile,
)
from .api import (  # noqa: F401
    activity_rate, analyze_memory_alignment, build_cfg, classify_opcode, coalescing_efficiency,
    compute_input_resources, compute_intensity, cwp, dvfs_frequency, dynamic_instruction_counts, dynamic_power,
    estimate_active_sms, estimate_trip_counts, evaluate_configs, execution_time, extract_features,
    generate_valid_configs, memory_power, mwp, pareto_explore, pareto_explore_sweep, pareto_front, pareto_front_bruteforce, parse_ptx,
    predict_energy, shape_power, sm_concurrency_power, transient_correction, wave_count,
)

__version__ = "0.1.0"
