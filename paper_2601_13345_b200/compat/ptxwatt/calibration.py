"""ptxwatt.calibration: the carrier half (calibration.py:43-134, 323-538).  The fitting routines
(calibration.py:137-320) are out of scope for this path and not provided."""
from paper_2601_13345_b200.model_types import UNIT_CLASSES, ArchitectureSpec, CalibrationProfile  # noqa: F401
from paper_2601_13345_b200.specs import (  # noqa: F401
    architecture_from_dict, architecture_to_dict, calibration_from_dict, calibration_to_dict, default_architecture,
    default_calibration, load_architecture, load_profile, load_profiles, save_profile,
)
