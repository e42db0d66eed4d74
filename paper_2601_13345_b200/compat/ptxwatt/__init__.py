"""`ptxwatt` import path over paper_2601_13345_b200 (see paper_2601_13345_b200/compat/__init__.py)."""
from paper_2601_13345_b200 import *  # noqa: F401,F403
from paper_2601_13345_b200 import __version__  # noqa: F401
from . import alignment, calibration, cfg, errors, explorer, features, launch, power_model, ptx, time_model  # noqa: F401
from .explorer import adaptive_power_cap  # noqa: E402,F401
