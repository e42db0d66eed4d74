"""Import-path compatibility with the reference package.

``sys.path.insert(0, paper_2601_13345_b200.compat.PATH); import ptxwatt`` gives a package named
``ptxwatt`` whose submodules (``ptxwatt.ptx``, ``.cfg``, ``.alignment``, ``.features``, ``.launch``,
``.time_model``, ``.power_model``, ``.explorer``, ``.calibration``, ``.errors``, ``.cli``) resolve to
the CUDA-backed drop-ins, so code and tests written against the reference's import paths
(pkg/src/ptxwatt/__init__.py:4-55, pkg/tests/*.py) run unchanged.  Names of the reference that are
out of scope for this path (calibration fitting, metrics, adaptive_power_cap; SURVEY §2 rows
10, 11, 14) are not provided.
"""
from pathlib import Path

PATH = str(Path(__file__).resolve().parent)
