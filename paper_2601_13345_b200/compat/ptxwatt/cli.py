"""ptxwatt.cli (pkg/src/ptxwatt/cli.py): analyze / predict / explore."""
from paper_2601_13345_b200.cli import build_parser, main  # noqa: F401
