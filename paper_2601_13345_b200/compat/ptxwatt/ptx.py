"""ptxwatt.ptx (pkg/src/ptxwatt/ptx.py) -> GPU lexer / classifier."""
from paper_2601_13345_b200.api import classify_opcode, parse_ptx  # noqa: F401
from paper_2601_13345_b200.model_types import OPCODE_CLASSES, STATE_SPACES, Instruction, PtxModule  # noqa: F401
