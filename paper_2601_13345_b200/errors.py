"""Exception names of the reference package, kept so callers can switch without
touching their ``except`` clauses (reference: pkg/src/ptxwatt/errors.py:11-138).

The C-ABI reports integer status codes (include/ffb.h, ``FFB_E_*``); ``raise_for_status``
maps them 1:1 onto these classes.  Exit codes follow the reference CLI convention:
input problems 2, model problems 3.
"""
from __future__ import annotations


class PtxWattError(Exception):
    exit_code = 3


class InputError(PtxWattError):
    exit_code = 2


class ModelError(PtxWattError):
    exit_code = 3


def _mk(name: str, base: type, doc: str) -> type:
    cls = type(name, (base,), {"__doc__": doc, "__module__": __name__})
    globals()[name] = cls
    return cls


_INPUT = {
    "MalformedPtx": "Unbalanced braces, branch to an undefined label, or empty kernel body.",
    "NoKernelFound": "No .entry in the source, or the named kernel is absent.",
    "AnnotationForUnknownLoop": "Trip annotation names a label that heads no loop.",
    "InvalidConfig": "Launch config breaks warp alignment or an architecture limit.",
    "SchemaViolation": "Profile / measurement file failed validation (message has the field path).",
    "SharedMemOverflow": "Workload wants more shared memory per block than one SM has.",
    "EmptyTrace": "Power trace without samples.",
    "ZeroBaseline": "Relative-change metric with a non-positive baseline.",
    "RecommendedExceedsTotal": "More recommended configs than candidates.",
    "NonpositiveInput": "Greenup/speedup/powerup inputs must be positive.",
    "LengthMismatch": "Rank-correlation inputs differ in length or are too short.",
    "DegenerateConstantInput": "Rank correlation undefined for a constant input.",
}
_MODEL = {
    "NegativeDelta": "Saturated power below idle power.",
    "ZeroRate": "Non-positive peak operation rate.",
    "ZeroSustained": "Non-positive sustained power in a transient pair.",
    "FitDiverged": "Least-squares iteration went non-finite.",
    "InsufficientSamples": "Too few distinct samples for the power law.",
    "InsufficientVariation": "Shape sweep lacks aspect-ratio / coalescing variation.",
    "ZeroDelay": "Non-positive departure delay.",
    "ZeroComputeCycles": "Zero compute cycles in CWP.",
    "ZeroBandwidth": "Effective bandwidth is zero while memory work remains.",
    "ZeroCycles": "Non-positive exec or issue cycles.",
    "CapAboveTdp": "Power cap above TDP, or non-positive.",
    "EmptyGrid": "Grid with zero blocks.",
    "NoFeasibleConfig": "Every candidate configuration was filtered out.",
}
for _n, _d in _INPUT.items():
    _mk(_n, InputError, _d)
for _n, _d in _MODEL.items():
    _mk(_n, ModelError, _d)


class NativeLibraryMissing(PtxWattError):
    """The CUDA extension (libffb.so) or a CUDA device is not available.

    There is no CPU path in this package: every analysis entry point runs on the GPU.
    """


class CapacityExceeded(PtxWattError):
    """A documented device-side capacity (line length, front size, blocks per kernel) was hit."""


# status code -> exception class; order mirrors include/ffb.h
STATUS_TABLE = {
    1: MalformedPtx,            # FFB_E_MALFORMED_PTX   # noqa: F821
    2: NoKernelFound,           # FFB_E_NO_KERNEL       # noqa: F821
    3: InvalidConfig,           # FFB_E_INVALID_CONFIG  # noqa: F821
    4: NoFeasibleConfig,        # FFB_E_NO_FEASIBLE     # noqa: F821
    5: EmptyGrid,               # FFB_E_EMPTY_GRID      # noqa: F821
    6: ZeroDelay,               # FFB_E_ZERO_DELAY      # noqa: F821
    7: ZeroComputeCycles,       # FFB_E_ZERO_COMPUTE    # noqa: F821
    8: ZeroBandwidth,           # FFB_E_ZERO_BANDWIDTH  # noqa: F821
    9: ZeroCycles,              # FFB_E_ZERO_CYCLES     # noqa: F821
    10: CapAboveTdp,            # FFB_E_CAP_ABOVE_TDP   # noqa: F821
    11: CapacityExceeded,       # FFB_E_CAPACITY
    12: NativeLibraryMissing,   # FFB_E_CUDA
    13: ValueError,             # FFB_E_BAD_ARGUMENT
}


def raise_for_status(code: int, what: str = "") -> None:
    if code == 0:
        return
    exc = STATUS_TABLE.get(code, PtxWattError)
    raise exc(f"{what} (native status {code})" if what else f"native status {code}")
