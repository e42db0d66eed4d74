"""Value types of the analysis path.

Field names, order and equality semantics follow the reference so that code
written against ``ptxwatt`` keeps working (reference files, all under
pkg/src/ptxwatt/): ptx.py:45-96 (Instruction, PtxModule), cfg.py:15-54 (Loop,
ControlFlowGraph), features.py:23-52 (KernelFeatures), launch.py:11-38
(LaunchConfig, InputResources), time_model.py:20-30, power_model.py:16-28,
explorer.py:36-52 (Prediction, ParetoSet), calibration.py:43-83 (specs).

All of them are immutable.  Objects produced by the GPU lexer carry a hidden
``_dev`` handle (excluded from ``==``/``repr``) so later stages can reuse the
device-resident instruction records instead of re-lexing.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Any

OPCODE_CLASSES = ("MemLoad", "MemStore", "FP32", "INT", "SFU", "ALU", "Sync", "Branch", "Other")
STATE_SPACES = ("global", "shared", "local", "param", "reg", "none")
COMPUTE_UNITS = ("FP32", "INT", "SFU", "ALU")
UNIT_CLASSES = ("FP32", "INT", "SFU", "ALU", "Mem")

TYPE_BYTES = {
    "b8": 1, "s8": 1, "u8": 1,
    "b16": 2, "s16": 2, "u16": 2, "f16": 2, "bf16": 2,
    "b32": 4, "s32": 4, "u32": 4, "f32": 4,
    "b64": 8, "s64": 8, "u64": 8, "f64": 8,
}


@dataclass(frozen=True)
class Instruction:
    opcode: str
    opcode_class: str
    state_space: str
    operands: tuple[str, ...]
    predicate: str | None
    source_line: int

    @property
    def base(self) -> str:
        return self.opcode.partition(".")[0]

    @property
    def is_memory(self) -> bool:
        return self.opcode_class == "MemLoad" or self.opcode_class == "MemStore"

    @property
    def access_bytes(self) -> int:
        # last type suffix wins, default 4; times v2/v4 (ptx.py:64-76)
        elem, lanes = 4, 1
        for tok in self.opcode.split(".")[1:]:
            if tok in TYPE_BYTES:
                elem = TYPE_BYTES[tok]
            elif tok == "v2":
                lanes = 2
            elif tok == "v4":
                lanes = 4
        return elem * lanes

    @property
    def address_operand(self) -> str | None:
        return next((op for op in self.operands if op.startswith("[")), None)


@dataclass(frozen=True)
class PtxModule:
    kernel_name: str
    parameters: tuple[tuple[str, str, int], ...]
    registers_declared: dict[str, int]
    static_shared_bytes: int
    instructions: tuple[Instruction, ...]
    labels: dict[str, int]
    _dev: Any = field(default=None, compare=False, repr=False, hash=False)


@dataclass(frozen=True)
class Loop:
    header: int
    body: frozenset[int]
    trip: float | None = None
    header_label: str | None = None


@dataclass(frozen=True)
class ControlFlowGraph:
    blocks: tuple[tuple[int, int], ...]
    edges: tuple[tuple[int, int], ...]
    loops: tuple[Loop, ...]
    _dev: Any = field(default=None, compare=False, repr=False, hash=False)

    def block_of(self, instr_index: int) -> int:
        lo, hi = 0, len(self.blocks)
        while lo < hi:
            mid = (lo + hi) // 2
            start, end = self.blocks[mid]
            if instr_index < start:
                hi = mid
            elif instr_index >= end:
                lo = mid + 1
            else:
                return mid
        raise IndexError(f"instruction index {instr_index} outside all blocks")

    def block_weights(self) -> list[float]:
        out = [1.0] * len(self.blocks)
        for loop in self.loops:
            if loop.trip is None:
                raise ValueError("trip counts not estimated; run estimate_trip_counts first")
            for b in loop.body:
                out[b] *= loop.trip
        return out


@dataclass(frozen=True)
class KernelFeatures:
    n_mem: float
    n_comp_by_unit: dict[str, float]
    n_comp: float
    n_sync: float
    aligned_fraction: float
    eta_coal: float
    warps: int
    blocks_per_sm: float
    registers_per_thread: int
    shared_bytes: int
    mem_bytes: float

    def as_report_dict(self) -> dict:
        keys = ("n_mem", "n_comp_by_unit", "n_comp", "n_sync", "aligned_fraction", "eta_coal",
                "warps", "blocks_per_sm", "registers_per_thread", "shared_bytes", "mem_bytes")
        out = {k: getattr(self, k) for k in keys}
        out["n_comp_by_unit"] = dict(self.n_comp_by_unit)
        return out


@dataclass(frozen=True, order=True)
class LaunchConfig:
    block_x: int
    block_y: int
    p_cap: float

    @property
    def threads(self) -> int:
        return self.block_x * self.block_y


@dataclass(frozen=True)
class InputResources:
    shared_mem_bytes: int
    grid_x: int = 1
    grid_y: int = 1
    grid_z: int = 1
    seq_len: int = 1
    batch: int = 1
    heads: int = 1

    @property
    def total_blocks(self) -> int:
        return self.grid_x * self.grid_y * self.grid_z


@dataclass(frozen=True)
class TimeBreakdown:
    mwp: float
    cwp: float
    bw_eff: float
    t_mem: float
    t_comp: float
    t_sync: float
    t_exec: float


@dataclass(frozen=True)
class PowerBreakdown:
    p_units: float
    p_shape: float
    p_mem: float
    p_sm: float
    p_dyn: float
    f_adj: float
    ci: float
    active_sms: int
    cap_limited: bool


@dataclass(frozen=True)
class Prediction:
    config: LaunchConfig
    time: TimeBreakdown
    power: PowerBreakdown
    e_pred: float


@dataclass(frozen=True)
class ParetoSet:
    entries: tuple[Prediction, ...]
    rho: float
    t_peak: float


@dataclass(frozen=True)
class ArchitectureSpec:
    name: str
    sm_count: int
    max_warps_per_sm: int
    max_shared_per_sm: int
    max_threads_per_block: int
    bw_max: float
    ipc: float
    f_base: float
    p_tdp: float
    p_static: float
    p_cap_min: float
    dvfs_exponent_k: int
    tau_short: float
    departure_delay: float
    t_barrier: float
    exec_cycles: dict[str, float]
    issue_cycles: dict[str, float]


@dataclass(frozen=True)
class CalibrationProfile:
    beta_u: dict[str, float]
    l_mem_coal: float
    l_mem_uncoal: float
    sm_power_alpha: float
    sm_power_beta: float
    sm_power_delta: float
    transient_ratio_r: float
    kappa: float
    lambda_: float
    p_base_shape: float
    p_mem_base: float
    time_weights: tuple[float, float, float] = (1.0, 1.0, 1.0)
    t_base: float = 0.0
    e_overhead: float = 0.0
