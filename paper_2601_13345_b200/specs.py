"""GPU-spec and calibration carriers: built-in synthetic part, JSON (de)serialisation
with field-path errors, and the packed fp64 row each spec becomes on the device.

Reference behaviour followed: calibration.py:94-134 (built-in 48-SM part and its
placeholder coefficients), :332-478 (schema rules), :500-538 (load/save, sorted
keys, round trip is the identity).  The fitting routines (calibration.py:137-320)
are out of scope for this path.

``pack_spec`` is new: it flattens (ArchitectureSpec, CalibrationProfile) into the
``FFB_SPEC_*`` fp64 row consumed by ``ffb_predict_grid`` (include/ffb.h).
"""
from __future__ import annotations

import json
import math
from pathlib import Path

from .errors import SchemaViolation  # type: ignore[attr-defined]
from .model_types import UNIT_CLASSES, ArchitectureSpec, CalibrationProfile


def default_architecture() -> ArchitectureSpec:
    units = dict(zip(UNIT_CLASSES, (4.0, 4.0, 16.0, 2.0, 400.0)))
    issue = dict(zip(UNIT_CLASSES, (1.0, 1.0, 4.0, 1.0, 4.0)))
    return ArchitectureSpec(
        name="synthetic-48sm", sm_count=48, max_warps_per_sm=48, max_shared_per_sm=49152,
        max_threads_per_block=1024, bw_max=448e9, ipc=4.0, f_base=1.5e9, p_tdp=250.0,
        p_static=40.0, p_cap_min=100.0, dvfs_exponent_k=3, tau_short=1e-5,
        departure_delay=40.0, t_barrier=1e-7, exec_cycles=units, issue_cycles=issue,
    )


def default_calibration() -> CalibrationProfile:
    return CalibrationProfile(
        beta_u=dict(zip(UNIT_CLASSES, (2e-3, 1.5e-3, 4e-3, 1e-3, 6e-3))),
        l_mem_coal=400.0, l_mem_uncoal=800.0,
        sm_power_alpha=2.2, sm_power_beta=0.75, sm_power_delta=32.0,
        transient_ratio_r=0.833, kappa=0.12, lambda_=0.3,
        p_base_shape=12.0, p_mem_base=18.0,
        time_weights=(1.0, 1.0, 1.0), t_base=2e-6, e_overhead=1e-4,
    )


# ---------------------------------------------------------------- JSON schema

_ARCH_POSITIVE = (
    "sm_count", "max_warps_per_sm", "max_shared_per_sm", "max_threads_per_block",
    "bw_max", "ipc", "f_base", "p_tdp", "p_static", "dvfs_exponent_K",
    "tau_short", "departure_delay", "t_barrier",
)
_ARCH_INTS = ("sm_count", "max_warps_per_sm", "max_shared_per_sm", "max_threads_per_block")
_CAL_NONNEG = ("sm_power_alpha", "sm_power_delta", "p_base_shape", "p_mem_base", "t_base", "e_overhead")


def _is_num(v) -> bool:
    return isinstance(v, (int, float)) and not isinstance(v, bool) and math.isfinite(v)


def _get(obj: dict, key: str, where: str):
    if key not in obj:
        raise SchemaViolation(f"{where}.{key}: missing")
    return obj[key]


def _num(obj: dict, key: str, where: str) -> float:
    v = _get(obj, key, where)
    if not _is_num(v):
        raise SchemaViolation(f"{where}.{key}: must be a finite number")
    return float(v)


def _unit_map(obj: dict, key: str, where: str, *, strictly_positive: bool, what: str) -> dict[str, float]:
    raw = _get(obj, key, where)
    if not isinstance(raw, dict):
        raise SchemaViolation(f"{where}.{key}: must be a mapping of unit class to {what}")
    out = {}
    for unit in UNIT_CLASSES:
        v = _num(raw, unit, f"{where}.{key}")
        if strictly_positive and v <= 0:
            raise SchemaViolation(f"{where}.{key}.{unit}: must be > 0")
        if not strictly_positive and v < 0:
            raise SchemaViolation(f"{where}.{key}.{unit}: must be >= 0")
        out[unit] = v
    return out


def architecture_from_dict(obj, path: str = "architecture") -> ArchitectureSpec:
    if not isinstance(obj, dict):
        raise SchemaViolation(f"{path}: must be an object")
    name = _get(obj, "name", path)
    if not isinstance(name, str) or not name:
        raise SchemaViolation(f"{path}.name: must be a non-empty string")
    nums = {k: _num(obj, k, path) for k in _ARCH_POSITIVE}
    for k, v in nums.items():
        if v <= 0:
            raise SchemaViolation(f"{path}.{k}: must be > 0")
    cap_min = _num(obj, "p_cap_min", path)
    if not 0 <= cap_min <= nums["p_tdp"]:
        raise SchemaViolation(f"{path}.p_cap_min: must be in [0, p_tdp]")
    k_exp = nums["dvfs_exponent_K"]
    if k_exp != int(k_exp) or int(k_exp) < 1:
        raise SchemaViolation(f"{path}.dvfs_exponent_K: must be a positive integer")
    ex = _unit_map(obj, "exec_cycles", path, strictly_positive=True, what="cycles")
    iss = _unit_map(obj, "issue_cycles", path, strictly_positive=True, what="cycles")
    return ArchitectureSpec(
        name=name, **{k: int(nums[k]) for k in _ARCH_INTS},
        bw_max=nums["bw_max"], ipc=nums["ipc"], f_base=nums["f_base"], p_tdp=nums["p_tdp"],
        p_static=nums["p_static"], p_cap_min=cap_min, dvfs_exponent_k=int(k_exp),
        tau_short=nums["tau_short"], departure_delay=nums["departure_delay"],
        t_barrier=nums["t_barrier"], exec_cycles=ex, issue_cycles=iss,
    )


def architecture_to_dict(arch: ArchitectureSpec) -> dict:
    d = {k: getattr(arch, k) for k in (
        "name", *_ARCH_INTS, "bw_max", "ipc", "f_base", "p_tdp", "p_static", "p_cap_min",
        "tau_short", "departure_delay", "t_barrier")}
    d["dvfs_exponent_K"] = arch.dvfs_exponent_k
    d["exec_cycles"] = dict(arch.exec_cycles)
    d["issue_cycles"] = dict(arch.issue_cycles)
    return d


def calibration_from_dict(obj, path: str = "calibration") -> CalibrationProfile:
    if not isinstance(obj, dict):
        raise SchemaViolation(f"{path}: must be an object")
    beta = _unit_map(obj, "beta_u", path, strictly_positive=False, what="W/(op/s)")
    l_coal, l_uncoal = _num(obj, "l_mem_coal", path), _num(obj, "l_mem_uncoal", path)
    if l_coal < 0:
        raise SchemaViolation(f"{path}.l_mem_coal: must be >= 0")
    if l_uncoal < l_coal:
        raise SchemaViolation(f"{path}.l_mem_uncoal: must be >= l_mem_coal")
    r = _num(obj, "transient_ratio_r", path)
    if not 0 < r <= 1:
        raise SchemaViolation(f"{path}.transient_ratio_r: must be in (0, 1]")
    kappa, lam = _num(obj, "kappa", path), _num(obj, "lambda", path)
    if kappa < 0:
        raise SchemaViolation(f"{path}.kappa: must be >= 0")
    if lam < 0:
        raise SchemaViolation(f"{path}.lambda: must be >= 0")
    nn = {}
    for k in _CAL_NONNEG:
        nn[k] = _num(obj, k, path)
        if nn[k] < 0:
            raise SchemaViolation(f"{path}.{k}: must be >= 0")
    sm_beta = _num(obj, "sm_power_beta", path)
    w = _get(obj, "time_weights", path)
    if not isinstance(w, (list, tuple)) or len(w) != 3 or any((not _is_num(x)) or x < 0 for x in w):
        raise SchemaViolation(f"{path}.time_weights: must be three numbers >= 0")
    return CalibrationProfile(
        beta_u=beta, l_mem_coal=l_coal, l_mem_uncoal=l_uncoal,
        sm_power_alpha=nn["sm_power_alpha"], sm_power_beta=sm_beta, sm_power_delta=nn["sm_power_delta"],
        transient_ratio_r=r, kappa=kappa, lambda_=lam,
        p_base_shape=nn["p_base_shape"], p_mem_base=nn["p_mem_base"],
        time_weights=tuple(float(x) for x in w), t_base=nn["t_base"], e_overhead=nn["e_overhead"],
    )


def calibration_to_dict(profile: CalibrationProfile) -> dict:
    d = {k: getattr(profile, k) for k in (
        "l_mem_coal", "l_mem_uncoal", "sm_power_alpha", "sm_power_beta", "sm_power_delta",
        "transient_ratio_r", "kappa", "p_base_shape", "p_mem_base", "t_base", "e_overhead")}
    d["beta_u"] = dict(profile.beta_u)
    d["lambda"] = profile.lambda_
    d["time_weights"] = list(profile.time_weights)
    return d


def _read_json(path) -> object:
    try:
        return json.loads(Path(path).read_text())
    except json.JSONDecodeError as exc:
        raise SchemaViolation(f"{path}: not valid JSON ({exc})") from exc


def load_profile(path) -> tuple[ArchitectureSpec, CalibrationProfile]:
    obj = _read_json(path)
    if not isinstance(obj, dict):
        raise SchemaViolation(f"{path}: top level must be an object")
    return (architecture_from_dict(_get(obj, "architecture", str(path))),
            calibration_from_dict(_get(obj, "calibration", str(path))))


def load_architecture(path) -> ArchitectureSpec:
    obj = _read_json(path)
    if isinstance(obj, dict) and "architecture" in obj:
        return architecture_from_dict(obj["architecture"])
    return architecture_from_dict(obj if isinstance(obj, dict) else {})


def save_profile(path, arch: ArchitectureSpec, profile: CalibrationProfile) -> None:
    payload = {"architecture": architecture_to_dict(arch), "calibration": calibration_to_dict(profile)}
    architecture_from_dict(payload["architecture"])   # a saved file must load
    calibration_from_dict(payload["calibration"])
    Path(path).write_text(json.dumps(payload, indent=2, sort_keys=True) + "\n")


# ---------------------------------------------------------------- device row

# Column order of one spec row; must match enum FfbSpecCol in include/ffb.h.
SPEC_COLUMNS = (
    "sm_count", "max_warps_per_sm", "max_shared_per_sm", "max_threads_per_block",
    "bw_max", "ipc", "f_base", "p_tdp", "p_static", "p_cap_min", "dvfs_exponent_k",
    "tau_short", "departure_delay", "t_barrier",
    "exec_FP32", "exec_INT", "exec_SFU", "exec_ALU", "exec_Mem",
    "issue_FP32", "issue_INT", "issue_SFU", "issue_ALU", "issue_Mem",
    "beta_FP32", "beta_INT", "beta_SFU", "beta_ALU", "beta_Mem",
    "l_mem_coal", "l_mem_uncoal", "sm_power_alpha", "sm_power_beta", "sm_power_delta",
    "transient_ratio_r", "kappa", "lambda", "p_base_shape", "p_mem_base",
    "w_mem", "w_comp", "w_sync", "t_base", "e_overhead",
    "regs_per_sm",      # extension: 0 = no register limit = reference behaviour
)
SPEC_WIDTH = 48  # padded row width in doubles


def pack_spec(arch: ArchitectureSpec, profile: CalibrationProfile, regs_per_sm: int = 0) -> list[float]:
    row = [
        arch.sm_count, arch.max_warps_per_sm, arch.max_shared_per_sm, arch.max_threads_per_block,
        arch.bw_max, arch.ipc, arch.f_base, arch.p_tdp, arch.p_static, arch.p_cap_min,
        arch.dvfs_exponent_k, arch.tau_short, arch.departure_delay, arch.t_barrier,
        *(arch.exec_cycles[u] for u in UNIT_CLASSES),
        *(arch.issue_cycles[u] for u in UNIT_CLASSES),
        *(profile.beta_u[u] for u in UNIT_CLASSES),
        profile.l_mem_coal, profile.l_mem_uncoal, profile.sm_power_alpha, profile.sm_power_beta,
        profile.sm_power_delta, profile.transient_ratio_r, profile.kappa, profile.lambda_,
        profile.p_base_shape, profile.p_mem_base, *profile.time_weights, profile.t_base,
        profile.e_overhead, regs_per_sm,
    ]
    assert len(row) == len(SPEC_COLUMNS)
    row = [float(x) for x in row]
    return row + [0.0] * (SPEC_WIDTH - len(row))


# ---------------------------------------------------------------- spec directories

SPEC_DIR = Path(__file__).resolve().parent / "spec_files"


def load_regs_per_sm(path) -> int:
    """Optional ``extensions.regs_per_sm`` of a profile file (the reference's loader ignores
    unknown keys, calibration.py:358-478; 0 = no register limit = reference behaviour)."""
    obj = _read_json(path)
    ext = obj.get("extensions", {}) if isinstance(obj, dict) else {}
    if not isinstance(ext, dict):
        raise SchemaViolation(f"{path}.extensions: must be an object")
    v = ext.get("regs_per_sm", 0)
    if not _is_num(v) or v < 0 or v != int(v):
        raise SchemaViolation(f"{path}.extensions.regs_per_sm: must be a non-negative integer")
    return int(v)


def load_profiles(directory=None, *, with_register_limit: bool = False):
    """Every ``*.json`` profile of a directory (default: the authored spec files shipped with the
    package), sorted by file name, as the packed SoA the grid kernel consumes.

    Returns ``(names, pairs, rows)``: architecture names, the ``(ArchitectureSpec,
    CalibrationProfile)`` pairs exactly as ``load_profile`` returns them, and a float64
    ``[S, SPEC_WIDTH]`` array (``pack_spec`` per file).  ``with_register_limit`` also packs the
    files' ``extensions.regs_per_sm`` (extension, off by default = reference behaviour)."""
    import numpy as np
    directory = Path(directory) if directory is not None else SPEC_DIR
    files = sorted(p for p in directory.glob("*.json"))
    if not files:
        raise SchemaViolation(f"{directory}: no *.json profile found")
    names, pairs, rows = [], [], []
    for f in files:
        arch, prof = load_profile(f)
        names.append(arch.name)
        pairs.append((arch, prof))
        rows.append(pack_spec(arch, prof, load_regs_per_sm(f) if with_register_limit else 0))
    if len(set(names)) != len(names):
        raise SchemaViolation(f"{directory}: duplicate architecture names {sorted(names)}")
    return names, pairs, np.ascontiguousarray(np.asarray(rows, dtype=np.float64).reshape(len(rows), SPEC_WIDTH))
