"""Drop-in entry points of the reference package, backed by the CUDA kernels.

Same names, argument meaning, return types and exceptions as ``ptxwatt`` (re-export list
pkg/src/ptxwatt/__init__.py:4-55) for the analysis path: every number these functions
return is computed by libffb on the GPU; the host side only validates arguments, slices
strings out of the source text at device-provided offsets and builds the (immutable)
result objects.  The two pieces of host-only work are the ``.param`` list of the kernel
header (metadata no model reads) and the integer resource rule of ``launch.py``.
"""
from __future__ import annotations

import math
import re
from dataclasses import dataclass, replace

import numpy as np
import torch

from . import corpus as _corpus
from . import engine, native
from .errors import (AnnotationForUnknownLoop, CapacityExceeded, InvalidConfig, MalformedPtx,  # type: ignore[attr-defined]
                     NoFeasibleConfig, SharedMemOverflow, raise_for_status)
from .model_types import (OPCODE_CLASSES, STATE_SPACES, TYPE_BYTES, UNIT_CLASSES, ArchitectureSpec,
                          CalibrationProfile, ControlFlowGraph, InputResources, Instruction, KernelFeatures,
                          LaunchConfig, Loop, ParetoSet, PowerBreakdown, Prediction, PtxModule, TimeBreakdown)
from .specs import default_architecture, default_calibration, pack_spec

RESOURCE_RULES = ("mha", "generic")
_N = native


# ============================================================ PTX front end (K1 + K1b)
@dataclass
class _KernelHandle:
    """Device-side state of one parsed kernel, kept on PtxModule._dev / ControlFlowGraph._dev."""
    corp: _corpus.Corpus
    lex: _corpus.LexResult
    source: bytes
    flow: _corpus.FlowResult | None = None
    default_trip: float = 32.0
    annotations: tuple = ()


def _clean_span(raw: bytes) -> str:
    """Text of a statement piece that spans lines or holds comments, as the reference sees it
    after comment stripping and line joining (ptx.py:139-141,257-266)."""
    txt = raw.decode("utf-8", "replace")
    if "/" in txt:
        txt = re.sub(r"/\*.*?\*/", lambda m: re.sub(r"[^\n]", " ", m.group(0)), txt, flags=re.S)
        txt = re.sub(r"//[^\n]*", "", txt)
    if "\n" in txt:
        txt = " ".join(p for p in (q.strip() for q in txt.split("\n")) if p)
    return txt.strip()


def _top_level_split(text: str) -> tuple:
    """Operand list -> operands, split at commas outside [..] {..} (..) (ptx.py:144-162); empty pieces are dropped."""
    parts, depth, start = [], 0, 0
    for i, ch in enumerate(text):
        if ch in "[{(":
            depth += 1
        elif ch in "]})":
            depth -= 1
        elif ch == "," and depth == 0:
            parts.append(text[start:i].strip())
            start = i + 1
    parts.append(text[start:].strip())
    return tuple(q for q in parts if q)


def _slice(src: bytes, off: int, length: int) -> str:
    raw = src[off: off + length]
    if b"\n" in raw or b"/" in raw:
        return _clean_span(raw)
    return raw.decode("utf-8", "replace")


_PARAM = re.compile(r"\.param\s+(?:\.align\s+\d+\s+)?\.(\w+)\s+([\w$]+)(?:\[(\d+)\])?")


def _header_parameters(src: bytes, name: str, name_off: int, body_off: int) -> tuple:
    """Kernel parameter list (ptx.py:190-204): header metadata, not consumed by any model.
    The header runs from the LAST `.entry` before the body (ptx.py:191, rfind) to the opening brace,
    on the comment-stripped text (ptx.py:139-141)."""
    head = src[:body_off].decode("utf-8", "replace")
    if "/" in head:
        head = re.sub(r"/\*.*?\*/", lambda m: re.sub(r"[^\n]", " ", m.group(0)), head, flags=re.S)
        head = re.sub(r"//[^\n]*", "", head)
    header = head[max(head.rfind(".entry"), 0):]
    lp = header.find("(")
    if lp < 0:
        return ()
    rp = header.find(")", lp)
    if rp < 0:
        raise MalformedPtx(f"kernel {name!r}: unterminated parameter list")
    out = []
    for ty, pname, arr in _PARAM.findall(header[lp:rp]):
        elem = TYPE_BYTES.get(ty, 0)
        out.append((pname, "param", int(arr) * elem if arr else elem))
    return tuple(out)


def _run_flow(h: _KernelHandle, default_trip: float, annotations: dict | None) -> _corpus.FlowResult:
    fl = _corpus.kernel_features(h.corp, h.lex, default_trip=default_trip, annotations=annotations, detail=True)
    status = int(fl.status.cpu()[0])
    if status:
        raise_for_status(status, "PTX analysis failed on the device")
    return fl


def parse_ptx(source: str, kernel_name: str | None = None) -> PtxModule:
    """ptx.py:207 — same result object, produced by the GPU lexer."""
    src = source.encode("utf-8")
    rt = native.get_runtime()
    corp = _corpus.upload_corpus(src, np.array([0, len(src)], dtype=np.int64), balance=False, rt=rt)
    lex = _corpus.lex_records(corp, kernel_name=kernel_name, spans=True, decls=True, rt=rt)
    info = lex.info_np()[0]
    status = int(info["status"])
    if status:
        what = {1: "malformed PTX (unbalanced braces, unterminated statement or empty body)",
                2: f"kernel {kernel_name!r} not found" if kernel_name else "no .entry kernel in source"}.get(status, "lexer")
        raise_for_status(status, what)
    handle = _KernelHandle(corp=corp, lex=lex, source=src)
    handle.flow = _run_flow(handle, 32.0, None)          # also validates branch targets (ptx.py:277-284)
    n = int(info["n_instr"])
    ins = lex.ins.cpu().numpy().view(_corpus.INS_DTYPE).reshape(-1)[:n]
    spans = lex.spans.cpu().numpy().view(_corpus.SPAN_DTYPE).reshape(-1)[:n]
    instructions = []
    for r, sp in zip(ins, spans):
        meta = int(r["meta"])
        n_ops = int(sp["n_ops"])
        ops = tuple(_slice(src, int(sp["op_off"][i]), int(sp["op_len"][i])) for i in range(min(n_ops, _corpus.MAX_SPAN_OPS)))
        if n_ops > _corpus.MAX_SPAN_OPS:
            # the span record holds 12 operands; the rest of the list is cut out of the statement's own text (device
            # offsets: the last recorded operand up to the statement's end) at its top-level commas (ptx.py:144-162)
            last = _corpus.MAX_SPAN_OPS - 1
            tail = _top_level_split(_clean_span(src[int(sp["op_off"][last]): int(r["off"]) + int(r["len"])]))
            ops = ops[:last] + tail
            if len(ops) != n_ops:
                raise CapacityExceeded(f"statement at line {int(r['line'])}: {n_ops} operands on the device, {len(ops)} in the text")
        pred = _slice(src, int(sp["pred_off"]), int(sp["pred_len"])) if (meta >> 18) & 1 else None
        instructions.append(Instruction(
            opcode=_slice(src, int(sp["opc_off"]), int(sp["opc_len"])),
            opcode_class=OPCODE_CLASSES[meta & 15], state_space=STATE_SPACES[(meta >> 4) & 7],
            operands=ops, predicate=pred, source_line=int(r["line"])))
    labels: dict[str, int] = {}
    lab = lex.labels.cpu().numpy().view(_corpus.LABEL_DTYPE).reshape(-1)[: int(info["n_labels"])]
    for rec in lab:
        off = int(rec["off"])
        labels[src[off: src.index(b":", off)].decode("utf-8", "replace")] = int(rec["index"])
    n_decls = int(info["n_decls"])
    if n_decls > _corpus.MAX_DECLS:
        raise CapacityExceeded(f"{n_decls} .reg declarations (limit {_corpus.MAX_DECLS})")
    regs: dict[str, int] = {}
    for d in lex.decls.cpu().numpy().view(_corpus.DECL_DTYPE).reshape(-1)[:n_decls]:
        cls = src[int(d["cls_off"]): int(d["cls_off"]) + int(d["cls_len"])].decode()
        regs[cls] = regs.get(cls, 0) + int(d["count"])
    name = src[int(info["name_off"]): int(info["name_off"]) + int(info["name_len"])].decode()
    return PtxModule(kernel_name=name,
                     parameters=_header_parameters(src, name, int(info["name_off"]), int(info["body_off"])),
                     registers_declared=regs, static_shared_bytes=int(info["static_shared"]),
                     instructions=tuple(instructions), labels=labels, _dev=handle)


def classify_opcodes(opcodes: list[str]) -> list[tuple[str, str, int]]:
    """Batch form of ptx.py:99 + :64: (class, state space, access bytes) per opcode string."""
    if not opcodes:
        return []
    rt = native.get_runtime()
    blobs = [o.encode("utf-8") for o in opcodes]
    offs = np.cumsum([0] + [len(b) for b in blobs]).astype(np.int64)
    text = rt.to_device(torch.frombuffer(bytearray(b"".join(blobs) + b"\0" * 16), dtype=torch.uint8))
    d_off = rt.to_device(torch.from_numpy(offs))
    out = rt.empty((len(opcodes), 3), torch.int32)
    rc = rt.lib.ffb_classify_opcodes(rt.ctx, native.ptr(text), native.ptr(d_off), len(opcodes), native.ptr(out), rt.stream())
    rt.check(rc, "ffb_classify_opcodes")
    return [(OPCODE_CLASSES[c], STATE_SPACES[s], int(b)) for c, s, b in out.cpu().tolist()]


def classify_opcode(opcode: str) -> tuple[str, str]:
    """ptx.py:99."""
    cls, space, _ = classify_opcodes([opcode])[0]
    return cls, space


def _handle_of(module: PtxModule) -> _KernelHandle:
    if module._dev is not None:
        return module._dev
    # a hand-built module: serialise it back to PTX and lex that on the device
    lines = [f".entry {module.kernel_name}()", "{"]
    # declarations carry numbers the models read (features.py:111 static shared, :126 registers)
    for n_decl, (cls, count) in enumerate(module.registers_declared.items()):
        tag = "".join(chr(ord("a") + int(d)) for d in str(n_decl))          # register names are letters only (ptx.py:37)
        lines.append(f".reg .{cls} %ffbdecl_{tag}<{int(count)}>;")
    if module.static_shared_bytes:
        lines.append(f".shared .b8 ffb_static_shared[{int(module.static_shared_bytes)}];")
    by_index: dict[int, list[str]] = {}
    for name, idx in module.labels.items():
        by_index.setdefault(idx, []).append(name)
    for i, ins in enumerate(module.instructions):
        lines += [f"{nm}:" for nm in by_index.get(i, [])]
        pred = f"@{ins.predicate} " if ins.predicate else ""
        lines.append(f"{pred}{ins.opcode} {', '.join(ins.operands)};")
    lines += [f"{nm}:" for nm in by_index.get(len(module.instructions), [])]
    lines.append("}")
    return parse_ptx("\n".join(lines) + "\n")._dev


def _cfg_from_flow(h: _KernelHandle, fl: _corpus.FlowResult, with_trips: bool) -> ControlFlowGraph:
    finfo = fl.flow.cpu().numpy().view(_corpus.FLOW_DTYPE).reshape(-1)[0]
    nb, ne, nl = int(finfo["n_blocks"]), int(finfo["n_edges"]), int(finfo["n_loops"])
    starts = fl.block_start.cpu().numpy()[: nb + 1]
    blocks = tuple((int(starts[i]), int(starts[i + 1])) for i in range(nb))
    edges = tuple((int(u), int(v)) for u, v in fl.edges.cpu().numpy()[:ne])
    loops_np = fl.loops.cpu().numpy().view(_corpus.LOOP_DTYPE).reshape(-1)[:nl]
    if nl * nb > int(fl.loop_body.numel()):
        raise CapacityExceeded("loop membership matrix exceeds the detail buffer")
    body = fl.loop_body.cpu().numpy()[: nl * nb].reshape(nl, nb) if nl else np.zeros((0, nb), dtype=np.uint8)
    loops = []
    for i, lr in enumerate(loops_np):
        label = None
        if int(lr["has_label"]):
            off = int(lr["label_off"])
            label = h.source[off: h.source.index(b":", off)].decode("utf-8", "replace")
        loops.append(Loop(header=int(lr["header"]), body=frozenset(int(b) for b in np.nonzero(body[i])[0]),
                          trip=float(lr["trip"]) if with_trips else None, header_label=label))
    return ControlFlowGraph(blocks=blocks, edges=edges, loops=tuple(loops),
                            _dev=replace(h, flow=fl) if with_trips else h)


def build_cfg(module: PtxModule) -> ControlFlowGraph:
    """cfg.py:57 — blocks, edges and natural loops (trip = None until estimate_trip_counts)."""
    h = _handle_of(module)
    return _cfg_from_flow(h, h.flow, with_trips=False)


def estimate_trip_counts(cfg: ControlFlowGraph, module: PtxModule, default_trip: float = 32.0,
                         annotations: dict[str, float] | None = None) -> ControlFlowGraph:
    """cfg.py:154 — annotation > detected counted loop > default, floored at 1."""
    annotations = dict(annotations or {})
    known = {loop.header_label for loop in cfg.loops if loop.header_label}
    for key in annotations:
        if key not in known:
            raise AnnotationForUnknownLoop(f"annotation {key!r} does not name a loop header (known: {sorted(known)})")
    h = _handle_of(module)
    fl = _run_flow(h, float(default_trip), annotations)
    h2 = replace(h, flow=fl, default_trip=float(default_trip), annotations=tuple(sorted(annotations.items())))
    return _cfg_from_flow(h2, fl, with_trips=True)


def _feature_row(module: PtxModule, cfg: ControlFlowGraph) -> np.ndarray:
    h = cfg._dev if cfg is not None and cfg._dev is not None else None
    if h is None or h.flow is None:
        raise ValueError("cfg carries no device analysis; obtain it from build_cfg / estimate_trip_counts")
    if any(loop.trip is None for loop in cfg.loops):
        raise ValueError("trip counts not estimated; run estimate_trip_counts first")
    return h.flow.feat.cpu().numpy()[0].copy()


def analyze_memory_alignment(module: PtxModule, cfg: ControlFlowGraph) -> float:
    """alignment.py:128."""
    return float(_feature_row(module, cfg)[_N.F_ALIGNED])


def dynamic_instruction_counts(module: PtxModule, cfg: ControlFlowGraph):
    """features.py:62 -> (n_mem, mem_bytes, by_unit, n_sync)."""
    row = _feature_row(module, cfg)
    by_unit = {"FP32": float(row[_N.F_FP32]), "INT": float(row[_N.F_INT]), "SFU": float(row[_N.F_SFU]),
               "ALU": float(row[_N.F_ALU])}
    return float(row[_N.F_N_MEM]), float(row[_N.F_MEM_BYTES]), by_unit, float(row[_N.F_N_SYNC])


# ============================================================ single-point plumbing (K2 + K3)
def _point(feat_row, arch: ArchitectureSpec, profile: CalibrationProfile, bx: int, by: int, cap: float,
           shared_dyn: int, total_blocks: int, *, strict: bool = True) -> np.ndarray:
    """One grid point through ffb_predict_grid; returns its FFB_D_* detail row."""
    feat = engine.features_tensor([feat_row])
    res = engine.resources_tensor([[int(shared_dyn), int(total_blocks)]])
    r = engine.score_grid(feat, res, engine.spec_rows([(arch, profile)]), engine.shape_rows([(int(bx), int(by))]),
                          np.array([float(cap)]), want=("detail",), strict=strict, check=strict)
    return r.detail.cpu().numpy().reshape(-1)


def _row_from_features(f: KernelFeatures, t_exec: float | None = None) -> list[float]:
    row = [0.0] * _N.FEAT_WIDTH
    u = f.n_comp_by_unit
    row[_N.F_N_MEM], row[_N.F_MEM_BYTES] = f.n_mem, f.mem_bytes
    row[_N.F_FP32], row[_N.F_INT] = u.get("FP32", 0.0), u.get("INT", 0.0)
    row[_N.F_SFU], row[_N.F_ALU] = u.get("SFU", 0.0), u.get("ALU", 0.0)
    row[_N.F_N_SYNC], row[_N.F_ALIGNED] = f.n_sync, f.aligned_fraction
    row[_N.F_OVR], row[_N.F_OVR_WARPS], row[_N.F_OVR_BPS] = 1.0, float(f.warps), f.blocks_per_sm
    row[_N.F_OVR_ETA], row[_N.F_OVR_NCOMP] = f.eta_coal, f.n_comp
    row[_N.F_OVR_TEXEC] = float("nan") if t_exec is None else float(t_exec)
    return row


def _time_of(d: np.ndarray) -> TimeBreakdown:
    return TimeBreakdown(mwp=float(d[_N.D_MWP]), cwp=float(d[_N.D_CWP]), bw_eff=float(d[_N.D_BW_EFF]),
                         t_mem=float(d[_N.D_T_MEM]), t_comp=float(d[_N.D_T_COMP]), t_sync=float(d[_N.D_T_SYNC]),
                         t_exec=float(d[_N.D_T_EXEC]))


def _power_of(d: np.ndarray) -> PowerBreakdown:
    return PowerBreakdown(p_units=float(d[_N.D_P_UNITS]), p_shape=float(d[_N.D_P_SHAPE]), p_mem=float(d[_N.D_P_MEM]),
                          p_sm=float(d[_N.D_P_SM]), p_dyn=float(d[_N.D_P_DYN]), f_adj=float(d[_N.D_F_ADJ]),
                          ci=float(d[_N.D_CI]), active_sms=int(d[_N.D_ACTIVE_SMS]),
                          cap_limited=bool(d[_N.D_CAP_LIMITED] != 0.0))


def coalescing_efficiency(block_x: int, aligned_fraction: float) -> float:
    """features.py:55."""
    if block_x < 1:
        raise InvalidConfig(f"block_x must be >= 1, got {block_x}")
    row = [0.0] * _N.FEAT_WIDTH
    row[_N.F_ALIGNED] = float(aligned_fraction)
    row[_N.F_OVR_TEXEC] = float("nan")
    a = default_architecture()
    d = _point(row, a, default_calibration(), block_x, 1, a.p_tdp, 0, 1, strict=False)
    return float(d[_N.D_ETA])


def extract_features(module: PtxModule, cfg: ControlFlowGraph, config: LaunchConfig, resources: InputResources,
                     arch: ArchitectureSpec) -> KernelFeatures:
    """features.py:84 — device counts from K1b, occupancy from K2."""
    threads = config.block_x * config.block_y
    if threads % 32 != 0:
        raise InvalidConfig(f"block {config.block_x}x{config.block_y}: {threads} threads not a multiple of 32")
    if not 32 <= threads <= arch.max_threads_per_block:
        raise InvalidConfig(f"block {config.block_x}x{config.block_y}: {threads} threads outside "
                            f"[32, {arch.max_threads_per_block}]")
    row = _feature_row(module, cfg)
    d = _point(row, arch, default_calibration(), config.block_x, config.block_y, arch.p_tdp,
               resources.shared_mem_bytes, max(resources.total_blocks, 1), strict=False)
    by_unit = {"FP32": float(row[_N.F_FP32]), "INT": float(row[_N.F_INT]), "SFU": float(row[_N.F_SFU]),
               "ALU": float(row[_N.F_ALU])}
    return KernelFeatures(
        n_mem=float(row[_N.F_N_MEM]), n_comp_by_unit=by_unit,
        n_comp=by_unit["FP32"] + by_unit["INT"] + by_unit["SFU"], n_sync=float(row[_N.F_N_SYNC]),
        aligned_fraction=float(row[_N.F_ALIGNED]), eta_coal=float(d[_N.D_ETA]), warps=int(d[_N.D_WARPS]),
        blocks_per_sm=float(d[_N.D_BLOCKS_PER_SM]), registers_per_thread=sum(module.registers_declared.values()),
        shared_bytes=module.static_shared_bytes + resources.shared_mem_bytes, mem_bytes=float(row[_N.F_MEM_BYTES]))


def execution_time(features: KernelFeatures, profile: CalibrationProfile, arch: ArchitectureSpec,
                   grid: InputResources) -> TimeBreakdown:
    """time_model.py:84."""
    d = _point(_row_from_features(features), arch, profile, 32, 1, arch.p_tdp, 0, grid.total_blocks)
    return _time_of(d)


def dynamic_power(features: KernelFeatures, profile: CalibrationProfile, arch: ArchitectureSpec,
                  config: LaunchConfig, resources: InputResources, t_exec: float) -> PowerBreakdown:
    """power_model.py:109 (``t_exec`` only feeds the transient test, as in the reference)."""
    d = _point(_row_from_features(features, t_exec=t_exec), arch, profile, config.block_x, config.block_y,
               config.p_cap, 0, resources.total_blocks)
    return _power_of(d)


def predict_energy(features: KernelFeatures, arch: ArchitectureSpec, profile: CalibrationProfile,
                   config: LaunchConfig, resources: InputResources) -> Prediction:
    """explorer.py:97."""
    d = _point(_row_from_features(features), arch, profile, config.block_x, config.block_y, config.p_cap, 0,
               resources.total_blocks)
    return Prediction(config=config, time=_time_of(d), power=_power_of(d), e_pred=float(d[_N.D_E_PRED]))


# ---- scalar helpers of time_model.py / power_model.py, evaluated by the same kernel ----------
def _probe_spec(**kw):
    a = replace(default_architecture(), sm_count=1, max_warps_per_sm=1 << 20, p_tdp=1e300, p_static=0.0, p_cap_min=0.0,
                tau_short=0.0, exec_cycles=dict(zip(UNIT_CLASSES, (1.0,) * 5)), issue_cycles=dict(zip(UNIT_CLASSES, (1.0,) * 5)))
    p = CalibrationProfile(beta_u=dict(zip(UNIT_CLASSES, (0.0,) * 5)), l_mem_coal=0.0, l_mem_uncoal=0.0,
                           sm_power_alpha=0.0, sm_power_beta=1.0, sm_power_delta=0.0, transient_ratio_r=1.0, kappa=0.0,
                           lambda_=0.0, p_base_shape=0.0, p_mem_base=0.0, time_weights=(1.0, 1.0, 1.0), t_base=0.0,
                           e_overhead=0.0)
    a_kw = {k: v for k, v in kw.items() if hasattr(a, k)}
    p_kw = {k: v for k, v in kw.items() if hasattr(p, k) and k not in a_kw}
    return replace(a, **a_kw), replace(p, **p_kw)


def _probe_row(**cols) -> list[float]:
    row = [0.0] * _N.FEAT_WIDTH
    row[_N.F_OVR], row[_N.F_OVR_WARPS], row[_N.F_OVR_BPS], row[_N.F_OVR_ETA] = 1.0, 1.0, 1.0, 1.0
    row[_N.F_OVR_TEXEC] = float("nan")
    for k, v in cols.items():
        row[getattr(_N, k)] = float(v)
    return row


def mwp(l_mem_coal: float, departure_delay: float) -> float:
    """time_model.py:33."""
    a, p = _probe_spec(departure_delay=departure_delay, l_mem_coal=l_mem_coal)
    return float(_point(_probe_row(), a, p, 32, 1, a.p_tdp, 0, 1)[_N.D_MWP])


def cwp(cycles_mem: float, cycles_comp: float) -> float:
    """time_model.py:40."""
    a, p = _probe_spec(l_mem_coal=cycles_mem, departure_delay=1.0)
    a = replace(a, exec_cycles={**a.exec_cycles, "FP32": float(cycles_comp)})
    return float(_point(_probe_row(F_FP32=1.0, F_OVR_NCOMP=1.0), a, p, 32, 1, a.p_tdp, 0, 1)[_N.D_CWP])


def wave_count(features: KernelFeatures, arch: ArchitectureSpec, resources: InputResources) -> float:
    """time_model.py:67."""
    d = _point(_row_from_features(features), arch, default_calibration(), 32, 1, arch.p_tdp, 0, resources.total_blocks)
    return float(d[_N.D_WAVES])


def activity_rate(inst_count: float, warps_per_sm: float, exec_cycles: float, issue_cycles: float) -> float:
    """power_model.py:31."""
    from .errors import ZeroCycles  # type: ignore[attr-defined]
    if exec_cycles <= 0 or issue_cycles <= 0:
        raise ZeroCycles(f"exec/issue cycles must be positive, got {exec_cycles}/{issue_cycles}")
    a, p = _probe_spec(departure_delay=1.0)
    a = replace(a, exec_cycles={**a.exec_cycles, "FP32": float(exec_cycles)},
                issue_cycles={**a.issue_cycles, "FP32": float(issue_cycles)})
    p = replace(p, beta_u={**p.beta_u, "FP32": 1.0})
    row = _probe_row(F_FP32=inst_count, F_OVR_BPS=warps_per_sm, F_OVR_NCOMP=0.0)
    return float(_point(row, a, p, 32, 32, a.p_tdp, 0, 1)[_N.D_P_UNITS])


def compute_intensity(n_comp: float, n_mem: float) -> float:
    """power_model.py:42."""
    a, p = _probe_spec(departure_delay=1.0)
    return float(_point(_probe_row(F_N_MEM=n_mem, F_OVR_NCOMP=n_comp), a, p, 32, 32, a.p_tdp, 0, 1)[_N.D_CI])


def shape_power(p_base: float, kappa: float, block_x: int, block_y: int, ci: float) -> float:
    """power_model.py:49."""
    if block_x < 1 or block_y < 1:
        raise ValueError(f"block dimensions must be >= 1, got {block_x}x{block_y}")
    a, p = _probe_spec(departure_delay=1.0, p_base_shape=p_base, kappa=kappa)
    row = _probe_row(F_N_MEM=0.0 if math.isinf(ci) else 1.0, F_OVR_NCOMP=0.0 if math.isinf(ci) else ci)
    return float(_point(row, a, p, block_x, block_y, a.p_tdp, 0, 1)[_N.D_P_SHAPE])


def memory_power(p_mem_base: float, lambda_: float, eta: float) -> float:
    """power_model.py:65."""
    a, p = _probe_spec(departure_delay=1.0, p_mem_base=p_mem_base, lambda_=lambda_)
    return float(_point(_probe_row(F_OVR_ETA=eta), a, p, 32, 32, a.p_tdp, 0, 1)[_N.D_P_MEM])


def sm_concurrency_power(n_active: int, alpha: float, beta: float, delta: float) -> float:
    """power_model.py:70."""
    if n_active < 0:
        raise ValueError(f"active SM count must be >= 0, got {n_active}")
    a, p = _probe_spec(departure_delay=1.0, sm_count=max(int(n_active), 1), sm_power_alpha=alpha, sm_power_beta=beta,
                       sm_power_delta=delta)
    return float(_point(_probe_row(), a, p, 32, 32, a.p_tdp, 0, int(n_active), strict=False)[_N.D_P_SM])


def estimate_active_sms(config: LaunchConfig, resources: InputResources, arch: ArchitectureSpec) -> int:
    """power_model.py:79."""
    d = _point(_probe_row(), arch, default_calibration(), config.block_x, config.block_y, arch.p_tdp, 0,
               resources.total_blocks)
    return int(d[_N.D_ACTIVE_SMS])


def transient_correction(p_dyn: float, t_exec: float, tau_short: float, r: float) -> float:
    """power_model.py:89."""
    a, p = _probe_spec(departure_delay=1.0, tau_short=tau_short, transient_ratio_r=r, sm_power_delta=p_dyn)
    return float(_point(_probe_row(F_OVR_TEXEC=t_exec), a, p, 32, 32, a.p_tdp, 0, 1)[_N.D_P_DYN])


def dvfs_frequency(f_base: float, p_cap: float, p_tdp: float, k: int) -> float:
    """power_model.py:98."""
    a, p = _probe_spec(departure_delay=1.0, f_base=f_base, p_tdp=p_tdp, dvfs_exponent_k=int(k))
    return float(_point(_probe_row(), a, p, 32, 32, p_cap, 0, 1)[_N.D_F_ADJ])


# ============================================================ exploration (K2 + K3 + K4)
def compute_input_resources(seq_len: int, batch: int, heads: int, head_dim: int, bytes_per_elem: int,
                            arch: ArchitectureSpec, rule: str = "mha") -> InputResources:
    """launch.py:44 — integer workload rule (host)."""
    if min(seq_len, batch, heads, head_dim, bytes_per_elem) < 1:
        raise ValueError("all workload dimensions must be >= 1")
    if rule not in RESOURCE_RULES:
        raise ValueError(f"unknown resource rule {rule!r}; expected one of {RESOURCE_RULES}")
    shared = bytes_per_elem * (head_dim + seq_len) if rule == "mha" else 0
    if shared > arch.max_shared_per_sm:
        raise SharedMemOverflow(f"workload needs {shared} B shared per block; architecture provides "
                                f"{arch.max_shared_per_sm} B per SM")
    return InputResources(shared_mem_bytes=shared, grid_x=heads, grid_y=batch, grid_z=1, seq_len=seq_len,
                          batch=batch, heads=heads)


def generate_valid_configs(arch: ArchitectureSpec, resources: InputResources, dim_candidates: list[int],
                           cap_candidates: list[float] | None = None) -> list[LaunchConfig]:
    """explorer.py:59 — canonical (threads, block_x, block_y, p_cap) order."""
    caps = sorted(set(cap_candidates)) if cap_candidates else [arch.p_tdp]
    caps = [float(c) for c in caps if arch.p_cap_min <= c <= arch.p_tdp]
    row = np.asarray(pack_spec(arch, default_calibration()), dtype=np.float64)
    shapes = engine.enumerate_shapes(row, resources.shared_mem_bytes, dim_candidates)
    return [LaunchConfig(block_x=int(bx), block_y=int(by), p_cap=c) for bx, by in shapes for c in caps]


def _config_key(c: LaunchConfig):
    return (c.threads, c.block_x, c.block_y, c.p_cap)


def evaluate_configs(module: PtxModule, cfg: ControlFlowGraph, arch: ArchitectureSpec, profile: CalibrationProfile,
                     resources: InputResources, configs: list[LaunchConfig], jobs: int = 1) -> list[Prediction]:
    """explorer.py:161 — one grid launch for all configs (``jobs`` is accepted for
    compatibility; the GPU evaluates every point in parallel and the result is identical)."""
    if not configs:
        return []
    for c in configs:
        th = c.block_x * c.block_y
        if th % 32 != 0:
            raise InvalidConfig(f"block {c.block_x}x{c.block_y}: {th} threads not a multiple of 32")
        if not 32 <= th <= arch.max_threads_per_block:
            raise InvalidConfig(f"block {c.block_x}x{c.block_y}: {th} threads outside [32, {arch.max_threads_per_block}]")
    row = _feature_row(module, cfg)
    shapes = sorted({(c.block_x, c.block_y) for c in configs})
    caps = sorted({float(c.p_cap) for c in configs})
    s_idx = {s: i for i, s in enumerate(shapes)}
    c_idx = {c: i for i, c in enumerate(caps)}
    r = engine.score_grid(engine.features_tensor([row]),
                          engine.resources_tensor([[resources.shared_mem_bytes, resources.total_blocks]]),
                          engine.spec_rows([(arch, profile)]), engine.shape_rows(shapes), np.asarray(caps),
                          want=("detail",), strict=True)
    det = r.detail.cpu().numpy()[0, 0].tolist()          # [shape][cap][DETAIL_WIDTH] as Python floats: one conversion, not 21 per row
    D = _N
    isfinite = math.isfinite
    out, keys = [], []
    for c in configs:
        d = det[s_idx[(c.block_x, c.block_y)]][c_idx[float(c.p_cap)]]
        t_exec, e_pred = d[D.D_T_EXEC], d[D.D_E_PRED]
        if not (isfinite(t_exec) and isfinite(e_pred)):
            # IEEE gives inf / nan where CPython raises (a zero divisor such as ipc = 0, time_model.py:116)
            raise ZeroDivisionError("float division by zero")
        out.append(Prediction(c, TimeBreakdown(d[D.D_MWP], d[D.D_CWP], d[D.D_BW_EFF], d[D.D_T_MEM], d[D.D_T_COMP], d[D.D_T_SYNC], t_exec),
                              PowerBreakdown(d[D.D_P_UNITS], d[D.D_P_SHAPE], d[D.D_P_MEM], d[D.D_P_SM], d[D.D_P_DYN], d[D.D_F_ADJ], d[D.D_CI],
                                             int(d[D.D_ACTIVE_SMS]), d[D.D_CAP_LIMITED] != 0.0), e_pred))
        keys.append((c.block_x * c.block_y, c.block_x, c.block_y, c.p_cap))
    if any(keys[i] > keys[i + 1] for i in range(len(keys) - 1)):     # explorer.py:182; generate_valid_configs' order needs no sort
        order = sorted(range(len(out)), key=keys.__getitem__)
        out = [out[i] for i in order]
    return out


def _front_order(predictions: list[Prediction], rho: float):
    n = len(predictions)
    e = np.fromiter((p.e_pred for p in predictions), dtype=np.float64, count=n)
    t = np.fromiter((p.time.t_exec for p in predictions), dtype=np.float64, count=n)
    cfgs = [p.config for p in predictions]
    keys = np.lexsort((np.arange(n), np.fromiter((c.p_cap for c in cfgs), dtype=np.float64, count=n),
                       np.fromiter((c.block_y for c in cfgs), dtype=np.int64, count=n),
                       np.fromiter((c.block_x for c in cfgs), dtype=np.int64, count=n)))     # (block_x, block_y, p_cap, position)
    tie = np.empty(n, dtype=np.int32)
    tie[keys] = np.arange(n, dtype=np.int32)
    rt = native.get_runtime()
    d_e, d_t = rt.to_device(torch.from_numpy(e)), rt.to_device(torch.from_numpy(t))
    try:
        fi, fn, tp = engine.skyline_groups(d_e, d_t, 1, n, tie=rt.to_device(torch.from_numpy(tie)), rho=rho, cap_front=n, rt=rt)
        k = int(fn.cpu()[0])
        return fi.cpu().numpy()[0, :k].tolist(), float(tp.cpu()[0])
    except CapacityExceeded:
        # the front does not fit one CTA's shared memory (e.g. > 10^4 mutually non-dominated points):
        # the streaming skyline takes any size; ids carry the tie rank so the order is still (e, t, bx, by, cap)
        inv = np.empty(n, dtype=np.int64)
        inv[tie] = np.arange(n)
        ids, _, _, t_peak = engine.skyline(d_e, d_t, ids=rt.to_device(torch.from_numpy(tie.astype(np.int64))), rho=rho,
                                           cap_front=n, rt=rt)
        return inv[ids.cpu().numpy()].tolist(), float(t_peak)


def pareto_front(predictions: list[Prediction]) -> list[Prediction]:
    """explorer.py:122 — strict dominance in (e_pred, t_exec); ties survive; (e, t, bx, by, cap) order."""
    if not predictions:
        return []
    idx, _ = _front_order(predictions, 0.0)
    return [predictions[i] for i in idx]


def pareto_front_bruteforce(predictions: list[Prediction]) -> ParetoSet:
    """explorer.py:143 — same set and order as the reference's O(n^2) ground truth."""
    if not predictions:
        raise NoFeasibleConfig("no predictions to rank")
    idx, t_peak = _front_order(predictions, 0.0)
    return ParetoSet(entries=tuple(predictions[i] for i in idx), rho=0.0, t_peak=t_peak)


def pareto_explore(module: PtxModule, cfg: ControlFlowGraph, arch: ArchitectureSpec, profile: CalibrationProfile,
                   resources: InputResources, dim_candidates: list[int], cap_candidates: list[float] | None = None,
                   rho: float = 0.95, jobs: int = 1) -> ParetoSet:
    """explorer.py:186."""
    if not 0 < rho <= 1:
        raise ValueError(f"rho must be in (0, 1], got {rho}")
    # Same values as generate_valid_configs -> evaluate_configs -> pareto_front (explorer.py:203-212), without building
    # the thousands of host objects only to drop most of them: the grid is scored in (block_x, block_y, p_cap) order -
    # which IS the tie order of explorer.py:113-119 -, ranked on the device, and Prediction objects are made for the
    # front members alone.
    caps = sorted(set(cap_candidates)) if cap_candidates else [arch.p_tdp]
    caps = [float(c) for c in caps if arch.p_cap_min <= c <= arch.p_tdp]
    spec_row = np.asarray(pack_spec(arch, default_calibration()), dtype=np.float64)
    shapes = sorted((int(bx), int(by)) for bx, by in engine.enumerate_shapes(spec_row, resources.shared_mem_bytes, dim_candidates))
    if not shapes or not caps:
        raise NoFeasibleConfig("no candidate configuration passed the hardware filters")
    row = _feature_row(module, cfg)
    r = engine.score_grid(engine.features_tensor([row]),
                          engine.resources_tensor([[resources.shared_mem_bytes, resources.total_blocks]]),
                          engine.spec_rows([(arch, profile)]), engine.shape_rows(shapes), np.asarray(caps),
                          want=("detail",), strict=True)
    D = _N
    det_dev = r.detail[0, 0]                                  # [shape][cap][DETAIL_WIDTH]
    n = len(shapes) * len(caps)
    d_e = det_dev[:, :, D.D_E_PRED].reshape(-1).contiguous()
    d_t = det_dev[:, :, D.D_T_EXEC].reshape(-1).contiguous()
    if not bool((torch.isfinite(d_e) & torch.isfinite(d_t)).all()):
        # IEEE gives inf / nan where CPython raises (a zero divisor such as ipc = 0, time_model.py:116)
        raise ZeroDivisionError("float division by zero")
    rt = native.get_runtime()
    try:
        fi, fn, tp = engine.skyline_groups(d_e, d_t, 1, n, rho=float(rho), cap_front=n, rt=rt)
        idx, t_peak = fi[0, : int(fn.cpu()[0])].cpu().numpy(), float(tp.cpu()[0])
    except CapacityExceeded:
        ids, _, _, t_peak = engine.skyline(d_e, d_t, ids=torch.arange(n, dtype=torch.int64, device=d_e.device), rho=float(rho),
                                           cap_front=n, rt=rt)
        idx, t_peak = ids.cpu().numpy(), float(t_peak)
    C = len(caps)
    rows = det_dev.reshape(n, -1)[torch.from_numpy(np.asarray(idx, dtype=np.int64)).to(det_dev.device)].cpu().numpy().tolist()
    entries = []
    for g, d in zip(idx.tolist(), rows):
        bx, by = shapes[g // C]
        entries.append(Prediction(LaunchConfig(block_x=bx, block_y=by, p_cap=caps[g % C]),
                                  TimeBreakdown(d[D.D_MWP], d[D.D_CWP], d[D.D_BW_EFF], d[D.D_T_MEM], d[D.D_T_COMP], d[D.D_T_SYNC], d[D.D_T_EXEC]),
                                  PowerBreakdown(d[D.D_P_UNITS], d[D.D_P_SHAPE], d[D.D_P_MEM], d[D.D_P_SM], d[D.D_P_DYN], d[D.D_F_ADJ], d[D.D_CI],
                                                 int(d[D.D_ACTIVE_SMS]), d[D.D_CAP_LIMITED] != 0.0), d[D.D_E_PRED]))
    return ParetoSet(entries=tuple(entries), rho=rho, t_peak=t_peak)


def pareto_explore_sweep(module: PtxModule, cfg: ControlFlowGraph, specs: list, resources: list[InputResources],
                         dim_candidates: list[int], cap_candidates: list[float], rho: float = 0.95) -> dict:
    """Per-spec, per-workload fronts from ONE grid launch and ONE skyline launch (the
    paper's per-sequence-length fronts).  ``specs`` is a list of (ArchitectureSpec,
    CalibrationProfile); ``resources`` a list of InputResources (e.g. compute_input_resources per
    seq_len).  Returns {(spec_index, resource_index): ParetoSet}; every entry equals
    ``pareto_explore(module, cfg, arch, profile, resources[r], dim_candidates, cap_candidates, rho)``
    (explorer.py:186-212), or the NoFeasibleConfig instance it would raise."""
    if not 0 < rho <= 1:
        raise ValueError(f"rho must be in (0, 1], got {rho}")
    if not cap_candidates:
        raise ValueError("the sweep needs an explicit cap list (the default cap is spec-dependent)")
    rt = native.get_runtime()
    row = _feature_row(module, cfg)
    caps = sorted({float(c) for c in cap_candidates})
    sp = engine.spec_rows(specs)
    # shape axis: union over specs (validity is masked per point on the device); canonical order is spec-independent
    seen = {}
    for s in range(len(specs)):
        for bx, by in engine.enumerate_shapes(sp[s], 0, dim_candidates, rt=rt).tolist():
            seen[(bx, by)] = None
    shapes = sorted(seen, key=lambda x: (x[0] * x[1], x[0], x[1]))
    if not shapes:
        return {(s, r): NoFeasibleConfig("no candidate configuration passed the hardware filters")
                for s in range(len(specs)) for r in range(len(resources))}
    J, Cn, S, R = len(shapes), len(caps), len(specs), len(resources)
    res_axis = torch.tensor([[r.shared_mem_bytes, r.total_blocks] for r in resources], dtype=torch.int64)
    g = engine.score_grid_sweep(engine.features_tensor([row]), rt.to_device(res_axis), sp, engine.shape_rows(shapes),
                                np.asarray(caps), want=("t", "e", "flags", "detail"), rt=rt)
    order = sorted(range(J), key=lambda j: (shapes[j][0], shapes[j][1]))
    rank = np.empty(J, dtype=np.int64)
    rank[order] = np.arange(J)
    tie = (rank[:, None] * Cn + np.arange(Cn)[None, :]).reshape(-1).astype(np.int32)
    G = J * Cn
    fi, fn, tp = engine.skyline_groups(g.e.reshape(-1), g.t.reshape(-1), R * S, G, tie=rt.to_device(torch.from_numpy(tie)),
                                       rho=float(rho), cap_front=G, rt=rt)
    fi, fn, tp = fi.cpu().numpy(), fn.cpu().numpy(), tp.cpu().numpy()
    det = g.detail.cpu().numpy().reshape(R * S, G, _N.DETAIL_WIDTH)
    valid = (g.flags.cpu().numpy().reshape(R * S, G) & _N.PT_VALID) != 0
    out = {}
    for r in range(R):
        for s in range(S):
            q = r * S + s
            if not valid[q].any():
                out[(s, r)] = NoFeasibleConfig("no candidate configuration passed the hardware filters")
                continue
            entries = []
            for i in fi[q, : int(fn[q])]:
                j, c = divmod(int(i), Cn)
                d = det[q, i]
                conf = LaunchConfig(block_x=shapes[j][0], block_y=shapes[j][1], p_cap=caps[c])
                entries.append(Prediction(config=conf, time=_time_of(d), power=_power_of(d), e_pred=float(d[_N.D_E_PRED])))
            out[(s, r)] = ParetoSet(entries=tuple(entries), rho=rho, t_peak=float(tp[q]))
    return out
