"""Batched corpus entry points: PTX text on the device -> histograms, declarations,
instruction records and per-kernel dynamic feature rows (K1 + K1b).

A corpus is one byte buffer plus a segment table; segment k is analysed exactly like
``parse_ptx(text[seg_off[k]:seg_off[k+1]])`` of the reference (ptx.py:207).
"""
from __future__ import annotations

import contextlib

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .errors import raise_for_status

SEG_DTYPE = np.dtype([("status", "<u4"), ("n_instr", "<u4"), ("n_labels", "<u4"), ("n_decls", "<u4"),
                      ("static_shared", "<u8"), ("regs_declared", "<u8"), ("name_off", "<u4"),
                      ("name_len", "<u4"), ("body_off", "<u4"), ("body_end", "<u4")])
INS_DTYPE = np.dtype([("meta", "<u4"), ("line", "<u4"), ("off", "<u4"), ("len", "<u4"), ("pred", "<u8"),
                      ("aux", "<u8"), ("op", "<u8", (4,))])
LABEL_DTYPE = np.dtype([("hash", "<u8"), ("index", "<u4"), ("off", "<u4")])
MAX_SPAN_OPS, MAX_DECLS = 12, 256
SPAN_DTYPE = np.dtype([("pred_off", "<u4"), ("pred_len", "<u4"), ("opc_off", "<u4"), ("opc_len", "<u4"),
                       ("n_ops", "<u4"), ("reserved", "<u4", (3,)), ("op_off", "<u4", (MAX_SPAN_OPS,)),
                       ("op_len", "<u4", (MAX_SPAN_OPS,))])
DECL_DTYPE = np.dtype([("cls_off", "<u4"), ("cls_len", "<u4"), ("count", "<u8")])
assert SEG_DTYPE.itemsize == 48 and INS_DTYPE.itemsize == 64 and LABEL_DTYPE.itemsize == 16
assert SPAN_DTYPE.itemsize == 128 and DECL_DTYPE.itemsize == 16


class LexDesc(C.Structure):
    _fields_ = [
        ("d_text", C.c_void_p), ("n_bytes", C.c_int64), ("d_seg_off", C.c_void_p), ("n_segs", C.c_int64),
        ("d_order", C.c_void_p), ("h_kernel_name", C.c_char_p), ("kernel_name_len", C.c_int32),
        ("d_hist", C.c_void_p), ("d_info", C.c_void_p), ("d_ins_base", C.c_void_p), ("d_lab_base", C.c_void_p),
        ("d_ins_cap", C.c_void_p), ("d_lab_cap", C.c_void_p), ("d_ins", C.c_void_p), ("d_labels", C.c_void_p), ("d_meta", C.c_void_p), ("d_spans", C.c_void_p),
        ("d_decls", C.c_void_p), ("flags", C.c_uint32), ("d_path_counts", C.c_void_p),
    ]


@dataclass
class Corpus:
    """Device-resident PTX text with its segment table."""
    text: torch.Tensor          # uint8, padded to a multiple of 16
    n_bytes: int                # true byte count
    seg_off: torch.Tensor       # int64 [K+1] on the device
    n_segs: int
    order: torch.Tensor | None = None   # int32 [K] longest-first processing order
    host_text: bytes | None = None
    host_off: np.ndarray | None = None
    kernel_mask: np.ndarray | None = None   # split_modules: False for gap segments that hold no kernel

    @property
    def padded_bytes(self) -> int:
        return int(self.text.numel())

    def host_sample(self):
        return self.host_text, self.host_off


def upload_corpus(text: bytes, seg_off: np.ndarray, *, keep_host: bool = True, balance: bool = True,
                  rt: native.Runtime | None = None) -> Corpus:
    rt = rt or native.get_runtime()
    n = len(text)
    padded = (n + 15) // 16 * 16 + 16
    host = torch.zeros(padded, dtype=torch.uint8)
    host[:n] = torch.frombuffer(bytearray(text), dtype=torch.uint8)
    host[n:] = 10
    seg_off = np.ascontiguousarray(seg_off, dtype=np.int64)
    assert seg_off[0] >= 0 and seg_off[-1] <= n and np.all(np.diff(seg_off) >= 0)
    order = None
    if balance and len(seg_off) > 2:
        order = rt.to_device(torch.from_numpy(np.argsort(-np.diff(seg_off), kind="stable").astype(np.int32)))
    return Corpus(text=rt.to_device(host), n_bytes=n, seg_off=rt.to_device(torch.from_numpy(seg_off)),
                  n_segs=len(seg_off) - 1, order=order, host_text=text if keep_host else None,
                  host_off=seg_off if keep_host else None)


@dataclass
class LexResult:
    hist: torch.Tensor          # int32 [K, 9]
    info: torch.Tensor          # uint8 [K, 48]  (SEG_DTYPE)
    ins_base: torch.Tensor | None = None
    lab_base: torch.Tensor | None = None
    ins: torch.Tensor | None = None      # uint8 [N, 64]
    labels: torch.Tensor | None = None   # uint8 [L, 16]
    meta: torch.Tensor | None = None     # int32 [N] compact meta words
    ins_cap: torch.Tensor | None = None  # single-pass mode: slots per segment
    lab_cap: torch.Tensor | None = None
    spans: torch.Tensor | None = None    # uint8 [N, 128]
    decls: torch.Tensor | None = None    # uint8 [K, 32, 16]
    n_ins: int = 0
    n_lab: int = 0
    path_counts: torch.Tensor | None = None   # int32 [4]: segments fast / exact, byte-serial statements, -

    def info_np(self) -> np.ndarray:
        return self.info.cpu().numpy().view(SEG_DTYPE).reshape(-1)

    def info_i32(self) -> torch.Tensor:
        return self.info.view(torch.int32).view(-1, 12)


LEX_EXACT_ONLY = 1
LEX_NO_LOCKSTEP = 2
FLOW_SEQUENTIAL_PASS = 1
FLOW_ONE_KERNEL = 2
FLOW_FLAGS_DEFAULT = 0         # FFB_FLOW_* bits for every call (tests flip this)
LEX_FLAGS_DEFAULT = 0          # extra FFB_LEX_* bits for every call (benchmark A/B switches)
EXACT_ONLY_DEFAULT = False      # tests flip this to run the exact statement walk alone


def _call_lex(rt, corp: Corpus, hist, info, *, kernel_name: bytes | None = None, ins_base=None, lab_base=None,
              ins_cap=None, lab_cap=None, ins=None, labels=None, meta=None, spans=None, decls=None,
              exact_only: bool = False, path_counts=None, seg_range: tuple[int, int] | None = None, order=None):
    if seg_range is not None:
        # a contiguous run of segments: every per-segment array is passed from its s0-th row on
        # (offsets into the text and the record buffers stay global)
        s0, s1 = seg_range
        sl = lambda x: None if x is None else x[s0:s1]      # noqa: E731
        d = LexDesc(
            d_text=native.ptr(corp.text), n_bytes=corp.padded_bytes, d_seg_off=native.ptr(corp.seg_off[s0:s1 + 1]),
            n_segs=s1 - s0, d_order=native.ptr(order),
            h_kernel_name=kernel_name, kernel_name_len=len(kernel_name) if kernel_name else 0,
            d_hist=native.ptr(hist[s0:s1]), d_info=native.ptr(info[s0:s1]), d_ins_base=native.ptr(sl(ins_base)),
            d_lab_base=native.ptr(sl(lab_base)), d_ins_cap=native.ptr(sl(ins_cap)), d_lab_cap=native.ptr(sl(lab_cap)),
            d_ins=native.ptr(ins), d_labels=native.ptr(labels), d_meta=native.ptr(meta), d_spans=native.ptr(spans),
            d_decls=native.ptr(sl(decls)),
            flags=(LEX_EXACT_ONLY if (exact_only or EXACT_ONLY_DEFAULT) else 0) | LEX_FLAGS_DEFAULT, d_path_counts=native.ptr(path_counts))
        rc = rt.lib.ffb_lex_corpus(rt.ctx, C.byref(d), rt.stream())
        rt.check(rc, "ffb_lex_corpus")
        return
    d = LexDesc(
        d_text=native.ptr(corp.text), n_bytes=corp.padded_bytes, d_seg_off=native.ptr(corp.seg_off),
        n_segs=corp.n_segs, d_order=native.ptr(corp.order),
        h_kernel_name=kernel_name, kernel_name_len=len(kernel_name) if kernel_name else 0,
        d_hist=native.ptr(hist), d_info=native.ptr(info), d_ins_base=native.ptr(ins_base),
        d_lab_base=native.ptr(lab_base), d_ins_cap=native.ptr(ins_cap), d_lab_cap=native.ptr(lab_cap), d_ins=native.ptr(ins), d_labels=native.ptr(labels),
        d_meta=native.ptr(meta), d_spans=native.ptr(spans), d_decls=native.ptr(decls),
        flags=(LEX_EXACT_ONLY if (exact_only or EXACT_ONLY_DEFAULT) else 0) | LEX_FLAGS_DEFAULT, d_path_counts=native.ptr(path_counts))
    rc = rt.lib.ffb_lex_corpus(rt.ctx, C.byref(d), rt.stream())
    rt.check(rc, "ffb_lex_corpus")


def lex_histogram(corp: Corpus, *, kernel_name: str | None = None, out: LexResult | None = None,
                  rt: native.Runtime | None = None) -> LexResult:
    """K1, histogram mode: class counts, declarations, status per segment.  No sync."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    res = out or LexResult(hist=rt.empty((K, native.N_CLASSES), torch.int32), info=rt.empty((K, 48), torch.uint8))
    if res.path_counts is None:
        res.path_counts = rt.empty((4,), torch.int32)
    _call_lex(rt, corp, res.hist, res.info, kernel_name=kernel_name.encode() if kernel_name else None,
              path_counts=res.path_counts)
    return res


def lex_records(corp: Corpus, *, kernel_name: str | None = None, spans: bool = False, decls: bool = False,
                rt: native.Runtime | None = None) -> LexResult:
    """K1, record mode (two passes: counts, then 64-byte instruction records).  Syncs once
    to size the record buffers."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    name = kernel_name.encode() if kernel_name else None
    res = lex_histogram(corp, kernel_name=kernel_name, rt=rt)
    i32 = res.info_i32()
    n_ins = i32[:, 1].to(torch.int64).contiguous()
    n_lab = i32[:, 2].to(torch.int64).contiguous()
    inc_i, inc_l = torch.cumsum(n_ins, dim=0), torch.cumsum(n_lab, dim=0)
    res.ins_base, res.lab_base = (inc_i - n_ins).contiguous(), (inc_l - n_lab).contiguous()
    res.n_ins, res.n_lab = (int(inc_i[-1]), int(inc_l[-1])) if K else (0, 0)
    res.ins = rt.empty((max(res.n_ins, 1), 64), torch.uint8)
    res.labels = rt.empty((max(res.n_lab, 1), 16), torch.uint8)
    res.meta = rt.empty((max(res.n_ins, 1),), torch.int32)
    res.spans = torch.zeros((max(res.n_ins, 1), 128), dtype=torch.uint8, device=rt.device) if spans else None
    res.decls = torch.zeros((K, MAX_DECLS, 16), dtype=torch.uint8, device=rt.device) if decls else None
    _call_lex(rt, corp, res.hist, res.info, kernel_name=name, ins_base=res.ins_base, lab_base=res.lab_base,
              ins=res.ins, labels=res.labels, meta=res.meta, spans=res.spans, decls=res.decls,
              path_counts=res.path_counts)
    return res


def lex_records_single_pass(corp: Corpus, *, bytes_per_ins: int = 12, bytes_per_label: int = 24,
                            out: LexResult | None = None, rt: native.Runtime | None = None,
                            seg_range: tuple[int, int] | None = None, order=None) -> LexResult:
    """K1, record mode in ONE pass: every segment gets len/bytes_per_ins + 8 record slots (and
    len/bytes_per_label + 8 label slots) up front, so no counting pass and no host sync are
    needed.  A segment whose statements are shorter than that on average comes back with status
    FFB_E_CAPACITY (use ``lex_records`` for it).  Buffers can be reused through ``out``."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    res = out
    if res is None:
        seg = corp.seg_off
        length = (seg[1:] - seg[:-1])
        ins_cap = (length // bytes_per_ins + 8).contiguous()
        lab_cap = (length // bytes_per_label + 8).contiguous()
        inc_i, inc_l = torch.cumsum(ins_cap, dim=0), torch.cumsum(lab_cap, dim=0)
        res = LexResult(hist=rt.empty((K, native.N_CLASSES), torch.int32), info=rt.empty((K, 48), torch.uint8))
        res.ins_base, res.lab_base = (inc_i - ins_cap).contiguous(), (inc_l - lab_cap).contiguous()
        res.ins_cap, res.lab_cap = ins_cap, lab_cap
        res.n_ins, res.n_lab = int(inc_i[-1]), int(inc_l[-1])          # capacities, not counts
        res.ins = rt.empty((max(res.n_ins, 1), 64), torch.uint8)
        res.labels = rt.empty((max(res.n_lab, 1), 16), torch.uint8)
        res.meta = rt.empty((max(res.n_ins, 1),), torch.int32)
        res.path_counts = rt.empty((4,), torch.int32)
    _call_lex(rt, corp, res.hist, res.info, ins_base=res.ins_base, lab_base=res.lab_base, ins_cap=res.ins_cap,
              lab_cap=res.lab_cap, ins=res.ins, labels=res.labels, meta=res.meta,
              path_counts=None if seg_range is not None else res.path_counts, seg_range=seg_range, order=order)
    return res


def raise_segment_status(status: int, what: str = "PTX segment") -> None:
    raise_for_status(int(status), what)


# ------------------------------------------------------------------------------ K1b
FLOW_DTYPE = np.dtype([("n_blocks", "<u4"), ("n_edges", "<u4"), ("n_loops", "<u4"), ("reserved", "<u4")])
LOOP_DTYPE = np.dtype([("header", "<u4"), ("n_body", "<u4"), ("trip", "<f8"), ("label_hash", "<u8"),
                       ("label_off", "<u4"), ("has_label", "<u4")])
assert LOOP_DTYPE.itemsize == 32


class FlowDesc(C.Structure):
    _fields_ = [
        ("n_segs", C.c_int64), ("d_info", C.c_void_p), ("d_ins_base", C.c_void_p), ("d_lab_base", C.c_void_p),
        ("d_ins", C.c_void_p), ("d_labels", C.c_void_p), ("d_meta", C.c_void_p), ("n_ins_total", C.c_int64),
        ("n_lab_total", C.c_int64),
        ("d_order", C.c_void_p), ("default_trip", C.c_double), ("h_ann_hash", C.c_void_p),
        ("h_ann_trip", C.c_void_p), ("n_ann", C.c_int32), ("d_ann_hit", C.c_void_p), ("d_feat", C.c_void_p),
        ("d_status", C.c_void_p), ("d_flow", C.c_void_p), ("d_block_start", C.c_void_p), ("d_edges", C.c_void_p),
        ("d_loops", C.c_void_p), ("d_loop_body", C.c_void_p), ("loop_body_cap", C.c_int64), ("d_weights", C.c_void_p),
        ("flags", C.c_uint32),
    ]


def name_hash(name: str, rt: native.Runtime | None = None) -> int:
    rt = rt or native.get_runtime()
    b = name.encode()
    return int(rt.lib.ffb_name_hash(b, len(b)))


@dataclass
class FlowResult:
    feat: torch.Tensor            # float64 [K, FEAT_WIDTH]
    status: torch.Tensor          # int32 [K]
    flow: torch.Tensor | None = None         # uint8 [K, 16] (FLOW_DTYPE)
    block_start: torch.Tensor | None = None
    edges: torch.Tensor | None = None
    loops: torch.Tensor | None = None
    loop_body: torch.Tensor | None = None
    weights: torch.Tensor | None = None
    ann_hit: torch.Tensor | None = None


def kernel_features(corp: Corpus, lex: LexResult, *, default_trip: float = 32.0, annotations: dict | None = None,
                    detail: bool = False, out_feat: torch.Tensor | None = None,
                    rt: native.Runtime | None = None, seg_range: tuple[int, int] | None = None, order=None,
                    out_status: torch.Tensor | None = None) -> FlowResult:
    """K1b over the records of ``lex_records``.  No sync.  ``seg_range`` restricts the call to a
    contiguous run of segments (chunked pipelines); outputs keep their global row positions."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    if seg_range is not None:
        assert not detail and not annotations and out_feat is not None and out_status is not None
        s0, s1 = seg_range
        d = FlowDesc(
            n_segs=s1 - s0, d_info=native.ptr(lex.info[s0:s1]), d_ins_base=native.ptr(lex.ins_base[s0:s1]),
            d_lab_base=native.ptr(lex.lab_base[s0:s1]), d_ins=native.ptr(lex.ins), d_labels=native.ptr(lex.labels),
            d_meta=native.ptr(lex.meta), n_ins_total=lex.n_ins, n_lab_total=lex.n_lab, d_order=native.ptr(order),
            default_trip=float(default_trip), h_ann_hash=None, h_ann_trip=None, n_ann=0, d_ann_hit=None,
            d_feat=native.ptr(out_feat[s0:s1]), d_status=native.ptr(out_status[s0:s1]), d_flow=None, d_block_start=None,
            d_edges=None, d_loops=None, d_loop_body=None, loop_body_cap=0, d_weights=None, flags=FLOW_FLAGS_DEFAULT)
        rc = rt.lib.ffb_kernel_features(rt.ctx, C.byref(d), rt.stream())
        rt.check(rc, "ffb_kernel_features")
        return FlowResult(feat=out_feat, status=out_status)
    assert lex.ins is not None, "kernel_features needs lex_records() output"
    feat = out_feat if out_feat is not None else rt.empty((K, native.FEAT_WIDTH), torch.float64)
    status = rt.empty((K,), torch.int32)
    res = FlowResult(feat=feat, status=status)
    n_slots = lex.n_ins + 2 * K + 8
    ann_hash = ann_trip = None
    n_ann = 0
    if annotations:
        keys = list(annotations)
        ann_hash = np.asarray([name_hash(k, rt) for k in keys], dtype=np.uint64)
        ann_trip = np.asarray([float(annotations[k]) for k in keys], dtype=np.float64)
        n_ann = len(keys)
        res.ann_hit = torch.zeros(n_ann, dtype=torch.uint8, device=rt.device)
    if detail:
        res.flow = torch.zeros((K, 16), dtype=torch.uint8, device=rt.device)
        res.block_start = torch.zeros(n_slots, dtype=torch.int32, device=rt.device)
        res.edges = torch.zeros((2 * n_slots, 2), dtype=torch.int32, device=rt.device)
        res.loops = torch.zeros((n_slots, 32), dtype=torch.uint8, device=rt.device)
        res.weights = torch.zeros(n_slots, dtype=torch.float64, device=rt.device)
        if K == 1:
            res.loop_body = torch.zeros(max(1, min((lex.n_ins + 1) ** 2, 1 << 26)), dtype=torch.uint8, device=rt.device)
    d = FlowDesc(
        n_segs=K, d_info=native.ptr(lex.info), d_ins_base=native.ptr(lex.ins_base), d_lab_base=native.ptr(lex.lab_base),
        d_ins=native.ptr(lex.ins), d_labels=native.ptr(lex.labels), d_meta=native.ptr(lex.meta), n_ins_total=lex.n_ins,
        n_lab_total=lex.n_lab,
        d_order=native.ptr(corp.order), default_trip=float(default_trip),
        h_ann_hash=ann_hash.ctypes.data if n_ann else None, h_ann_trip=ann_trip.ctypes.data if n_ann else None,
        n_ann=n_ann, d_ann_hit=native.ptr(res.ann_hit), d_feat=native.ptr(feat), d_status=native.ptr(status),
        d_flow=native.ptr(res.flow), d_block_start=native.ptr(res.block_start), d_edges=native.ptr(res.edges),
        d_loops=native.ptr(res.loops), d_loop_body=native.ptr(res.loop_body),
        loop_body_cap=int(res.loop_body.numel()) if res.loop_body is not None else 0, d_weights=native.ptr(res.weights),
        flags=FLOW_FLAGS_DEFAULT)
    rc = rt.lib.ffb_kernel_features(rt.ctx, C.byref(d), rt.stream())
    rt.check(rc, "ffb_kernel_features")
    return res


def analyze_corpus(corp: Corpus, *, default_trip: float = 32.0, rt: native.Runtime | None = None):
    """text -> (LexResult, FlowResult): class histograms + one feature row per kernel."""
    lex = lex_records(corp, rt=rt)
    return lex, kernel_features(corp, lex, default_trip=default_trip, rt=rt)


# ------------------------------------------------------------------------------ bench / smoke helpers
def bench_corpus(seed: int, target_bytes: int, n_kernels: int | None, *, base_kernels: int = 1200,
                 rt: native.Runtime | None = None) -> Corpus:
    """Synthetic corpus of about ``target_bytes``: ``base_kernels`` generated kernels (seeded
    grammar, synth.ptx_corpus) tiled on the device.  With ``n_kernels`` given the kernel count is
    exact and the byte size follows (each kernel is ~40 KB on average)."""
    from . import synth
    if n_kernels is not None:
        base_kernels = min(base_kernels, n_kernels)
        reps = max(1, n_kernels // base_kernels)
        base_kernels = n_kernels // reps
    text, offs = synth.ptx_corpus(seed, base_kernels)
    if n_kernels is None:
        reps = max(1, int(round(target_bytes / max(len(text), 1))))
        if reps == 1 and len(text) > 2 * target_bytes:          # small CPU samples: cut at a kernel boundary
            k = max(1, int(np.searchsorted(offs, target_bytes, side="right")) - 1)
            text, offs = text[: int(offs[k])], offs[: k + 1]
    rt = rt or native.get_runtime()
    n = len(text)
    dev_base = rt.to_device(torch.frombuffer(bytearray(text), dtype=torch.uint8))
    total = n * reps
    padded = (total + 15) // 16 * 16 + 16
    dev = torch.full((padded,), 10, dtype=torch.uint8, device=rt.device)
    dev[:total].view(reps, n).copy_(dev_base.unsqueeze(0).expand(reps, n))
    seg = (offs[None, :-1] + (np.arange(reps, dtype=np.int64) * n)[:, None]).reshape(-1)
    seg = np.concatenate([seg, [total]]).astype(np.int64)
    order = rt.to_device(torch.from_numpy(np.argsort(-np.diff(seg), kind="stable").astype(np.int32)))
    return Corpus(text=dev, n_bytes=total, seg_off=rt.to_device(torch.from_numpy(seg)), n_segs=len(seg) - 1,
                  order=order, host_text=text, host_off=offs)


def _gen_piece(args):
    from . import synth
    seed, first, count, irregular = args
    return synth.ptx_corpus(seed, count, irregular=irregular, first=first)


def generate_unique(seed: int, n_kernels: int, *, irregular: float = 0.0, workers: int | None = None, piece: int = 600):
    """Host side of ``bench_corpus_unique``: [(text, offsets)] pieces of ``piece`` kernels each, produced by a process
    pool (every piece has its own seed, names are unique over the corpus).  Touches no CUDA state, so it can run
    before the device context and the process group exist."""
    import multiprocessing as mp
    import os
    jobs = [(seed * 100_003 + i, i * piece, min(piece, n_kernels - i * piece), irregular) for i in range((n_kernels + piece - 1) // piece)]
    workers = max(1, min(len(jobs), workers or os.cpu_count() or 1))
    with mp.get_context("fork").Pool(workers) as pool:
        return pool.map(_gen_piece, jobs)


def bench_corpus_unique(seed: int, n_kernels: int, *, irregular: float = 0.0, workers: int | None = None, piece: int = 600,
                        rt: native.Runtime | None = None, parts=None) -> Corpus:
    """``n_kernels`` DIFFERENT generated kernels (no tiling), uploaded piece by piece (``parts``: the output of
    ``generate_unique`` when the text was produced earlier).
    ``irregular``: share of kernels with one construct that only the exact walk parses (synth.ptx_corpus)."""
    if parts is None:
        parts = generate_unique(seed, n_kernels, irregular=irregular, workers=workers, piece=piece)
    rt = rt or native.get_runtime()
    total = sum(len(p[0]) for p in parts)
    padded = (total + 15) // 16 * 16 + 16
    dev = torch.full((padded,), 10, dtype=torch.uint8, device=rt.device)
    seg, pos = [np.zeros(1, dtype=np.int64)], 0
    for text, offs in parts:
        dev[pos: pos + len(text)].copy_(rt.to_device(torch.frombuffer(bytearray(text), dtype=torch.uint8)))
        seg.append(offs[1:] + pos)
        pos += len(text)
    seg = np.concatenate(seg).astype(np.int64)
    order = rt.to_device(torch.from_numpy(np.argsort(-np.diff(seg), kind="stable").astype(np.int32)))
    host = b"".join(p[0] for p in parts)
    return Corpus(text=dev, n_bytes=total, seg_off=rt.to_device(torch.from_numpy(seg)), n_segs=len(seg) - 1,
                  order=order, host_text=host, host_off=seg)


def replicated_corpus(unit: bytes, unit_off: np.ndarray, target_bytes: int, rt: native.Runtime | None = None) -> Corpus:
    """``unit`` (a few kernels, e.g. real compiler output) repeated on the device up to about ``target_bytes``."""
    rt = rt or native.get_runtime()
    n = len(unit)
    reps = max(1, int(round(target_bytes / max(n, 1))))
    total = n * reps
    padded = (total + 15) // 16 * 16 + 16
    dev = torch.full((padded,), 10, dtype=torch.uint8, device=rt.device)
    dev[:total].view(reps, n).copy_(rt.to_device(torch.frombuffer(bytearray(unit), dtype=torch.uint8)).unsqueeze(0).expand(reps, n))
    unit_off = np.asarray(unit_off, dtype=np.int64)
    seg = (unit_off[None, :-1] + (np.arange(reps, dtype=np.int64) * n)[:, None]).reshape(-1)
    seg = np.concatenate([seg, [total]]).astype(np.int64)
    order = rt.to_device(torch.from_numpy(np.argsort(-np.diff(seg), kind="stable").astype(np.int32)))
    return Corpus(text=dev, n_bytes=total, seg_off=rt.to_device(torch.from_numpy(seg)), n_segs=len(seg) - 1,
                  order=order, host_text=unit, host_off=unit_off)


def chunk_schedule(total: int, chunk_bytes: int, head_bytes: int = 0, tail_bytes: int = 0) -> list[int]:
    """Target sizes of the upload chunks: an optional small first chunk (the kernels start ``head_bytes`` into the
    upload instead of ``chunk_bytes``), full chunks, then - when ``tail_bytes`` > 0 - chunks that halve down to
    ``tail_bytes``, so that little work is left when the last byte arrives."""
    sizes, left = [], int(total)
    if 0 < head_bytes < left:
        sizes.append(int(head_bytes))
        left -= int(head_bytes)
    while left > 0:
        if tail_bytes > 0:
            size = left if left <= tail_bytes * 3 // 2 else min(chunk_bytes, max(tail_bytes, left // 2))
        else:
            size = min(chunk_bytes, left)
        sizes.append(int(size))
        left -= int(size)
    return sizes


class StreamedAnalysis:
    """text in PINNED HOST memory -> feature rows, with the host->device copy overlapped with the
    kernels: the corpus is cut at segment boundaries into chunks (``chunk_schedule``); a copy
    stream uploads chunk c+1 while chunk c runs K1 (single-pass record mode) and K1b.  With
    ``pipelines`` > 1 the chunks alternate between that many compute streams, each with its own
    libffb context (scratch, work queues): every launch ends with a few long kernels on one warp
    each, and the next chunk's launches fill the SMs those tails leave idle.  Results are
    identical to ``analyze_corpus`` on the resident text."""

    def __init__(self, rt: native.Runtime, corp: Corpus, host_text: torch.Tensor, *, chunk_bytes: int = 384 << 20,
                 lex: LexResult | None = None, feat: torch.Tensor | None = None, pipelines: int = 1,
                 head_bytes: int = 0, tail_bytes: int = 0):
        assert host_text.is_pinned() and host_text.numel() == corp.padded_bytes
        self.rt, self.corp, self.host = rt, corp, host_text
        seg = corp.seg_off.cpu().numpy()
        bounds, s0 = [], 0
        for size in chunk_schedule(int(seg[-1]), chunk_bytes, head_bytes, tail_bytes):
            if s0 >= corp.n_segs:
                break
            s1 = int(np.searchsorted(seg, seg[s0] + size, side="left"))
            s1 = min(max(s1, s0 + 1), corp.n_segs)
            bounds.append((s0, s1))
            s0 = s1
        if s0 < corp.n_segs:
            bounds.append((s0, corp.n_segs))
        self.bounds = bounds
        # copy ranges: 16-byte aligned supersets of the chunks' bytes (neighbouring bytes are re-sent, harmless)
        self.ranges = [(int(seg[a]) // 16 * 16, min((int(seg[b]) + 15) // 16 * 16 + 16, corp.padded_bytes)) for a, b in bounds]
        self.orders = [rt.to_device(torch.from_numpy(np.argsort(-np.diff(seg[a:b + 1]), kind="stable").astype(np.int32)))
                       for a, b in bounds]
        self.lex = lex if lex is not None else lex_records_single_pass(corp, rt=rt)
        self.feat = feat if feat is not None else rt.empty((corp.n_segs, native.FEAT_WIDTH), torch.float64)
        self.status = rt.empty((corp.n_segs,), torch.int32)
        cuda = rt.device.type == "cuda"
        self.copy_stream = torch.cuda.Stream(device=rt.device) if cuda else None
        self.events = [torch.cuda.Event() for _ in bounds] if cuda else []
        # compute pipelines: (runtime, stream); pipeline 0 is the caller's runtime on the caller's stream
        self.pipes = [(rt, None)]
        if cuda:
            for _ in range(1, max(1, int(pipelines))):
                self.pipes.append((native.Runtime(native.load_library(), rt.device, rt.device.index or 0),
                                   torch.cuda.Stream(device=rt.device)))

    def run(self, default_trip: float = 32.0, on_chunk=None, timeline: list | None = None) -> torch.Tensor:
        """``on_chunk(c, s0, s1, rt)`` runs on the chunk's compute stream (the current stream during the
        call) right after chunk c's feature rows are enqueued, with the runtime whose scratch that
        stream owns (e.g. to score and rank those kernels while later chunks are still uploading).
        ``timeline``: when a list, timing events are appended as (label, event) - one after every chunk's
        upload (copy stream) and after its lexer / dataflow / on_chunk work (compute stream)."""
        rt, corp = self.rt, self.corp

        def mark(label, stream=None):
            if timeline is not None:
                ev = torch.cuda.Event(enable_timing=True)
                ev.record(stream if stream is not None else torch.cuda.current_stream(rt.device))
                timeline.append((label, ev))

        main = None
        if self.copy_stream is not None:
            main = torch.cuda.current_stream(rt.device)
            mark("start")
            self.copy_stream.wait_stream(main)            # earlier readers of the text buffer are done
            for _, st in self.pipes[1:]:
                st.wait_stream(main)
            with torch.cuda.stream(self.copy_stream):
                for c, ((lo, hi), ev) in enumerate(zip(self.ranges, self.events)):
                    corp.text[lo:hi].copy_(self.host[lo:hi], non_blocking=True)
                    ev.record(self.copy_stream)
                    mark(f"h2d[{c}]", self.copy_stream)
        else:
            corp.text.copy_(self.host)
        for c, (s0, s1) in enumerate(self.bounds):
            rt_c, st = self.pipes[c % len(self.pipes)]
            with (torch.cuda.stream(st) if st is not None else contextlib.nullcontext()):
                if self.copy_stream is not None:
                    torch.cuda.current_stream(rt.device).wait_event(self.events[c])
                lex_records_single_pass(corp, out=self.lex, rt=rt_c, seg_range=(s0, s1), order=self.orders[c])
                mark(f"lex[{c}]")
                kernel_features(corp, self.lex, default_trip=default_trip, out_feat=self.feat, out_status=self.status, rt=rt_c,
                                seg_range=(s0, s1), order=self.orders[c])
                mark(f"flow[{c}]")
                if on_chunk is not None:
                    on_chunk(c, s0, s1, rt_c)
                    mark(f"score+front[{c}]")
        for _, st in self.pipes[1:]:
            main.wait_stream(st)                          # the caller's stream sees every chunk's results
        return self.feat


class BenchLexState:
    """Preallocated buffers so the timed loop launches kernels only: ONE lexer pass in
    single-pass record mode (slots sized from the segment lengths, nothing is learnt from a
    previous pass over the same text) followed by the dataflow kernel."""

    def __init__(self, rt: native.Runtime, corp: Corpus, chunk_bytes: int = 384 << 20, pipelines: int = 1,
                 head_bytes: int = 0, tail_bytes: int = 0):
        self.rt, self.corp, self.chunk_bytes = rt, corp, chunk_bytes
        self.pipelines, self.head_bytes, self.tail_bytes = pipelines, head_bytes, tail_bytes
        self.lex = lex_records_single_pass(corp, rt=rt)
        self.feat = rt.empty((corp.n_segs, native.FEAT_WIDTH), torch.float64)
        self.host_text = None
        self.streamed = None

    def pin_host(self):
        if self.host_text is None:
            self.host_text = torch.empty(self.corp.padded_bytes, dtype=torch.uint8).pin_memory()
            self.host_text.copy_(self.corp.text)
        return self.host_text

    def run(self, resident: bool = True, mark=None, on_chunk=None, timeline: list | None = None) -> torch.Tensor:
        rt, corp = self.rt, self.corp
        if not resident:
            # host text -> feature rows through the public streamed path: H2D inside the timed
            # region, overlapped chunk by chunk with K1 / K1b
            if self.streamed is None:
                self.streamed = StreamedAnalysis(rt, corp, self.pin_host(), lex=self.lex, feat=self.feat, chunk_bytes=self.chunk_bytes,
                                                 pipelines=self.pipelines, head_bytes=self.head_bytes, tail_bytes=self.tail_bytes)
            self.streamed.run(on_chunk=on_chunk, timeline=timeline)
            if mark is not None:
                mark.record()
            return self.feat
        lex_records_single_pass(corp, out=self.lex, rt=rt)                # K1: histogram + records
        if mark is not None:
            mark.record()
        kernel_features(corp, self.lex, out_feat=self.feat, rt=rt)        # K1b
        return self.feat


# ------------------------------------------------------------------------------ multi-kernel modules
def split_modules(text: bytes, module_off: np.ndarray | None = None, *, max_kernels_per_module: int = 1 << 16,
                  rt: native.Runtime | None = None) -> Corpus:
    """One corpus segment per ``.entry`` kernel of every module.

    The reference parses ONE kernel per ``parse_ptx`` call (first or named, ptx.py:168-184); here
    round i lexes the i-th kernel of every module at once (histogram mode stops at the closing
    brace of the kernel body) and the next round resumes right behind it, so the whole corpus is
    read once.  Segment k then behaves like ``parse_ptx(module, kernel_name=<k-th name>)`` — same
    instructions, labels and features; only ``source_line`` is relative to the segment.
    """
    rt = rt or native.get_runtime()
    n = len(text)
    module_off = np.asarray([0, n] if module_off is None else module_off, dtype=np.int64)
    whole = upload_corpus(text, module_off, balance=False, rt=rt)
    starts, ends = module_off[:-1].copy(), module_off[1:].copy()
    alive = np.arange(len(starts))
    pieces: list[tuple[int, int, int]] = []          # (module, start, stop)
    for _ in range(max_kernels_per_module):
        if alive.size == 0:
            break
        seg = np.empty(2 * alive.size, dtype=np.int64)
        seg[0::2], seg[1::2] = starts[alive], ends[alive]
        # alternate "kernel remainder" / "gap" segments keep the table ascending; gaps are empty or ignored
        table = np.concatenate([seg, [ends[alive[-1]]]])
        round_corp = Corpus(text=whole.text, n_bytes=whole.n_bytes, seg_off=rt.to_device(torch.from_numpy(table)),
                            n_segs=len(table) - 1, order=None)
        info = lex_histogram(round_corp, rt=rt).info_np()[0::2]
        nxt = []
        for m, inf in zip(alive, info):
            if int(inf["status"]) == 2:              # NoKernelFound: module exhausted
                continue
            if int(inf["status"]) != 0 or int(inf["body_end"]) == 0:
                # malformed kernel: keep the remainder as one segment so the error is reported, stop this module
                pieces.append((int(m), int(starts[m]), int(ends[m])))
                continue
            stop = int(starts[m]) + int(inf["body_end"]) + 1
            pieces.append((int(m), int(starts[m]), stop))
            starts[m] = stop
            nxt.append(m)
        alive = np.asarray(nxt, dtype=np.int64)
    pieces.sort(key=lambda p: p[1])
    if not pieces:
        return Corpus(text=whole.text, n_bytes=n, seg_off=rt.to_device(torch.zeros(1, dtype=torch.int64)), n_segs=0)
    # consecutive pieces of one module are contiguous; pieces of different modules may leave gaps,
    # which become (kernel-less) segments of their own so that the table stays a partition
    bounds = [pieces[0][1]]
    keep = []
    for _, a, b in pieces:
        if a != bounds[-1]:
            bounds.append(a)
            keep.append(False)
        bounds.append(b)
        keep.append(True)
    seg_off = np.asarray(bounds, dtype=np.int64)
    corp = Corpus(text=whole.text, n_bytes=n, seg_off=rt.to_device(torch.from_numpy(seg_off)), n_segs=len(seg_off) - 1,
                  host_text=text, host_off=seg_off)
    corp.kernel_mask = np.asarray(keep, dtype=bool)      # False for gap segments
    return corp
