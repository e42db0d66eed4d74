"""Batched corpus entry points: PTX text on the device -> histograms, declarations,
instruction records and per-kernel dynamic feature rows (K1 + K1b).

A corpus is one byte buffer plus a segment table; segment k is analysed exactly like
``parse_ptx(text[seg_off[k]:seg_off[k+1]])`` of the reference (ptx.py:207).
"""
from __future__ import annotations

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
MAX_SPAN_OPS, MAX_DECLS = 12, 32
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
        ("d_ins", C.c_void_p), ("d_labels", C.c_void_p), ("d_spans", C.c_void_p), ("d_decls", C.c_void_p),
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
    spans: torch.Tensor | None = None    # uint8 [N, 128]
    decls: torch.Tensor | None = None    # uint8 [K, 32, 16]
    n_ins: int = 0
    n_lab: int = 0

    def info_np(self) -> np.ndarray:
        return self.info.cpu().numpy().view(SEG_DTYPE).reshape(-1)

    def info_i32(self) -> torch.Tensor:
        return self.info.view(torch.int32).view(-1, 12)


def _call_lex(rt, corp: Corpus, hist, info, *, kernel_name: bytes | None = None, ins_base=None, lab_base=None,
              ins=None, labels=None, spans=None, decls=None):
    d = LexDesc(
        d_text=native.ptr(corp.text), n_bytes=corp.padded_bytes, d_seg_off=native.ptr(corp.seg_off),
        n_segs=corp.n_segs, d_order=native.ptr(corp.order),
        h_kernel_name=kernel_name, kernel_name_len=len(kernel_name) if kernel_name else 0,
        d_hist=native.ptr(hist), d_info=native.ptr(info), d_ins_base=native.ptr(ins_base),
        d_lab_base=native.ptr(lab_base), d_ins=native.ptr(ins), d_labels=native.ptr(labels),
        d_spans=native.ptr(spans), d_decls=native.ptr(decls))
    rc = rt.lib.ffb_lex_corpus(rt.ctx, C.byref(d), rt.stream())
    rt.check(rc, "ffb_lex_corpus")


def lex_histogram(corp: Corpus, *, kernel_name: str | None = None, out: LexResult | None = None,
                  rt: native.Runtime | None = None) -> LexResult:
    """K1, histogram mode: class counts, declarations, status per segment.  No sync."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    res = out or LexResult(hist=rt.empty((K, native.N_CLASSES), torch.int32), info=rt.empty((K, 48), torch.uint8))
    _call_lex(rt, corp, res.hist, res.info, kernel_name=kernel_name.encode() if kernel_name else None)
    return res


def lex_records(corp: Corpus, *, kernel_name: str | None = None, spans: bool = False, decls: bool = False,
                rt: native.Runtime | None = None) -> LexResult:
    """K1, record mode (two passes: counts, then 64-byte instruction records).  Syncs once
    to size the record buffers."""
    rt = rt or native.get_runtime()
    K = corp.n_segs
    name = kernel_name.encode() if kernel_name else None
    res = lex_histogram(corp, kernel_name=kernel_name, rt=rt)
    counts = res.info_i32()[:, 1:3].to(torch.int64)
    incl = torch.cumsum(counts, dim=0)
    base = (incl - counts).contiguous()
    totals = incl[-1].cpu() if K else torch.zeros(2, dtype=torch.int64)
    res.n_ins, res.n_lab = int(totals[0]), int(totals[1])
    res.ins_base, res.lab_base = base[:, 0].contiguous(), base[:, 1].contiguous()
    res.ins = rt.empty((max(res.n_ins, 1), 64), torch.uint8)
    res.labels = rt.empty((max(res.n_lab, 1), 16), torch.uint8)
    res.spans = torch.zeros((max(res.n_ins, 1), 128), dtype=torch.uint8, device=rt.device) if spans else None
    res.decls = torch.zeros((K, MAX_DECLS, 16), dtype=torch.uint8, device=rt.device) if decls else None
    _call_lex(rt, corp, res.hist, res.info, kernel_name=name, ins_base=res.ins_base, lab_base=res.lab_base,
              ins=res.ins, labels=res.labels, spans=res.spans, decls=res.decls)
    return res


def raise_segment_status(status: int, what: str = "PTX segment") -> None:
    raise_for_status(int(status), what)
