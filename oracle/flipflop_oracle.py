"""CPU oracle for the FlipFlop analysis path — TEST INFRASTRUCTURE ONLY.

A from-scratch restatement, in plain Python + numpy, of what the reference package
(`/root/reference/pkg/src/ptxwatt`, pure Python) computes on the hot path.  It exists so
that the CUDA kernels can be checked on the GPU box, where the reference itself is not
present.  Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs may import
it; nothing under paper_2601_13345_b200/ does.

Parity status: PINNED.  tests/test_oracle_golden.py checks every function here against
(a) the reference's own golden vectors (manifest.json hand counts, the classification /
trip / alignment / model known-answer values copied into tests/golden/ref_kats.json with
their source lines) and (b) outputs of the reference itself, generated in the build
container by tests/golden/make_golden.py (committed next to its outputs).

Each function cites the reference lines it restates.  Where the reference leans on `re`,
this file uses explicit character scanning — the same formulation the GPU lexer uses — so
agreement with the regex-based reference is a real check, not a tautology.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

CLASSES = ("MemLoad", "MemStore", "FP32", "INT", "SFU", "ALU", "Sync", "Branch", "Other")
UNITS = ("FP32", "INT", "SFU", "ALU", "Mem")

# Python's str.strip()/split() whitespace restricted to ASCII, which is also what `\s`
# matches for str patterns: \t \n \v \f \r, FS GS RS US, space.
WS = frozenset("\t\n\x0b\x0c\r\x1c\x1d\x1e\x1f ")
_WORD = frozenset("abcdefghijklmnopqrstuvwxyzABCDEFGHIJKLMNOPQRSTUVWXYZ0123456789_")

_TYPE_BYTES = {"b8": 1, "s8": 1, "u8": 1, "b16": 2, "s16": 2, "u16": 2, "f16": 2, "bf16": 2,
               "b32": 4, "s32": 4, "u32": 4, "f32": 4, "b64": 8, "s64": 8, "u64": 8, "f64": 8}


class OracleError(Exception):
    def __init__(self, kind: str, msg: str = ""):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# ------------------------------------------------------------------ a1: comments
def clean_comments(src: str) -> str:
    """ptx.py:139-141.  Pass 1: every ``/* ... */`` (leftmost, shortest, only if a closing
    ``*/`` exists) becomes spaces with newlines kept.  Pass 2: ``//`` to end of line is
    removed.  Returned text has line comments replaced by nothing, like the reference."""
    out = []
    i, n = 0, len(src)
    while i < n:
        if src[i] == "/" and i + 1 < n and src[i + 1] == "*":
            close = src.find("*/", i + 2)
            if close >= 0:
                out.extend("\n" if ch == "\n" else " " for ch in src[i:close + 2])
                i = close + 2
                continue
        out.append(src[i])
        i += 1
    mid = "".join(out)
    out = []
    i, n = 0, len(mid)
    while i < n:
        if mid[i] == "/" and i + 1 < n and mid[i + 1] == "/":
            while i < n and mid[i] != "\n":
                i += 1
            continue
        out.append(mid[i])
        i += 1
    return "".join(out)


# ------------------------------------------------------------------ a2: kernel location
def _is_name_start(ch: str) -> bool:
    return ch.isalpha() and ch.isascii() or ch in "_$"


def _is_name_char(ch: str) -> bool:
    return ch in _WORD or ch == "$"


def entry_matches(clean: str):
    """Yield (name, end_of_match) for every ``.entry <ws>+ NAME`` (ptx.py:33; the optional
    .visible/.weak prefix does not change where the name or the match end is)."""
    pos = 0
    while True:
        k = clean.find(".entry", pos)
        if k < 0:
            return
        j = k + 6
        q = j
        while q < len(clean) and clean[q] in WS:
            q += 1
        if q > j and q < len(clean) and _is_name_start(clean[q]):
            r = q + 1
            while r < len(clean) and _is_name_char(clean[r]):
                r += 1
            yield clean[q:r], r
            pos = r
        else:
            pos = k + 1


def locate_kernel(clean: str, wanted: str | None = None):
    """ptx.py:165-187 -> (name, body_start, body_end); body excludes the outer braces."""
    seen = []
    for name, end in entry_matches(clean):
        seen.append(name)
        if wanted is not None and name != wanted:
            continue
        brace = clean.find("{", end)
        if brace < 0:
            raise OracleError("MalformedPtx", f"kernel {name!r} has no body")
        depth = 0
        for i in range(brace, len(clean)):
            ch = clean[i]
            if ch == "{":
                depth += 1
            elif ch == "}":
                depth -= 1
                if depth == 0:
                    return name, brace + 1, i
        raise OracleError("MalformedPtx", f"unbalanced braces in kernel {name!r}")
    if wanted is not None and seen:
        raise OracleError("NoKernelFound", f"kernel {wanted!r} not found")
    raise OracleError("NoKernelFound", "no .entry kernel in source")


# ------------------------------------------------------------------ a5/a6: classification
def classify(opcode: str):
    """ptx.py:99-136 -> (class, space).  Order of the tests matters."""
    toks = opcode.split(".")
    base, rest = toks[0], toks[1:]
    if base in ("bar", "barrier") or opcode.endswith(".sync"):
        return "Sync", "none"
    if base in ("ld", "ldu", "st"):
        space = "none"
        for tk in rest:
            if tk in ("global", "shared", "local", "param", "const"):
                space = "param" if tk == "const" else tk
                break
        return ("MemStore" if base == "st" else "MemLoad"), space
    if base == "bra":
        return "Branch", "none"
    if base in ("add", "sub", "mul", "mad", "fma", "div"):
        if any(tk in ("f32", "f64") for tk in rest):
            return "FP32", "none"
        if any(tk in ("s32", "u32", "s64", "u64") for tk in rest):
            return "INT", "none"
        return "Other", "none"
    if base in ("sin", "cos", "ex2", "lg2", "rcp", "rsqrt"):
        return "SFU", "none"
    if base == "sqrt" and "approx" in toks:
        return "SFU", "none"
    if base in ("mov", "setp", "and", "or", "shl", "shr", "cvt", "selp"):
        return "ALU", "none"
    return "Other", "none"


def access_bytes(opcode: str) -> int:
    """ptx.py:64-76: LAST type suffix (default 4) times LAST v2/v4 (default 1)."""
    elem, vec = 4, 1
    for tk in opcode.split(".")[1:]:
        if tk in _TYPE_BYTES:
            elem = _TYPE_BYTES[tk]
        if tk == "v2":
            vec = 2
        elif tk == "v4":
            vec = 4
    return elem * vec


# ------------------------------------------------------------------ a3/a4/a7: statements
@dataclass
class Ins:
    opcode: str
    cls: str
    space: str
    operands: tuple
    pred: str | None
    line: int

    @property
    def base(self):
        return self.opcode.split(".", 1)[0]


@dataclass
class Kernel:
    name: str
    params: tuple
    regs: dict
    shared: int
    ins: list = field(default_factory=list)
    labels: dict = field(default_factory=dict)


def _strip(s: str) -> str:
    a, b = 0, len(s)
    while a < b and s[a] in WS:
        a += 1
    while b > a and s[b - 1] in WS:
        b -= 1
    return s[a:b]


def split_operands(text: str) -> tuple:
    """ptx.py:144-162: commas at bracket depth 0 split; pieces are stripped; empties dropped."""
    parts, cur, depth = [], [], 0
    for ch in text:
        if ch in "[{(":
            depth += 1
        elif ch in "]})":
            depth -= 1
        if ch == "," and depth == 0:
            parts.append(_strip("".join(cur)))
            cur = []
        else:
            cur.append(ch)
    parts.append(_strip("".join(cur)))
    return tuple(p for p in parts if p)


def _label_prefix(line: str):
    """ptx.py:41 `^([\\w$.]+):\\s*` -> (label, rest) or None."""
    k = 0
    while k < len(line) and (line[k] in _WORD or line[k] in "$."):
        k += 1
    if k == 0 or k >= len(line) or line[k] != ":":
        return None
    r = k + 1
    while r < len(line) and line[r] in WS:
        r += 1
    return line[:k], line[r:]


def _scan_ws(s, i):
    while i < len(s) and s[i] in WS:
        i += 1
    return i


def _scan_word(s, i, extra=""):
    j = i
    while j < len(s) and (s[j] in _WORD or s[j] in extra):
        j += 1
    return j


def _scan_digits(s, i):
    j = i
    while j < len(s) and s[j] in "0123456789":
        j += 1
    return j


def _reg_decl(stmt: str):
    """ptx.py:37 `^\\.reg\\s+\\.(\\w+)\\s+%[A-Za-z_]+<(\\d+)>\\s*;?$` on stmt (no ';' inside)."""
    if not stmt.startswith(".reg"):
        return None
    i = _scan_ws(stmt, 4)
    if i == 4 or i >= len(stmt) or stmt[i] != ".":
        return None
    j = _scan_word(stmt, i + 1)
    if j == i + 1:
        return None
    cls = stmt[i + 1:j]
    k = _scan_ws(stmt, j)
    if k == j or k >= len(stmt) or stmt[k] != "%":
        return None
    m = k + 1
    while m < len(stmt) and (stmt[m].isascii() and stmt[m].isalpha() or stmt[m] == "_"):
        m += 1
    if m == k + 1 or m >= len(stmt) or stmt[m] != "<":
        return None
    d = _scan_digits(stmt, m + 1)
    if d == m + 1 or d >= len(stmt) or stmt[d] != ">":
        return None
    if _scan_ws(stmt, d + 1) != len(stmt):
        return None
    return cls, int(stmt[m + 1:d])


def _shared_decl(stmt: str):
    """ptx.py:38-40 `^\\.shared\\s+(?:\\.align\\s+\\d+\\s+)?\\.(\\w+)\\s+[\\w$]+(?:\\[(\\d+)\\])?\\s*;?$`."""
    if not stmt.startswith(".shared"):
        return None
    i = _scan_ws(stmt, 7)
    if i == 7:
        return None
    if stmt.startswith(".align", i):
        a = _scan_ws(stmt, i + 6)
        b = _scan_digits(stmt, a)
        c = _scan_ws(stmt, b)
        if a > i + 6 and b > a and c > b:
            i = c       # the optional group matched; otherwise fall through and fail below
    if i >= len(stmt) or stmt[i] != ".":
        return None
    j = _scan_word(stmt, i + 1)
    if j == i + 1:
        return None
    ty = stmt[i + 1:j]
    k = _scan_ws(stmt, j)
    if k == j:
        return None
    m = _scan_word(stmt, k, "$")
    if m == k:
        return None
    count = 1
    if m < len(stmt) and stmt[m] == "[":
        d = _scan_digits(stmt, m + 1)
        if d == m + 1 or d >= len(stmt) or stmt[d] != "]":
            return None
        count = int(stmt[m + 1:d])
        m = d + 1
    if _scan_ws(stmt, m) != len(stmt):
        return None
    return _TYPE_BYTES.get(ty, 1) * count


def _params(clean: str, name: str, body_start: int) -> tuple:
    """ptx.py:190-204.  Regex `\\.param\\s+(?:\\.align\\s+\\d+\\s+)?\\.(\\w+)\\s+([\\w$]+)(?:\\[(\\d+)\\])?`."""
    h0 = clean.rfind(".entry", 0, body_start)
    header = clean[h0:body_start]
    lp = header.find("(")
    if lp < 0:
        return ()
    rp = header.find(")", lp)
    if rp < 0:
        raise OracleError("MalformedPtx", f"kernel {name!r}: unterminated parameter list")
    text = header[lp:rp]
    out, pos = [], 0
    while True:
        k = text.find(".param", pos)
        if k < 0:
            break
        pos = k + 1
        i = _scan_ws(text, k + 6)
        if i == k + 6:
            continue
        if text.startswith(".align", i):
            a = _scan_ws(text, i + 6)
            b = _scan_digits(text, a)
            c = _scan_ws(text, b)
            if a > i + 6 and b > a and c > b:
                i = c
        if i >= len(text) or text[i] != ".":
            continue
        j = _scan_word(text, i + 1)
        if j == i + 1:
            continue
        ty = text[i + 1:j]
        q = _scan_ws(text, j)
        if q == j:
            continue
        m = _scan_word(text, q, "$")
        if m == q:
            continue
        pname = text[q:m]
        arr = None
        if m < len(text) and text[m] == "[":
            d = _scan_digits(text, m + 1)
            if d > m + 1 and d < len(text) and text[d] == "]":
                arr = int(text[m + 1:d])
                m = d + 1
        elem = _TYPE_BYTES.get(ty, 0)
        out.append((pname, "param", arr * elem if arr is not None else elem))
        pos = m
    return tuple(out)


def parse_kernel(src: str, wanted: str | None = None) -> Kernel:
    """ptx.py:207-293."""
    clean = clean_comments(src)
    name, b0, b1 = locate_kernel(clean, wanted)
    kern = Kernel(name=name, params=_params(clean, name, b0), regs={}, shared=0)
    first_line = clean.count("\n", 0, b0) + 1
    pending, pending_line, has_pending = "", first_line, False
    for off, raw in enumerate(clean[b0:b1].split("\n")):
        lineno = first_line + off
        line = _strip(raw)
        while line:
            if not has_pending:
                lab = _label_prefix(line)
                if lab is not None:
                    kern.labels[lab[0]] = len(kern.ins)
                    line = _strip(lab[1])
                    continue
                if line == "{" or line == "}":
                    break
                if line[0] == ".":
                    semi = line.find(";")
                    stmt = _strip(line if semi < 0 else line[:semi])
                    line = "" if semi < 0 else _strip(line[semi + 1:])
                    rd = _reg_decl(stmt)
                    if rd is not None:
                        kern.regs[rd[0]] = kern.regs.get(rd[0], 0) + rd[1]
                        continue
                    sd = _shared_decl(stmt)
                    if sd is not None:
                        kern.shared += sd
                    continue
            semi = line.find(";")
            if semi < 0:
                if not has_pending:
                    pending_line, has_pending = lineno, True
                pending += " " + line
                break
            stmt, line = line[:semi], _strip(line[semi + 1:])
            full = _strip(pending + " " + stmt)
            at = pending_line if has_pending else lineno
            pending, has_pending = "", False
            if full:
                kern.ins.append(_instruction(full, at))
    if _strip(pending):
        raise OracleError("MalformedPtx", f"kernel {name!r}: unterminated statement")
    if not kern.ins:
        raise OracleError("MalformedPtx", f"kernel {name!r} has an empty body")
    for ins in kern.ins:
        if ins.cls == "Branch":
            tgt = ins.operands[-1] if ins.operands else ""
            if tgt not in kern.labels:
                raise OracleError("MalformedPtx", f"branch to undefined label {tgt!r} (line {ins.line})")
    return kern


def _instruction(text: str, line: int) -> Ins:
    """ptx.py:296-313; predicate regex `^@(!?%[\\w$]+)\\s+`."""
    pred = None
    if text[0] == "@":
        i = 1
        if i < len(text) and text[i] == "!":
            i += 1
        if i < len(text) and text[i] == "%":
            j = _scan_word(text, i + 1, "$")
            k = _scan_ws(text, j)
            if j > i + 1 and k > j:
                pred = text[1:j]
                text = _strip(text[k:])
    i = 0
    while i < len(text) and text[i] not in WS:
        i += 1
    opcode = text[:i]
    rest = text[i:]
    # str.split(None, 1): a second part exists only when something non-blank follows
    ops = split_operands(rest) if _strip(rest) else ()
    cls, space = classify(opcode)
    return Ins(opcode, cls, space, ops, pred, line)


# ------------------------------------------------------------------ a8: CFG and loops
def build_blocks(k: Kernel):
    """cfg.py:57-151 -> (blocks, edges, loops[(header, frozenset body, header_label)])."""
    n = len(k.ins)
    leaders = {0} | {i for i in k.labels.values() if i < n}
    for i, ins in enumerate(k.ins):
        if (ins.cls == "Branch" or ins.base in ("ret", "exit")) and i + 1 < n:
            leaders.add(i + 1)
    starts = sorted(leaders)
    blocks = [(s, starts[j + 1] if j + 1 < len(starts) else n) for j, s in enumerate(starts)]
    at = {s: j for j, (s, _) in enumerate(blocks)}
    edges = []
    for b, (_, end) in enumerate(blocks):
        last = k.ins[end - 1]
        if last.cls == "Branch":
            tgt = k.labels[last.operands[-1]]
            if tgt < n:
                edges.append((b, at[tgt]))
            if last.pred is not None and b + 1 < len(blocks):
                edges.append((b, b + 1))
        elif last.base in ("ret", "exit"):
            continue
        elif b + 1 < len(blocks):
            edges.append((b, b + 1))
    nb = len(blocks)
    preds = [[] for _ in range(nb)]
    for u, v in edges:
        preds[v].append(u)
    everything = (1 << nb) - 1
    dom = [everything] * nb
    dom[0] = 1
    changed = True
    while changed:
        changed = False
        for b in range(1, nb):
            acc = everything
            for p in preds[b]:
                acc &= dom[p]
            acc |= 1 << b
            if acc != dom[b]:
                dom[b], changed = acc, True
    bodies = {}
    for u, h in edges:
        if not (dom[u] >> h) & 1:
            continue
        body, stack = {h, u}, [u]
        while stack:
            x = stack.pop()
            if x == h:
                continue
            for p in preds[x]:
                if p not in body:
                    body.add(p)
                    stack.append(p)
        bodies.setdefault(h, set()).update(body)
    label_at = {}
    for nm, idx in k.labels.items():
        label_at[idx] = nm          # later definitions of the same index win, as dict order does
    loops = [(h, frozenset(bodies[h]), label_at.get(blocks[h][0])) for h in sorted(bodies)]
    return blocks, edges, loops


# ------------------------------------------------------------------ a9: trip counts
def py_int_literal(text: str):
    """Python ``int(text, 0)`` or None."""
    try:
        return int(text, 0)
    except ValueError:
        return None


_INVERT = {"lt": "ge", "ge": "lt", "le": "gt", "gt": "le", "eq": "ne", "ne": "eq"}


def detect_trip(k: Kernel, blocks, loop):
    """cfg.py:191-279; returns float or None."""
    header, body, _ = loop
    h0 = blocks[header][0]
    idxs = [i for b in sorted(body) for i in range(*blocks[b])]
    latch = None
    for i in idxs:
        ins = k.ins[i]
        if ins.cls == "Branch" and ins.pred is not None and k.labels.get(ins.operands[-1]) == h0:
            latch = ins
    if latch is None:
        return None
    neg = latch.pred.startswith("!")
    preg = latch.pred.lstrip("!")
    cmp_ins = None
    for i in idxs:
        ins = k.ins[i]
        if ins.base == "setp" and ins.operands and ins.operands[0] == preg:
            cmp_ins = ins
    if cmp_ins is None or len(cmp_ins.operands) < 3:
        return None
    counter, bound = cmp_ins.operands[1], py_int_literal(cmp_ins.operands[2])
    if bound is None or not counter.startswith("%"):
        return None
    rel = next((tk for tk in cmp_ins.opcode.split(".") if tk in _INVERT), None)
    if rel is None:
        return None
    if neg:
        rel = _INVERT[rel]
    stride = None
    for i in idxs:
        ins = k.ins[i]
        if ins.base in ("add", "sub") and len(ins.operands) == 3 \
                and ins.operands[0] == counter and ins.operands[1] == counter:
            imm = py_int_literal(ins.operands[2])
            if imm is None or stride is not None:
                return None
            stride = -imm if ins.base == "sub" else imm
    if not stride:
        return None
    init = None
    for i in range(h0):
        ins = k.ins[i]
        if ins.operands and ins.operands[0] == counter:
            init = py_int_literal(ins.operands[1]) if (ins.base == "mov" and len(ins.operands) == 2) else None
    if init is None:
        return None
    if rel == "lt" and stride > 0:
        trips = math.ceil((bound - init) / stride)
    elif rel == "le" and stride > 0:
        trips = math.floor((bound - init) / stride) + 1
    elif rel == "gt" and stride < 0:
        trips = math.ceil((init - bound) / -stride)
    elif rel == "ge" and stride < 0:
        trips = math.floor((init - bound) / -stride) + 1
    elif rel == "ne":
        span = bound - init
        if span % stride == 0 and span // stride > 0:
            trips = span // stride
        else:
            return None
    else:
        return None
    return float(max(1, trips))


def loop_trips(k: Kernel, blocks, loops, default_trip=32.0, annotations=None):
    """cfg.py:154-182 -> list of trips; raises AnnotationForUnknownLoop."""
    annotations = dict(annotations or {})
    known = {lab for _, _, lab in loops if lab}
    for key in annotations:
        if key not in known:
            raise OracleError("AnnotationForUnknownLoop", key)
    out = []
    for loop in loops:
        if loop[2] in annotations:
            trip = float(annotations[loop[2]])
        else:
            d = detect_trip(k, blocks, loop)
            trip = d if d is not None else float(default_trip)
        out.append(max(1.0, trip))
    return out


def block_weights(blocks, loops, trips):
    w = [1.0] * len(blocks)
    for (_, body, _), trip in zip(loops, trips):
        for b in body:
            w[b] *= trip
    return w


# ------------------------------------------------------------------ a10: alignment
def _ends_uniform_special(op: str) -> bool:
    """alignment.py:17-19 searched with $-anchors."""
    if op.endswith("%gridid") or op.endswith("WARP_SZ"):
        return True
    if len(op) >= 2 and op[-1] in "xyz" and op[-2] == ".":
        stem = op[:-2]
        return stem.endswith("%ctaid") or stem.endswith("%nctaid") or stem.endswith("%ntid")
    return False


def operand_scale(op: str, scales: dict):
    """alignment.py:31-47."""
    if op == "%tid.x":
        return 1
    if op.startswith("%tid.") or op in ("%laneid", "%warpid"):
        return None
    if _ends_uniform_special(op):
        return 0
    if op.startswith("%"):
        return scales.get(op)
    return 0


def _mul_scale(a, b, scales):
    sa, sb = operand_scale(a, scales), operand_scale(b, scales)
    ia, ib = py_int_literal(a), py_int_literal(b)
    if sa == 0 and sb == 0:
        return 0
    if ib is not None and sa is not None:
        return sa * ib
    if ia is not None and sb is not None:
        return ia * sb
    return None


def address_base(addr: str):
    """alignment.py:21 `^\\[\\s*([^\\]+]+?)\\s*(?:\\+\\s*-?\\d+)?\\s*\\]$` -> stripped base or None."""
    if len(addr) < 2 or addr[0] != "[" or addr[-1] != "]":
        return None
    inner = addr[1:-1]
    if "]" in inner:
        return None
    plus = inner.find("+")
    left, right = (inner, None) if plus < 0 else (inner[:plus], inner[plus + 1:])
    if not left:
        return None
    base = _strip(left)     # an all-blank interior still matches the regex: group(1) = one blank
    if right is not None:
        r = _strip(right)
        if r.startswith("-"):
            r = r[1:]
        if not r or any(ch not in "0123456789" for ch in r):
            return None
    return base


def address_scales(k: Kernel) -> dict:
    """alignment.py:61-125."""
    scales, out = {}, {}
    for idx, ins in enumerate(k.ins):
        ops = ins.operands
        if ins.cls in ("MemLoad", "MemStore"):
            addr = next((o for o in ops if o.startswith("[")), None)
            if addr is not None:
                base = address_base(addr)
                if base is None:
                    out[idx] = None
                elif base.startswith("%"):
                    out[idx] = scales.get(base)
                else:
                    out[idx] = 0
            if ins.cls == "MemLoad" and ops and ops[0].startswith("%"):
                scales[ops[0]] = 0 if ins.space == "param" else None
            continue
        if not ops or not ops[0].startswith("%"):
            continue
        dst, base = ops[0], ins.base
        sc = lambda o: operand_scale(o, scales)  # noqa: E731
        if base == "mov" and len(ops) == 2:
            scales[dst] = sc(ops[1])
        elif base in ("cvt", "cvta") and len(ops) >= 2:
            scales[dst] = sc(ops[-1])
        elif base in ("add", "sub") and len(ops) == 3:
            a, b = sc(ops[1]), sc(ops[2])
            scales[dst] = None if a is None or b is None else (a + b if base == "add" else a - b)
        elif base == "mul" and len(ops) == 3:
            scales[dst] = _mul_scale(ops[1], ops[2], scales)
        elif base in ("mad", "fma") and len(ops) == 4:
            p, c = _mul_scale(ops[1], ops[2], scales), sc(ops[3])
            scales[dst] = None if p is None or c is None else p + c
        elif base == "shl" and len(ops) == 3:
            a, imm = sc(ops[1]), py_int_literal(ops[2])
            scales[dst] = None if a is None or imm is None else a * (1 << imm)
        elif base == "setp":
            pass
        else:
            srcs = [sc(o) for o in ops[1:]]
            scales[dst] = 0 if srcs and all(s == 0 for s in srcs) else None
    return out


def block_index(blocks, i):
    for b, (s, e) in enumerate(blocks):
        if s <= i < e:
            return b
    raise IndexError(i)


def aligned_fraction(k: Kernel, blocks, weights) -> float:
    """alignment.py:128-147."""
    asc = address_scales(k)
    hit = tot = 0.0
    for idx, ins in enumerate(k.ins):
        if ins.cls not in ("MemLoad", "MemStore") or ins.space != "global":
            continue
        w = weights[block_index(blocks, idx)]
        tot += w
        s = asc.get(idx)
        if s is not None and abs(s) == access_bytes(ins.opcode):
            hit += w
    return 1.0 if tot == 0.0 else hit / tot


# ------------------------------------------------------------------ a11: dynamic counts
def dynamic_counts(k: Kernel, blocks, weights):
    """features.py:62-81 -> (n_mem, mem_bytes, {FP32,INT,SFU,ALU}, n_sync)."""
    n_mem = mem_bytes = n_sync = 0.0
    unit = {u: 0.0 for u in ("FP32", "INT", "SFU", "ALU")}
    for idx, ins in enumerate(k.ins):
        w = weights[block_index(blocks, idx)]
        if ins.cls in ("MemLoad", "MemStore"):
            if ins.space in ("global", "shared", "local", "none"):
                n_mem += w
                mem_bytes += w * access_bytes(ins.opcode)
        elif ins.cls in unit:
            unit[ins.cls] += w
        elif ins.cls == "Sync":
            n_sync += w
    return n_mem, mem_bytes, unit, n_sync


def class_histogram(k: Kernel):
    h = [0] * len(CLASSES)
    for ins in k.ins:
        h[CLASSES.index(ins.cls)] += 1
    return h


def kernel_feature_row(src: str, default_trip: float = 32.0, annotations=None, wanted=None):
    """Everything K1+K1b produce for one kernel: the FFB_F_* row (first 11 columns)."""
    k = parse_kernel(src, wanted)
    blocks, _edges, loops = build_blocks(k)
    trips = loop_trips(k, blocks, loops, default_trip, annotations)
    w = block_weights(blocks, loops, trips)
    n_mem, mem_bytes, unit, n_sync = dynamic_counts(k, blocks, w)
    al = aligned_fraction(k, blocks, w)
    return [n_mem, mem_bytes, unit["FP32"], unit["INT"], unit["SFU"], unit["ALU"], n_sync, al,
            float(k.shared), float(sum(k.regs.values())), float(len(k.ins))]


# ------------------------------------------------------------------ a13-a17: models
def _pmin(a, b):
    return b if b < a else a


def _pmax(a, b):
    return b if b > a else a


def occupancy_ext(arch: dict, bx: int, by: int, bz: int = 1, regs: int = 0, regs_per_sm: int = 0,
                  shared: int = 0):
    """Occupancy of one block shape, with the two EXTENSION axes north_star (2) names and the
    reference does not define (it records registers, features.py:126, and never limits on them;
    LaunchConfig has no block_z, launch.py:11-21) - "parity unpinned", this function IS the definition:

      threads = bx*by*bz;  warps = threads // 32                      (features.py:96,110 with z)
      bps = max_warps / warps                                          (features.py:112)
      if shared > 0:  bps = min(bps, max_shared / shared)              (features.py:113-114)
      if regs_per_sm > 0 and regs > 0:                                 (extension)
          bps = min(bps, regs_per_sm / (regs * threads))      registers a resident block needs
      valid iff 32 <= threads <= max_threads, threads % 32 == 0, warps <= max_warps and, with a
      register limit, regs_per_sm / (regs * threads) >= 1.0           (explorer.py:79-88 style)

    With bz = 1 and regs_per_sm = 0 every line is the reference's.  Returns (valid, warps, bps)."""
    threads = bx * by * bz
    if threads < 32 or threads > arch["max_threads_per_block"] or threads % 32:
        return False, 0, 0.0
    warps = threads // 32
    bps = arch["max_warps_per_sm"] / warps
    valid = warps <= arch["max_warps_per_sm"]
    if shared > 0:
        bps = _pmin(bps, arch["max_shared_per_sm"] / shared)
    if regs_per_sm > 0 and regs > 0:
        lim = float(regs_per_sm) / float(regs * threads)
        bps = _pmin(bps, lim)
        valid = valid and lim >= 1.0
    return valid, warps, bps


def score_point(feat, arch: dict, cal: dict, bx: int, by: int, cap: float, shared_dyn: int,
                total_blocks: int, bz: int = 1, regs: int = 0, regs_per_sm: int = 0):
    """features.py:96-114, time_model.py:67-129, power_model.py:124-170, explorer.py:105-108.
    feat: dict with n_mem, mem_bytes, FP32, INT, SFU, ALU, n_sync, aligned, static_shared.
    bz / regs / regs_per_sm: extension axes, see occupancy_ext (defaults = the reference).
    Returns dict(t_exec, p_dyn, e_pred, cap_limited, blocks_per_sm, warps, eta)."""
    threads = bx * by * bz
    warps = threads // 32
    shared = int(feat["static_shared"]) + shared_dyn
    bps = arch["max_warps_per_sm"] / warps
    if shared > 0:
        bps = _pmin(bps, arch["max_shared_per_sm"] / shared)
    if regs_per_sm > 0 and regs > 0:
        bps = _pmin(bps, float(regs_per_sm) / float(regs * threads))
    eta = _pmin(1.0, bx / 32.0) * feat["aligned"]
    resident = _pmin(bps * warps, float(arch["max_warps_per_sm"]))
    lanes = arch["sm_count"] * resident * 32.0
    waves = _pmax(1.0, (total_blocks * warps) * 32.0 / lanes)
    mwp = _pmax(1.0, cal["l_mem_coal"] / arch["departure_delay"])
    tot = wsum = 0.0
    for u in ("FP32", "INT", "SFU"):
        wsum += feat[u] * (arch["exec_cycles"][u] / arch["issue_cycles"][u])
        tot += feat[u]
    window = wsum / tot if tot > 0 else arch["exec_cycles"]["ALU"] / arch["issue_cycles"]["ALU"]
    cwp = _pmax(1.0, (cal["l_mem_coal"] + window) / window)
    floor = cal["l_mem_coal"] / cal["l_mem_uncoal"] if cal["l_mem_uncoal"] > 0 else 0.0
    bw_eff = arch["bw_max"] * _pmax(eta, floor)
    mb = feat["mem_bytes"] * waves
    t_mem = mb / (mwp * bw_eff) if mb > 0 else 0.0
    n_comp = feat["FP32"] + feat["INT"] + feat["SFU"]
    nc = n_comp * waves
    t_comp = nc / (cwp * arch["ipc"] * arch["f_base"]) if nc > 0 else 0.0
    t_sync = feat["n_sync"] * waves * arch["t_barrier"]
    a, b, g = cal["time_weights"]
    t_exec = a * t_mem + b * t_comp + g * t_sync + cal["t_base"]

    wps = _pmin(warps * bps, float(arch["max_warps_per_sm"]))
    p_units = 0.0
    for u in UNITS:
        cnt = feat["n_mem"] if u == "Mem" else feat[u]
        ex = cal["l_mem_coal"] if u == "Mem" else arch["exec_cycles"][u]
        if ex <= 0:
            continue
        p_units += cal["beta_u"][u] * (cnt * wps / (ex / arch["issue_cycles"][u]))
    if feat["n_mem"] == 0:
        p_shape = cal["p_base_shape"]
    else:
        ci = n_comp / feat["n_mem"]
        p_shape = cal["p_base_shape"] * (1.0 + cal["kappa"] * abs(math.log(bx / by)) / (1.0 + ci))
    p_mem = cal["p_mem_base"] * (1.0 + cal["lambda"] * (1.0 - eta))
    active = min(arch["sm_count"], total_blocks)
    p_sm = cal["sm_power_delta"] if active == 0 else \
        cal["sm_power_alpha"] * float(active) ** cal["sm_power_beta"] + cal["sm_power_delta"]
    p_dyn = p_units + p_shape + p_mem + p_sm
    if t_exec < arch["tau_short"]:
        p_dyn = p_dyn * cal["transient_ratio_r"]
    f_adj = arch["f_base"] * (cap / arch["p_tdp"]) ** (1.0 / arch["dvfs_exponent_K"])
    p_dyn *= f_adj / arch["f_base"]
    limited = False
    if p_dyn + arch["p_static"] > cap:
        p_dyn = _pmax(0.0, cap - arch["p_static"])
        limited = True
    e = t_exec * (p_dyn + arch["p_static"]) + cal["e_overhead"]
    return dict(t_exec=t_exec, p_dyn=p_dyn, e_pred=e, cap_limited=limited, blocks_per_sm=bps,
                warps=warps, eta=eta)


def enumerate_configs(arch: dict, shared_dyn: int, dims, caps=None):
    """explorer.py:59-94 -> [(bx, by, cap)] in canonical order."""
    caps = sorted(set(caps)) if caps else [arch["p_tdp"]]
    out = []
    for bx in dims:
        for by in dims:
            th = bx * by
            if th < 32 or th > arch["max_threads_per_block"] or th % 32:
                continue
            bps = arch["max_warps_per_sm"] / (th // 32)
            if shared_dyn > 0:
                bps = min(bps, arch["max_shared_per_sm"] / shared_dyn)
            if bps < 1.0:
                continue
            for c in caps:
                if arch["p_cap_min"] <= c <= arch["p_tdp"]:
                    out.append((bx, by, float(c)))
    out.sort(key=lambda x: (x[0] * x[1], x[0], x[1], x[2]))
    return out


def score_grid_numpy(feat_rows: np.ndarray, res_rows: np.ndarray, arch: dict, cal: dict,
                     shapes: np.ndarray, caps: np.ndarray, regs_per_sm: int = 0, return_occ: bool = False):
    """Vectorised score_point over kernels x shapes x caps for ONE spec (numpy elementwise
    ops are the same IEEE operations as the scalar code, in the same order).
    feat_rows [K, >=9] (FFB_F_* order), res_rows [K,2], shapes [J,2] valid shapes, or [J,4]
    {bx, by, bz, regs} with the extension axes of occupancy_ext.
    Returns t, e as [K,J,C] (and blocks_per_sm [K,J] with return_occ)."""
    f = np.asarray(feat_rows, dtype=np.float64)
    K = f.shape[0]
    shapes = np.asarray(shapes)
    bx = shapes[:, 0].astype(np.int64)[None, :]
    by = shapes[:, 1].astype(np.int64)[None, :]
    bz = shapes[:, 2].astype(np.int64)[None, :] if shapes.shape[1] > 2 else np.ones_like(bx)
    regs = shapes[:, 3].astype(np.int64)[None, :] if shapes.shape[1] > 3 else np.zeros_like(bx)
    n_mem, mem_bytes = f[:, 0:1], f[:, 1:2]
    u = {"FP32": f[:, 2:3], "INT": f[:, 3:4], "SFU": f[:, 4:5], "ALU": f[:, 5:6]}
    n_sync, aligned = f[:, 6:7], f[:, 7:8]
    shared = (f[:, 8].astype(np.int64) + res_rows[:, 0])[:, None]
    total_blocks = res_rows[:, 1][:, None]
    warps = (bx * by * bz) // 32
    wf = warps.astype(np.float64)
    bps = np.broadcast_to(arch["max_warps_per_sm"] / wf, (K, wf.shape[1])).copy()
    with np.errstate(divide="ignore"):
        lim = np.where(shared > 0, arch["max_shared_per_sm"] / np.maximum(shared, 1).astype(np.float64), np.inf)
    bps = np.where(lim < bps, lim, bps)
    if regs_per_sm > 0:
        need = (regs * bx * by * bz).astype(np.float64)
        with np.errstate(divide="ignore"):
            rlim = np.where(regs > 0, float(regs_per_sm) / np.maximum(need, 1.0), np.inf)
        bps = np.where(rlim < bps, rlim, bps)
    r = bx / 32.0
    eta = np.where(r < 1.0, r, 1.0) * aligned
    mw = float(arch["max_warps_per_sm"])
    resident = bps * wf
    resident = np.where(mw < resident, mw, resident)
    lanes = arch["sm_count"] * resident * 32.0
    waves = (total_blocks * warps).astype(np.float64) * 32.0 / lanes
    waves = np.where(waves > 1.0, waves, 1.0)
    mwp = _pmax(1.0, cal["l_mem_coal"] / arch["departure_delay"])
    wsum = np.zeros((K, 1))
    tot = np.zeros((K, 1))
    for name in ("FP32", "INT", "SFU"):
        wsum = wsum + u[name] * (arch["exec_cycles"][name] / arch["issue_cycles"][name])
        tot = tot + u[name]
    with np.errstate(invalid="ignore", divide="ignore"):
        window = np.where(tot > 0, wsum / tot, arch["exec_cycles"]["ALU"] / arch["issue_cycles"]["ALU"])
    cwp = (cal["l_mem_coal"] + window) / window
    cwp = np.where(cwp > 1.0, cwp, 1.0)
    floor = cal["l_mem_coal"] / cal["l_mem_uncoal"] if cal["l_mem_uncoal"] > 0 else 0.0
    bw_eff = arch["bw_max"] * np.where(floor > eta, floor, eta)
    mb = mem_bytes * waves
    with np.errstate(invalid="ignore", divide="ignore"):
        t_mem = np.where(mb > 0, mb / (mwp * bw_eff), 0.0)
    n_comp = u["FP32"] + u["INT"] + u["SFU"]
    nc = n_comp * waves
    t_comp = np.where(nc > 0, nc / (cwp * arch["ipc"] * arch["f_base"]), 0.0)
    t_sync = n_sync * waves * arch["t_barrier"]
    a, b, g = cal["time_weights"]
    t_exec = a * t_mem + b * t_comp + g * t_sync + cal["t_base"]
    wps = wf * bps
    wps = np.where(mw < wps, mw, wps)
    p_units = np.zeros_like(wps)
    for name in UNITS:
        cnt = n_mem if name == "Mem" else u[name]
        ex = cal["l_mem_coal"] if name == "Mem" else arch["exec_cycles"][name]
        if ex <= 0:
            continue
        p_units = p_units + cal["beta_u"][name] * (cnt * wps / (ex / arch["issue_cycles"][name]))
    logs = np.array([abs(math.log(int(x) / int(y))) for x, y in shapes[:, :2]], dtype=np.float64)[None, :]
    with np.errstate(invalid="ignore", divide="ignore"):
        ci = n_comp / n_mem
        p_shape = np.where(n_mem == 0, cal["p_base_shape"],
                           cal["p_base_shape"] * (1.0 + cal["kappa"] * logs / (1.0 + ci)))
    p_mem = cal["p_mem_base"] * (1.0 + cal["lambda"] * (1.0 - eta))
    active = np.minimum(arch["sm_count"], total_blocks)
    p_sm = np.array([cal["sm_power_delta"] if int(x) == 0 else
                     cal["sm_power_alpha"] * float(int(x)) ** cal["sm_power_beta"] + cal["sm_power_delta"]
                     for x in active[:, 0]], dtype=np.float64)[:, None]
    p_pre = p_units + p_shape + p_mem + p_sm
    p_pre = np.where(t_exec < arch["tau_short"], p_pre * cal["transient_ratio_r"], p_pre)
    scale = np.array([(arch["f_base"] * (float(c) / arch["p_tdp"]) ** (1.0 / arch["dvfs_exponent_K"])) / arch["f_base"]
                      for c in caps], dtype=np.float64)[None, None, :]
    capv = np.asarray(caps, dtype=np.float64)[None, None, :]
    p_dyn = p_pre[:, :, None] * scale
    over = p_dyn + arch["p_static"] > capv
    room = capv - arch["p_static"]
    p_dyn = np.where(over, np.where(room > 0.0, room, 0.0), p_dyn)
    t3 = np.broadcast_to(t_exec[:, :, None], p_dyn.shape)
    e = t3 * (p_dyn + arch["p_static"]) + cal["e_overhead"]
    if return_occ:
        return np.ascontiguousarray(t3), e, np.ascontiguousarray(bps)
    return np.ascontiguousarray(t3), e


# ------------------------------------------------------------------ a19/a20: Pareto
def pareto_indices(e, t, tie=None, rho: float = 0.0):
    """explorer.py:122-140 with the floor of :209-211.  Returns (indices in (e,t,tie) order, t_peak).
    Sort-and-sweep: best_t only ever takes values from STRICTLY lower energies."""
    e = np.asarray(e, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    n = e.size
    if n == 0:
        return [], math.inf
    tie = np.arange(n) if tie is None else np.asarray(tie)
    t_peak = float(t.min())
    ok = t <= (t_peak / rho) if rho > 0 else np.ones(n, dtype=bool)
    idx = np.nonzero(ok & np.isfinite(e) & np.isfinite(t))[0]
    order = idx[np.lexsort((tie[idx], t[idx], e[idx]))]
    kept, best, i = [], math.inf, 0
    while i < order.size:
        j = i
        while j < order.size and e[order[j]] == e[order[i]]:
            j += 1
        grp = order[i:j]
        kept.extend(int(p) for p in grp if t[p] <= best)
        best = min(best, float(t[grp].min()))
        i = j
    return kept, t_peak


def pareto_indices3(e, t, occ, tie=None, rho: float = 0.0):
    """Three-objective EXTENSION (no reference semantics; parity unpinned - this function is the
    definition the kernel is tested against): after the floor of explorer.py:209-211, candidate i is
    dropped iff some j has e_j < e_i, t_j < t_i and occ_j >= occ_i.  With a constant occ this is
    explorer.py:122-140.  O(n^2); order (e, t, tie) as pareto_indices."""
    e = np.asarray(e, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    occ = np.asarray(occ, dtype=np.float64)
    n = e.size
    if n == 0:
        return [], math.inf
    tie = np.arange(n) if tie is None else np.asarray(tie)
    t_peak = float(t.min())
    ok = t <= (t_peak / rho) if rho > 0 else np.ones(n, dtype=bool)
    idx = np.nonzero(ok & np.isfinite(e) & np.isfinite(t))[0]
    keep = [int(i) for i in idx if not np.any((e[idx] < e[i]) & (t[idx] < t[i]) & (occ[idx] >= occ[i]))]
    keep = np.asarray(keep, dtype=np.int64)
    order = keep[np.lexsort((tie[keep], t[keep], e[keep]))] if keep.size else keep
    return [int(i) for i in order], t_peak


def pareto_bruteforce(e, t):
    """explorer.py:143-158: O(n^2) ground truth (membership only, as a set)."""
    e = np.asarray(e, dtype=np.float64)
    t = np.asarray(t, dtype=np.float64)
    return {i for i in range(e.size) if not np.any((e < e[i]) & (t < t[i]))}


def arch_dict(a) -> dict:
    """Accepts any object with the ArchitectureSpec field names."""
    return dict(sm_count=a.sm_count, max_warps_per_sm=a.max_warps_per_sm, max_shared_per_sm=a.max_shared_per_sm,
                max_threads_per_block=a.max_threads_per_block, bw_max=a.bw_max, ipc=a.ipc, f_base=a.f_base,
                p_tdp=a.p_tdp, p_static=a.p_static, p_cap_min=a.p_cap_min, dvfs_exponent_K=a.dvfs_exponent_k,
                tau_short=a.tau_short, departure_delay=a.departure_delay, t_barrier=a.t_barrier,
                exec_cycles=dict(a.exec_cycles), issue_cycles=dict(a.issue_cycles))


def cal_dict(p) -> dict:
    return dict(beta_u=dict(p.beta_u), l_mem_coal=p.l_mem_coal, l_mem_uncoal=p.l_mem_uncoal,
                sm_power_alpha=p.sm_power_alpha, sm_power_beta=p.sm_power_beta,
                sm_power_delta=p.sm_power_delta, transient_ratio_r=p.transient_ratio_r, kappa=p.kappa,
                p_base_shape=p.p_base_shape, p_mem_base=p.p_mem_base, time_weights=tuple(p.time_weights),
                t_base=p.t_base, e_overhead=p.e_overhead, **{"lambda": p.lambda_})
