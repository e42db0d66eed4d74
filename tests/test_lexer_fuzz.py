"""Differential fuzz of the two lexer kernels: seeded random edits of generated kernels (comments with
structural characters, blank and brace lines, labels, vector operands, spacing, joined statements, CRLF,
header variations, long lines); whichever kernel finishes a segment, statuses, histograms, segment infos,
instruction and label records must be byte-identical to the exact walk alone."""
from __future__ import annotations

import numpy as np
import pytest

from paper_2601_13345_b200 import corpus, synth

JUNK = ["{", "}", "{ }", ":", ";", ".entry ghost()", "L9:", "a; b;", "[%rd1+4]", "@%p1 bra L0;", "/", "*/", "%tid.x", "\t", " "]


def _mutate(rng: np.random.Generator, src: str) -> str:
    lines = src.split("\n")
    body0 = next((i for i, l in enumerate(lines) if l.strip() == "{" or l.rstrip().endswith(" {")), 5) + 1
    n_edits = int(rng.integers(1, 9))
    for _ in range(n_edits):
        kind = int(rng.integers(0, 16))
        at = int(rng.integers(body0, max(body0 + 1, len(lines) - 2)))
        junk = " ".join(rng.choice(JUNK, size=int(rng.integers(1, 4))))
        if kind == 0:
            lines[at] += " \t// " + junk
        elif kind == 1:
            lines.insert(at, "\t// " + junk)
        elif kind == 2:
            lines.insert(at, rng.choice(["", " ", "\t\t", " \t "]))
        elif kind == 3:                                   # balanced nested scope around one line
            lines.insert(at, "\t{" + rng.choice(["", " // callseq"]))
            lines.insert(min(at + 2, len(lines) - 2), "\t}")
        elif kind == 4:
            lines.insert(at, rng.choice(["LX%d:" % at, "  $L__x%d:  " % at, "LX%d: // c" % at, "LX%d :" % at, "LX%d: ret;" % at]))
        elif kind == 5:
            lines.insert(at, "\tld.global.v4.f32 \t{%f1, %f2,%f3 , %f4}, [%rd6+" + str(at) + "];")
        elif kind == 6:
            lines[at] = lines[at].replace(", ", rng.choice([",", " , ", ",\t"])).replace(";", rng.choice([" ;", ";  ", "\t;"]))
        elif kind == 7:                                   # two statements on one line / statement split over two
            if rng.random() < 0.5:
                lines[at] = lines[at] + " " + lines[at].strip()
            else:
                lines[at] = lines[at].replace(", ", ",\n\t\t", 1)
        elif kind == 8:
            lines.insert(at, rng.choice(["\t@%p1 bra \tLZ;", "\t@!%p2 bra.uni LZ;", "\t@%p1 add.s32 %r1, %r1, 1;", "\t@ %p1 ret;"]))
            lines.insert(body0, "LZ:")
        elif kind == 9:
            lines.insert(at, "\tmad.lo.s32 \t%r1, " + ", ".join("%r" + str(int(x)) for x in rng.integers(1, 60, size=int(rng.integers(2, 30)))) + ";")
        elif kind == 10:
            lines.insert(at, rng.choice([".loc 1 2 3", "\t.pragma \"nounroll\";", "\t.reg .b32 %extra<" + str(at) + ">;", "\t.shared .align 8 .b8 buf" + str(at) + "[64];",
                                         "\t.reg .b32 %a<2>; .reg .b32 %b<3>;", "\t.local .align 4 .b8 loc[16];"]))
        elif kind == 11:
            lines.insert(at, "\tmov.u32 %r1, " + rng.choice(["0x1F", "017", "1_000", "-0", "+5", "4294967296", "0f3F800000", "WARP_SZ", "%laneid", "%ctaid.z"]) + ";")
        elif kind == 12:                                  # header variations
            h = next(i for i, l in enumerate(lines) if ".entry" in l)
            lines[h] = rng.choice(["// .entry fake() {\n", "", "/* c */ ", "// {\n"]) + lines[h]
            if rng.random() < 0.3:
                b = next((i for i, l in enumerate(lines) if l.strip() == "{"), None)
                if b is not None and b > 0:
                    lines[b - 1] += rng.choice([" // x {", " {", " // y"])
                    if lines[b - 1].endswith(" {"):
                        del lines[b]
        elif kind == 13:
            lines.insert(at, "\t/* " + junk.replace("*/", "") + " */" + rng.choice(["", " ret;"]))
        elif kind == 14:
            lines.insert(at, "\tst.global.v2.f32 \t[%rd7], {%f1, %f2}; // {" )
        else:
            lines.insert(at, rng.choice(["\t;", ";;", "\tret", "\tbar.sync \t0 ;  // sync: all", "\ttex.2d.v4.f32.f32 {%f1,%f2,%f3,%f4}, [t, {%f5,%f6}];"]))
    out = "\n".join(lines)
    if rng.random() < 0.05:
        out = out.replace("\n", "\r\n")
    return out


@pytest.mark.parametrize("seed", [1, 2, 3, 4])
def test_fast_path_and_exact_walk_agree_on_mutated_kernels(backend, seed):
    rng = np.random.default_rng(1000 + seed)
    n = 24 if backend == "emul" else 400
    text, offs = synth.ptx_corpus(seed=40 + seed, n_kernels=n, lo=15, hi=160 if backend == "emul" else 1500)
    srcs = [_mutate(rng, text[offs[i]:offs[i + 1]].decode("ascii")) for i in range(n)]
    blobs = [s.encode("ascii") for s in srcs]
    corp = corpus.upload_corpus(b"".join(blobs), np.cumsum([0] + [len(b) for b in blobs]))
    fast = corpus.lex_records(corp)
    corpus.EXACT_ONLY_DEFAULT = True
    try:
        exact = corpus.lex_records(corp)
    finally:
        corpus.EXACT_ONLY_DEFAULT = False
    fast_hist = corpus.lex_histogram(corp)                         # histogram mode: its own opcode shortcut
    taken = fast.path_counts.cpu().tolist()
    assert taken[0] + taken[1] == n and taken[0] > 0            # some of these stay regular
    fi, ei = fast.info_np(), exact.info_np()
    assert np.array_equal(fi["status"], ei["status"])
    ok = fi["status"] == 0
    assert ok.any()
    assert np.array_equal(fast.info.cpu().numpy()[ok], exact.info.cpu().numpy()[ok])
    assert np.array_equal(fast.hist.cpu().numpy()[ok], exact.hist.cpu().numpy()[ok])
    assert np.array_equal(fast_hist.hist.cpu().numpy()[ok], exact.hist.cpu().numpy()[ok])
    assert np.array_equal(fast_hist.info.cpu().numpy()[ok], exact.info.cpu().numpy()[ok])
    assert np.array_equal(fast.ins_base.cpu().numpy(), exact.ins_base.cpu().numpy())
    fins, eins = fast.ins.cpu().numpy(), exact.ins.cpu().numpy()
    flab, elab = fast.labels.cpu().numpy(), exact.labels.cpu().numpy()
    ib, lb = fast.ins_base.cpu().numpy(), fast.lab_base.cpu().numpy()
    for k in np.nonzero(ok)[0]:
        a, b = int(ib[k]), int(ib[k]) + int(fi["n_instr"][k])
        assert np.array_equal(fins[a:b], eins[a:b]), (seed, int(k), srcs[k][:200])
        a, b = int(lb[k]), int(lb[k]) + int(fi["n_labels"][k])
        assert np.array_equal(flab[a:b], elab[a:b]), (seed, int(k))
    # and the oracle agrees with both (statuses, histograms, declarations, feature rows)
    from test_corpus_parity import _check
    _check(srcs[: 12 if backend == "emul" else 60])
