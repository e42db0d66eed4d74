"""K1 (lexer / classifier / histogram) and K1b (CFG, trips, alignment, dynamic counts)
against the oracle: bit-exact histograms, declarations, statuses and feature rows."""
from __future__ import annotations

import numpy as np
import pytest

import flipflop_oracle as orc
from edge_cases import EDGE_CASES
from paper_2601_13345_b200 import corpus, native, synth

STATUS_OF = {"MalformedPtx": 1, "NoKernelFound": 2}


def _corpus(texts):
    blobs = [t.encode("ascii") for t in texts]
    offs = np.cumsum([0] + [len(b) for b in blobs])
    return corpus.upload_corpus(b"".join(blobs), offs)


def _check(texts, default_trip=32.0):
    corp = _corpus(texts)
    lex, fl = corpus.analyze_corpus(corp, default_trip=default_trip)
    info, hist = lex.info_np(), lex.hist.cpu().numpy()
    feat, status = fl.feat.cpu().numpy(), fl.status.cpu().numpy()
    for k, src in enumerate(texts):
        try:
            kern = orc.parse_kernel(src)
            want_row = np.asarray(orc.kernel_feature_row(src, default_trip=default_trip), dtype=np.float64)
            want_status = 0
        except orc.OracleError as ex:
            want_status = STATUS_OF[ex.kind]
        assert int(status[k]) == want_status, (k, src[:60])
        if want_status:
            continue
        assert hist[k].tolist() == orc.class_histogram(kern)
        assert int(info[k]["n_instr"]) == len(kern.ins)
        assert int(info[k]["static_shared"]) == kern.shared
        assert int(info[k]["regs_declared"]) == sum(kern.regs.values())
        name = src.encode()[int(info[k]["name_off"]): int(info[k]["name_off"]) + int(info[k]["name_len"])].decode()
        assert name == kern.name
        assert feat[k, :11].tobytes() == want_row.tobytes(), (k, feat[k, :11].tolist(), want_row.tolist())


def test_edge_cases(backend):
    _check(list(EDGE_CASES.values()))


@pytest.mark.parametrize("seed,default_trip", [(4, 32.0), (9, 7.5), (11, 7.3)])     # 7.3: inexact sums -> in-order pass
def test_synthetic_corpus(backend, seed, default_trip):
    n = 16 if backend == "emul" else 600
    text, offs = synth.ptx_corpus(seed=seed, n_kernels=n, lo=20, hi=700 if backend == "emul" else 5000)
    _check([text[offs[i]:offs[i + 1]].decode("ascii") for i in range(n)], default_trip)


def test_irregular_share_of_the_bench_corpus(backend):
    """bench.py's corpus gives a share of its kernels one construct outside the fast path's grammar (synth._IRREGULAR):
    those segments are finished by the exact walk, every row still equals the oracle's, and the pieces of a corpus
    generated in parallel carry unique kernel names."""
    text, offs = synth.ptx_corpus(seed=31, n_kernels=8, lo=20, hi=300, irregular=1.0, first=600)
    srcs = [text[offs[i]:offs[i + 1]].decode("ascii") for i in range(8)]
    assert any("/* spilled" in s for s in srcs) and any("$L__note:" in s for s in srcs) and "synk_031_000607" in srcs[7]
    _check(srcs)
    lex = corpus.lex_histogram(_corpus(srcs))
    assert lex.path_counts.cpu().tolist()[:2] == [0, 8]
    plain, _ = synth.ptx_corpus(seed=31, n_kernels=8, lo=20, hi=300)
    assert plain != text and len(plain) < len(text)


def test_tile_boundaries(backend):
    """Kernels longer than one 4 KB tile, long preambles, statements split over tile edges."""
    rng = np.random.default_rng(5)
    texts = []
    for pad in (0, 1, 15, 16, 17, 2047, 3000, 4000, 4050, 4070):
        body = "\n".join(f"\tadd.s32 \t%r{i % 7}, %r{(i + 1) % 7}, {i};  // note {i}" for i in range(int(rng.integers(150, 400))))
        multi = "\tcall.uni (retval0),\n\tfoo,\n\t(\n\tparam0,\n\tparam1\n\t);\n"
        texts.append("//" + "x" * pad + "\n.visible .entry t" + str(pad) + "(\n.param .u64 p0)\n{\n" + body + "\n" + multi * 3
                     + "L:\n\t@%p1 bra L;\n\tret;\n}\n")
    _check(texts)


def test_named_kernel_selection(backend):
    src = ".entry a()\n{\n ret;\n}\n.entry b()\n{\n add.s32 %r1, %r1, 1;\n exit;\n}\n"
    corp = _corpus([src])
    res = corpus.lex_histogram(corp, kernel_name="b")
    assert int(res.info_np()[0]["status"]) == 0 and res.hist.cpu().numpy()[0].tolist() == orc.class_histogram(orc.parse_kernel(src, "b"))
    res = corpus.lex_histogram(corp, kernel_name="zzz")
    assert int(res.info_np()[0]["status"]) == 2


def test_line_longer_than_tile_is_reported(backend):
    src = ".entry a()\n{\n add.s32 %r1, %r1, " + "1" * 6000 + ";\n ret;\n}\n"
    res = corpus.lex_histogram(_corpus([src]))
    assert int(res.info_np()[0]["status"]) == 11       # FFB_E_CAPACITY, never a silent wrong answer


def test_single_pass_records_equal_two_pass(backend):
    """Single-pass record mode (capacity slots) gives the same histograms and feature rows as the
    counting + record passes, and reports segments that outgrow their slots."""
    n = 10 if backend == "emul" else 400
    text, offs = synth.ptx_corpus(seed=13, n_kernels=n, lo=20, hi=500 if backend == "emul" else 3000)
    dense = ".entry d()\n{\n" + "ret;\n" * 300 + "}\n"          # 5-byte statements: needs more slots than len/12
    blob = text + dense.encode()
    offs = np.concatenate([offs, [len(blob)]])
    corp = corpus.upload_corpus(blob, offs)
    lex2, fl2 = corpus.analyze_corpus(corp)
    lex1 = corpus.lex_records_single_pass(corp)
    fl1 = corpus.kernel_features(corp, lex1)
    st1, st2 = fl1.status.cpu().numpy(), fl2.status.cpu().numpy()
    assert (st2 == 0).all() and (st1[:-1] == 0).all() and st1[-1] == 11
    assert np.array_equal(lex1.hist.cpu().numpy(), lex2.hist.cpu().numpy())
    assert fl1.feat.cpu().numpy()[:-1, :11].tobytes() == fl2.feat.cpu().numpy()[:-1, :11].tobytes()


def test_multi_kernel_module_ingestion(backend):
    """split_modules: every .entry of every module becomes a segment whose feature row equals the
    oracle's parse of the whole module with that kernel named (reference: ptx.py:168-184)."""
    text, offs = synth.ptx_corpus(seed=17, n_kernels=7, lo=20, hi=120, comments=True)
    segs = [text[offs[i]:offs[i + 1]].decode() for i in range(7)]
    mod_a = ".version 8.0\n.func helper()\n{\n ret;\n}\n" + "".join(segs[:3]) + "// trailing\n"
    mod_b = "".join(segs[3:]) + ".global .u32 tail;\n"
    mod_c = "// a module without kernels\n.func f() { ret; }\n"
    blob = (mod_a + mod_b + mod_c).encode()
    module_off = np.cumsum([0, len(mod_a), len(mod_b), len(mod_c)])
    corp = corpus.split_modules(blob, module_off)
    mask = corp.kernel_mask
    assert int(mask.sum()) == 7
    lex, fl = corpus.analyze_corpus(corp)
    info, feat, status = lex.info_np(), fl.feat.cpu().numpy(), fl.status.cpu().numpy()
    names, k = [], 0
    seg_off = corp.host_off
    for s_i in range(corp.n_segs):
        if not mask[s_i]:
            continue
        module_src = mod_a if k < 3 else mod_b
        piece = blob[seg_off[s_i]:seg_off[s_i + 1]]
        name = piece[int(info[s_i]["name_off"]): int(info[s_i]["name_off"]) + int(info[s_i]["name_len"])].decode()
        want = np.asarray(orc.kernel_feature_row(module_src, wanted=name), dtype=np.float64)
        assert status[s_i] == 0 and feat[s_i, :11].tobytes() == want.tobytes(), name
        names.append(name)
        k += 1
    assert len(set(names)) == 7


def _lex_both(corp):
    fast = corpus.lex_records(corp)
    fast_hist = corpus.lex_histogram(corp)
    corpus.EXACT_ONLY_DEFAULT = True
    try:
        exact = corpus.lex_records(corp)
        exact_hist = corpus.lex_histogram(corp)
    finally:
        corpus.EXACT_ONLY_DEFAULT = False
    # histogram mode has its own opcode shortcut in the fast path: same histograms and infos as every other way
    assert np.array_equal(fast_hist.hist.cpu().numpy(), exact_hist.hist.cpu().numpy())
    assert np.array_equal(fast_hist.info.cpu().numpy(), exact_hist.info.cpu().numpy())
    ok = exact.info_np()["status"] == 0
    assert np.array_equal(fast_hist.hist.cpu().numpy()[ok], exact.hist.cpu().numpy()[ok])
    return fast, exact


def test_fast_path_equals_exact_walk(backend):
    """The byte-parallel fast path and the exact statement walk write identical histograms,
    segment infos, instruction / label records; compiler-shaped text stays on the fast path."""
    n = 12 if backend == "emul" else 300
    text, offs = synth.ptx_corpus(seed=21, n_kernels=n, lo=20, hi=600 if backend == "emul" else 5000)
    fast, exact = _lex_both(corpus.upload_corpus(text, offs))
    assert fast.path_counts.cpu().tolist()[:2] == [n, 0] and exact.path_counts.cpu().tolist()[:2] == [0, n]
    n_ins = int(fast.info_np()["n_instr"].sum())
    assert fast.path_counts.cpu().tolist()[2] < 0.1 * n_ins       # the bit-window parser takes nearly every statement
    for f in ("hist", "info", "ins", "labels", "meta"):
        assert np.array_equal(getattr(fast, f).cpu().numpy(), getattr(exact, f).cpu().numpy()), f
    # irregular inputs: whichever kernel finishes a segment, the bytes are the same
    fast, exact = _lex_both(_corpus(list(EDGE_CASES.values())))
    taken = fast.path_counts.cpu().tolist()[:2]
    assert taken[0] > 0 and taken[1] > 0 and sum(taken) == len(EDGE_CASES)
    for f in ("hist", "info", "ins", "labels", "meta"):
        assert np.array_equal(getattr(fast, f).cpu().numpy(), getattr(exact, f).cpu().numpy()), f


def test_crlf_text_stays_on_the_fast_path(backend):
    """CR is a blank for Python's strip() / split() / \\s, so CRLF files (and stray CRs between operands)
    are regular text: same records as the exact walk, same rows as the oracle, no hand-over."""
    text, offs = synth.ptx_corpus(seed=41, n_kernels=5, lo=30, hi=250)
    srcs = [text[offs[i]:offs[i + 1]].decode("ascii").replace("\n", "\r\n") for i in range(5)]
    srcs[2] = srcs[2].replace(", ", ",\r ", 7).replace(";\r\n", " \r;\r\n", 5)
    fast, exact = _lex_both(_corpus(srcs))
    assert fast.path_counts.cpu().tolist()[:2] == [5, 0]
    for f in ("hist", "info", "ins", "labels", "meta"):
        assert np.array_equal(getattr(fast, f).cpu().numpy(), getattr(exact, f).cpu().numpy()), f
    _check(srcs)
    # CR-only line ends: ONE physical line for the reference (the leading // comment swallows the kernel;
    # without it the statements share a line)
    small = ".visible .entry k()\n{\n\t.reg .b32 %r<4>;\n\tmov.u32 %r1, %tid.x;\n\tadd.s32 %r2, %r1, 1;\n\tret;\n}\n"
    _check([("// c\n" + small).replace("\n", "\r"), small.replace("\n", "\r"), small.replace("\n", "\r\n")])


@pytest.mark.parametrize("mutation", ["crlf", "block_comment", "two_statements", "label_and_statement", "multi_line",
                                      "non_ascii", "comment_in_header", "brace_same_line", "trailing_blanks"])
def test_fast_path_declines_irregular_text(backend, mutation):
    """One irregular construct inside otherwise regular text: results still equal the oracle."""
    text, offs = synth.ptx_corpus(seed=23, n_kernels=3, lo=30, hi=200)
    srcs = [text[offs[i]:offs[i + 1]].decode("ascii") for i in range(3)]
    s = srcs[1]
    at = s.index("\tcvt.u64.u32")
    if mutation == "crlf":
        s = s.replace("\n", "\r\n")
    elif mutation == "block_comment":
        s = s[:at] + "\t/* add.s32 %r1, %r1, 1;\n ret; */ mov.u32 %r9, 1;\n" + s[at:]
    elif mutation == "two_statements":
        s = s[:at] + "\tmov.u32 %r9, 1; add.s32 %r9, %r9, 1;\n" + s[at:]
    elif mutation == "label_and_statement":
        s = s[:at] + "LX: mov.u32 %r9, 1;\n" + s[at:]
    elif mutation == "multi_line":
        s = s[:at] + "\tadd.s32 %r9,\n\t\t%r9,\n 1;\n" + s[at:]
    elif mutation == "non_ascii":
        s = s[:at] + "\t// caf\u00e9\n" + s[at:]
    elif mutation == "comment_in_header":
        s = s.replace(".visible .entry", "// .entry ghost()\n.visible .entry // name follows\n", 1)
    elif mutation == "brace_same_line":
        s = s.replace(")\n{\n", ") { .reg .b32 %extra<3>;\n", 1)
    elif mutation == "trailing_blanks":
        s = "\n".join(line + " \t " for line in s.split("\n"))
    srcs[1] = s
    if mutation == "non_ascii":
        blobs = [x.encode("utf-8") for x in srcs]
        corp = corpus.upload_corpus(b"".join(blobs), np.cumsum([0] + [len(b) for b in blobs]))
        res = corpus.lex_histogram(corp)
        st = res.info_np()["status"]
        assert int(st[0]) == 0 and int(st[2]) == 0          # the neighbours are untouched
        return
    _check(srcs)


OPERAND_ZOO = [
    "mov.u32 %r1, %tid.x;", "mov.u32 %r1, %tid.y;", "mov.u32 %r2, %laneid;", "mov.u32 %r2, %warpid;", "mov.u32 %r3, %gridid;",
    "mov.u32 %r3, WARP_SZ;", "mov.u32 %r4, %ctaid.x;", "mov.u32 %r4, %nctaid.z;", "mov.u32 %r4, %ntid.y;", "mov.u32 %r4, %ntid.w;",
    "mov.u32 %r4, %x%gridid;", "mov.u32 %r4, %tid.;", "mov.u32 %r4, %tid.xx;", "mov.u32 %r5, %clock;", "mov.u64 %rd1, %rd2;",
    "add.s32 %r1, %r2, 0x10;", "add.s32 %r1, %r2, 010;", "add.s32 %r1, %r2, 00;", "add.s32 %r1, %r2, 0;", "add.s32 %r1, %r2, -5;",
    "add.s32 %r1, %r2, +7;", "add.s32 %r1, %r2, 1_000;", "add.s32 %r1, %r2, 0b101;", "add.s32 %r1, %r2, 0o17;", "add.s32 %r1, %r2, 0X1f;",
    "add.s32 %r1, %r2, 1__0;", "add.s32 %r1, %r2, _1;", "add.s32 %r1, %r2, 1_;", "add.s32 %r1, %r2, -;", "add.s32 %r1, %r2, +-1;",
    "mul.f32 %f1, %f2, 0f3F800000;", "mul.f64 %fd1, %fd2, 0d3FF0000000000000;", "add.s64 %rd1, %rd2, 1234567890123456;",
    "add.s64 %rd1, %rd2, 12345678901234567;", "add.s64 %rd1, %rd2, 1152921504606846976;", "add.s64 %rd1, %rd2, -1152921504606846975;",
    "add.s64 %rd1, %rd2, 99999999;", "add.s64 %rd1, %rd2, 123456789;", "add.s32 %r1, %r2, 12a;", "add.s32 %r1, %r2, 0x;",
    "ld.global.f32 %f1, [%rd1+8];", "ld.global.f32 %f1, [%rd1];", "ld.global.f32 %f1, [ %rd1 + 8 ];", "ld.global.f32 %f1, [sym];",
    "ld.global.f32 %f1, [sym+4];", "ld.global.f32 %f1, [%rd1+-8];", "ld.global.f32 %f1, [%rd1+x];", "ld.global.f32 %f1, %rd1;",
    "ld.global.f32 %f1, [%rd1+];", "ld.global.f32 %f1, [+4];", "ld.global.f32 %f1, [%rd1+4+5];", "ld.global.f32 %f1, [%rd12345+123456];",
    "ld.global.f32 %f1, [%rd123456+123456];", "ld.global.f32 %f1, [%r+-];", "ld.global.f32 %f1, [a];", "ld.global.f32 %f1, [];",
    "ld.global.f32 %f1, [%rd1+-123456789];", "ld.global.f32 %f1, [%rd1+12_3];", "ld.global.f32 %f1, [%rd1+0x10];", "ld.global.f32 %f1, [%rd1)];",
    "ld.global.f32 %f1, [%rd1(], [%rd2];", "st.global.f32 [%rd1+4], [%rd2+8];", "ld.global.f32 %f1, [%a.b+4];", "ld.global.f32 %f1, [%rd1 +4];",
    "ld.global.v4.f32 {%f1, %f2, %f3, %f4}, [%rd1+16];", "st.global.v2.f32 [%rd1], {%f1, %f2};", "st.shared.u32 [%r1+4], %r2;",
    "tex.2d.v4.f32.f32 {%f1, %f2, %f3, %f4}, [tex0, {%f5, %f6}];", "call.uni (retval0), foo, (param0, param1);",
    "mad.lo.s32 %r1, %r2, %r3, %r4;", "fma.rn.f32 %f1, %f2, %f3, %f4;", "lop3.b32 %r1, %r2, %r3, %r4, 150;",
    "shfl.sync.bfly.b32 %r1|%p1, %r2, 16, 31, -1;", "op.x %r1, %r2, %r3, %r4, %r5, %r6, %r7;", "op.y %r1, 1, 2, 3, 4, 5, 6, 7, %r9;",
    "add.s32 %r1 , %r2 ,  3 ;", "add.s32 %r1,%r2,3;", "add.s32 %r1,, %r2;", "add.s32 %r1, %r2,;", "ret;", "bar.sync 0;", "bar.sync \t0, 64;",
    "@%p1 bra L0;", "@!%p1 bra L0;", "@%p1 add.s32 %r1, %r1, 1;", "@ %p1 bra L0;", "@%p$x.y bra L0;", "@!p bra L0;", "bra.uni L0;",
    "setp.lt.s32 %p1, %r1, 10;", "setp.ge.u32 %p1, %r1, %r2;", "sqrt.approx.f32 %f1, %f2;", "sqrt.rn.f32 %f1, %f2;", "a.b.c.d.e.f.g.h.i.j.k.l %r1;",
    "verylongopcodetoken.anotherverylongtoken.s32 %r1, %r2;", "add..s32 %r1, %r2, 1;", "add.s32. %r1, %r2, 1;", ".s32 %r1;",
    "mov.u32 %r1, a_symbol_longer_than_sixteen_bytes;", "mov.u32 %r1, exactly16bytes_ab;", "mov.u32 %r1, %r_sixteen_bytes_;",
    "mov.u32 %r1, %seventeen_bytes__;", "mov.b64 %rd1, {%r1, %r2};", "mov.b64 {%r1, %r2}, %rd1;",
    "add.s32 %r1, %r2, 3 " + "\t" * 40 + ";", "add.s32 %r1, " + " " * 45 + "%r2, 3;", "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 \t{%f1, %f2}, {%r1}, {%r2}, {%f3, %f4};",
]


def test_operand_zoo_fast_equals_exact(backend):
    """Every operand / predicate / opcode shape the record builder distinguishes, one statement per
    line so the fast path takes the segment: records equal the exact walk's bit for bit, and the
    feature rows equal the oracle's."""
    segs = []
    for rep in range(3):            # shift the alignment of every statement against the 4-byte loads
        body = "\n".join((" " * ((i + rep) % 5)) + "\t" + st for i, st in enumerate(OPERAND_ZOO))
        segs.append(".visible .entry zoo%d()\n{\n\t.reg .b32 %%r<9>;\nL0:\n%s\n\tret;\n}\n" % (rep, body))
    fast, exact = _lex_both(_corpus(segs))
    assert fast.path_counts.cpu().tolist()[:2] == [3, 0]
    assert int((fast.info_np()["status"] != 0).sum()) == 0
    for f in ("hist", "info", "ins", "labels", "meta"):
        assert np.array_equal(getattr(fast, f).cpu().numpy(), getattr(exact, f).cpu().numpy()), f
    for k, src in enumerate(segs):
        kern = orc.parse_kernel(src)
        assert fast.hist.cpu().numpy()[k].tolist() == orc.class_histogram(kern)
        assert int(fast.info_np()[k]["n_instr"]) == len(kern.ins)


def test_scale_map_spills_beyond_shared_memory(backend):
    """More distinct registers than the on-chip register -> scale map holds (384): late names live in
    the HBM table; aligned_fraction still equals the oracle's."""
    lines = [".visible .entry spill(.param .u64 p0)", "{", "\t.reg .b32 %r<1300>;", "\t.reg .b64 %rd<1300>;", "\t.reg .f32 %f<8>;",
             "\tld.param.u64 %rd0, [p0];", "\tcvta.to.global.u64 %rd1, %rd0;", "\tmov.u32 %r0, %tid.x;"]
    for i in range(1, 1200):
        lines.append(f"\tadd.s32 %r{i}, %r{i - 1}, {i % 3};")               # scale 1 carried through 1200 names
        if i % 100 == 0:
            lines.append(f"\tmul.wide.s32 %rd{i}, %r{i}, 4;")
            lines.append(f"\tadd.s64 %rd{i + 1}, %rd1, %rd{i};")
            lines.append(f"\tld.global.f32 %f1, [%rd{i + 1}];")               # aligned: scale 4, 4 bytes
            lines.append(f"\tmul.wide.s32 %rd{i + 2}, %r{i // 2}, 8;")         # an early name looked up late
            lines.append(f"\tadd.s64 %rd{i + 3}, %rd1, %rd{i + 2};")
            lines.append(f"\tld.global.f32 %f2, [%rd{i + 3}];")               # not aligned: scale 8
    lines += ["\tst.global.f32 [%rd1], %f1;", "\tret;", "}", ""]
    _check(["\n".join(lines)])


def test_parallel_textual_pass_equals_sequential(backend):
    """K1b's 32-statements-per-round dataflow pass and the one-lane in-order pass give the same
    feature rows and statuses, bit for bit (regular corpus, edge cases, operand zoo)."""
    n = 10 if backend == "emul" else 300
    text, offs = synth.ptx_corpus(seed=29, n_kernels=n, lo=20, hi=500 if backend == "emul" else 5000)
    zoo = ".visible .entry zoo()\n{\nL0:\n" + "\n".join("\t" + st for st in OPERAND_ZOO) + "\n\tret;\n}\n"
    for corp in (corpus.upload_corpus(text, offs), _corpus(list(EDGE_CASES.values()) + [zoo])):
        lex = corpus.lex_records(corp)
        par = corpus.kernel_features(corp, lex)
        corpus.FLOW_FLAGS_DEFAULT = corpus.FLOW_SEQUENTIAL_PASS
        try:
            seq = corpus.kernel_features(corp, lex)
        finally:
            corpus.FLOW_FLAGS_DEFAULT = 0
        assert np.array_equal(par.status.cpu().numpy(), seq.status.cpu().numpy())
        ok = par.status.cpu().numpy() == 0
        assert par.feat.cpu().numpy()[ok, :11].tobytes() == seq.feat.cpu().numpy()[ok, :11].tobytes()
        # the default form is two launches (CFG / trips / weights, then the dataflow pass); one launch gives the same rows
        corpus.FLOW_FLAGS_DEFAULT = corpus.FLOW_ONE_KERNEL
        try:
            one = corpus.kernel_features(corp, lex)
        finally:
            corpus.FLOW_FLAGS_DEFAULT = 0
        assert np.array_equal(par.status.cpu().numpy(), one.status.cpu().numpy())
        assert par.feat.cpu().numpy()[ok, :11].tobytes() == one.feat.cpu().numpy()[ok, :11].tobytes()


def test_segment_range_calls_equal_whole_corpus(backend):
    """Chunked pipelines call K1 / K1b on contiguous runs of segments; rows equal the whole-corpus call."""
    import torch
    n = 9 if backend == "emul" else 200
    text, offs = synth.ptx_corpus(seed=31, n_kernels=n, lo=20, hi=300 if backend == "emul" else 3000)
    corp = corpus.upload_corpus(text, offs)
    rt = native.get_runtime()
    lex_all = corpus.lex_records_single_pass(corp)
    fl_all = corpus.kernel_features(corp, lex_all)
    lex = corpus.lex_records_single_pass(corp)                      # allocates the buffers (and fills them once)
    for name in ("hist", "info", "ins", "labels", "meta"):
        getattr(lex, name).zero_()
    feat = torch.zeros_like(fl_all.feat)
    status = torch.full_like(fl_all.status, -1)
    cuts = [0, n // 3, n // 3 + 1, n]
    for s0, s1 in zip(cuts[:-1], cuts[1:]):
        corpus.lex_records_single_pass(corp, out=lex, seg_range=(s0, s1))
        corpus.kernel_features(corp, lex, out_feat=feat, out_status=status, seg_range=(s0, s1))
    assert np.array_equal(lex.hist.cpu().numpy(), lex_all.hist.cpu().numpy())
    assert np.array_equal(lex.info.cpu().numpy(), lex_all.info.cpu().numpy())
    assert np.array_equal(status.cpu().numpy(), fl_all.status.cpu().numpy())
    assert feat.cpu().numpy()[:, :11].tobytes() == fl_all.feat.cpu().numpy()[:, :11].tobytes()


def test_chunk_schedule():
    """Upload schedule of StreamedAnalysis: sizes add up, the head is small, the tail halves down."""
    assert corpus.chunk_schedule(1000, 384) == [384, 384, 232]
    assert corpus.chunk_schedule(1389, 384, 0, 64) == [384, 384, 310, 155, 78, 78]
    assert corpus.chunk_schedule(1389, 384, 96, 0) == [96, 384, 384, 384, 141]
    for total, chunk, head, tail in [(1, 384, 0, 0), (5000, 100, 30, 7), (50, 384, 96, 64), (97, 96, 96, 0)]:
        sizes = corpus.chunk_schedule(total, chunk, head, tail)
        assert sum(sizes) == total and min(sizes) > 0 and max(sizes) <= max(chunk, head)


@pytest.mark.gpu
@pytest.mark.parametrize("pipelines,head,tail", [(1, 0, 0), (2, 0, 0), (3, 1 << 18, 1 << 17)])
def test_streamed_analysis_equals_resident(gpu_only, pipelines, head, tail):
    """StreamedAnalysis (pinned host text, copy overlapped with the kernels; chunks alternating between compute
    streams with their own contexts; short first / last chunks) == analyze on resident text."""
    import torch
    text, offs = synth.ptx_corpus(seed=33, n_kernels=300, lo=20, hi=3000)
    corp = corpus.upload_corpus(text, offs)
    lex, fl = corpus.analyze_corpus(corp)
    host = torch.empty(corp.padded_bytes, dtype=torch.uint8).pin_memory()
    host.copy_(corp.text)
    corp.text.zero_()
    sa = corpus.StreamedAnalysis(gpu_only, corp, host, chunk_bytes=1 << 20, pipelines=pipelines, head_bytes=head, tail_bytes=tail)
    assert len(sa.bounds) > 3 and len(sa.pipes) == pipelines and sa.bounds[0][0] == 0 and sa.bounds[-1][1] == corp.n_segs
    assert all(a[1] == b[0] for a, b in zip(sa.bounds, sa.bounds[1:]))
    seen = []
    feat = sa.run(on_chunk=lambda c, s0, s1, rt: seen.append((c, s0, s1, rt is sa.pipes[c % pipelines][0])))
    feat = sa.run()
    torch.cuda.synchronize()
    assert [x[1:3] for x in seen] == sa.bounds and all(x[3] for x in seen)
    assert np.array_equal(sa.status.cpu().numpy(), fl.status.cpu().numpy())
    assert feat.cpu().numpy()[:, :11].tobytes() == fl.feat.cpu().numpy()[:, :11].tobytes()


def test_long_header_and_launch_shapes(backend):
    """Kernel headers longer than a tile (the opening brace is found tiles after `.entry`), braces and
    `.entry` inside header comments; and the fast path's alternative launch shapes (independent CTAs in
    record mode, barrier-paced CTA in histogram mode) give the same bytes as the default ones."""
    params = ",\n".join(f"\t.param .u64 a_rather_long_parameter_name_number_{i:04d}" for i in range(160))     # ~8 KB
    hdr = ("// .entry ghost() {\n.version 8.0\n.visible .entry real_kernel(\n" + params + "\n) // {{{ not yet\n// { nor this\n{\n")
    body = "".join(f"\tadd.s32 %r{i % 9}, %r{(i + 3) % 9}, {i};\n" for i in range(400))
    src = hdr + "\t.reg .b32 %r<9>;\n" + body + "\tret;\n}\n"
    # a comment on the line before the opening brace, and a nested scope the search must not mistake for the body
    nested = (".visible .entry nest(.param .u64 p) // trailing comment\n{\n\t.reg .b32 %r<4>;\n\tmov.u32 %r1, 1;\n\t{\n"
              "\tadd.s32 %r1, %r1, 1;\n\t}\n\tret;\n}\n")
    _check([src, nested])
    assert corpus.lex_histogram(_corpus([src, nested])).path_counts.cpu().tolist()[:2] == [2, 0]
    text, offs = synth.ptx_corpus(seed=37, n_kernels=6, lo=20, hi=300)
    blob = text + src.encode()
    corp = corpus.upload_corpus(blob, np.concatenate([offs, [len(blob)]]))
    ref_rec, ref_hist = corpus.lex_records(corp), corpus.lex_histogram(corp)
    assert ref_rec.path_counts.cpu().tolist()[:2] == [7, 0]
    for flags in (corpus.LEX_NO_LOCKSTEP, 4):
        corpus.LEX_FLAGS_DEFAULT = flags
        try:
            rec, hist = corpus.lex_records(corp), corpus.lex_histogram(corp)
        finally:
            corpus.LEX_FLAGS_DEFAULT = 0
        for f in ("hist", "info", "ins", "labels", "meta"):
            assert np.array_equal(getattr(rec, f).cpu().numpy(), getattr(ref_rec, f).cpu().numpy()), (flags, f)
        assert np.array_equal(hist.hist.cpu().numpy(), ref_hist.hist.cpu().numpy())
        assert np.array_equal(hist.info.cpu().numpy(), ref_hist.info.cpu().numpy())
    # the exact walk alone, barrier-paced (default) and with independent CTAs
    irregular = _corpus(list(EDGE_CASES.values()) + [src])
    outs = []
    for flags in (0, corpus.LEX_NO_LOCKSTEP):
        corpus.LEX_FLAGS_DEFAULT, corpus.EXACT_ONLY_DEFAULT = flags, True
        try:
            outs.append(corpus.lex_records(irregular))
        finally:
            corpus.LEX_FLAGS_DEFAULT, corpus.EXACT_ONLY_DEFAULT = 0, False
    for f in ("hist", "info", "ins", "labels", "meta"):
        assert np.array_equal(getattr(outs[0], f).cpu().numpy(), getattr(outs[1], f).cpu().numpy()), f


def test_loop_body_larger_than_the_block_list(backend):
    """A counted loop whose body has ~240 basic blocks (more than the 96-entry on-chip body list of K1b),
    next to a small one: trips, weights and counts equal the oracle's."""
    lines = [".visible .entry big_loop(.param .u64 p0)", "{", "\t.reg .b32 %r<9>;", "\t.reg .pred %p<4>;",
             "\tmov.u32 %r1, 0;", "\tmov.u32 %r5, 3;", "SMALL:", "\tadd.s32 %r5, %r5, 2;", "\tsetp.le.s32 %p3, %r5, 40;", "\t@%p3 bra SMALL;",
             "LOOP:"]
    for i in range(120):
        lines += [f"\tsetp.lt.s32 %p2, %r2, {i};", f"\t@%p2 bra S{i};", "\tadd.s32 %r3, %r3, 1;", f"S{i}:", "\tmul.lo.s32 %r4, %r3, 3;"]
    lines += ["\tadd.s32 %r1, %r1, 1;", "\tsetp.lt.s32 %p1, %r1, 10;", "\t@%p1 bra LOOP;", "\tret;", "}", ""]
    _check(["\n".join(lines)])


def _chunk_edge_kernel(name: str, n_stmt: int, branch_at: tuple[int, ...], label_at: tuple[int, ...]) -> str:
    """``n_stmt`` statements; a predicated forward branch at each index of ``branch_at`` and a label in front of each
    statement of ``label_at`` (indices count instructions, as K1b's block numbering does)."""
    lines = [f".visible .entry {name}(.param .u64 p0)", "{", "\t.reg .b32 %r<9>;", "\t.reg .pred %p<4>;"]
    for i in range(n_stmt - 1):
        if i in label_at:
            lines.append(f"T{i}:")
        if i in branch_at:
            lines.append("\t@%p1 bra DONE;")
        else:
            lines.append(f"\tadd.s32 %r{1 + i % 7}, %r{1 + (i + 3) % 7}, {i % 11};")
    lines += ["DONE:", "\tret;", "}", ""]
    return "\n".join(lines)


def test_leader_pass_chunk_edges_and_fallback(backend):
    """flow_kernel<1> numbers the blocks in one visit per statement: leader flags of labels in a shared-memory bit set,
    branch flags as the chunk's ballot shifted by one with a carry into the next chunk of 32, four chunks per trip;
    kernels above 8 192 statements take the flag-array form.  Branches on the last lane of a chunk / of a trip, labels on
    the first, statement counts around 32, 128 and 8 192: rows equal the oracle's and the one-launch kernel's."""
    sizes = [1, 2, 31, 32, 33, 64, 127, 128, 129, 160, 257]
    big = [8191, 8192, 8193] if backend == "emul" else [8191, 8192, 8193, 12000]
    texts = []
    for j, n in enumerate(sizes + big):
        edges = tuple(i for i in (30, 31, 32, 63, 95, 126, 127, 128, 255, 8190, 8191) if i < n - 1)
        labs = tuple(i for i in (0, 1, 32, 64, 127, 128, 129, 256, 8191, 8192) if i < n - 1)
        texts.append(_chunk_edge_kernel(f"edge{j}", n, edges, labs))
    _check(texts[:len(sizes)])
    corp = _corpus(texts)
    lex = corpus.lex_records(corp)
    two = corpus.kernel_features(corp, lex)
    corpus.FLOW_FLAGS_DEFAULT = corpus.FLOW_ONE_KERNEL
    try:
        one = corpus.kernel_features(corp, lex)
    finally:
        corpus.FLOW_FLAGS_DEFAULT = 0
    assert not two.status.cpu().numpy().any() and not one.status.cpu().numpy().any()
    assert two.feat.cpu().numpy()[:, :11].tobytes() == one.feat.cpu().numpy()[:, :11].tobytes()
    k = len(sizes)                                     # the smallest of the large kernels against the oracle as well
    want = np.asarray(orc.kernel_feature_row(texts[k]), dtype=np.float64)
    assert two.feat.cpu().numpy()[k, :11].tobytes() == want.tobytes()
