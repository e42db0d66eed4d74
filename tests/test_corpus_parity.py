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


@pytest.mark.parametrize("seed,default_trip", [(4, 32.0), (9, 7.5)])
def test_synthetic_corpus(backend, seed, default_trip):
    n = 16 if backend == "emul" else 600
    text, offs = synth.ptx_corpus(seed=seed, n_kernels=n, lo=20, hi=700 if backend == "emul" else 5000)
    _check([text[offs[i]:offs[i + 1]].decode("ascii") for i in range(n)], default_trip)


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
