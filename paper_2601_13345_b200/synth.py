"""Seeded synthetic inputs of the shapes BASELINE.json names (no network, no datasets).

* ``feature_rows``   — per-kernel dynamic-count rows for the config-grid benchmarks;
* ``ptx_kernel`` / ``ptx_corpus`` — nvcc-shaped PTX text: one ``.entry`` per segment, register
  and shared declarations, pointer arithmetic seeded from ``%tid.x``, counted do-while
  loops, barriers, ``.loc`` lines and comments, opcode mix drawn per kernel from a
  Dirichlet over the nine classes;
* ``candidate_cloud`` — (e, t) clouds for the skyline benchmarks (config C5).

Everything is a pure function of its seed.
"""
from __future__ import annotations

import numpy as np

from .native import FEAT_WIDTH, F_OVR_TEXEC

_POOLS = {
    "MemLoad": ["ld.global.f32 \t%f{a}, [%rd{p}+{o}];", "ld.global.v2.f32 \t{{%f{a}, %f{b}}}, [%rd{p}];",
                "ld.shared.f32 \t%f{a}, [%rd{q}+{o}];", "ld.global.nc.v4.u32 \t{{%r{a}, %r{b}, %r{c}, %r{d}}}, [%rd{p}+{o}];",
                "ld.global.f64 \t%fd{a}, [%rd{p}];", "ld.const.u32 \t%r{a}, [kconst+{o}];",
                "ld.local.u32 \t%r{a}, [%rd{q}];", "ldu.global.f32 \t%f{a}, [%rd{p}];"],
    "MemStore": ["st.global.f32 \t[%rd{p}+{o}], %f{a};", "st.shared.f32 \t[%rd{q}], %f{a};",
                 "st.global.v4.f32 \t[%rd{p}], {{%f{a}, %f{b}, %f{c}, %f{d}}};", "st.global.u64 \t[%rd{p}], %rd{q};"],
    "FP32": ["fma.rn.f32 \t%f{a}, %f{b}, %f{c}, %f{a};", "add.f32 \t%f{a}, %f{b}, %f{c};", "mul.f32 \t%f{a}, %f{b}, 0f3F000000;",
             "sub.f64 \t%fd{a}, %fd{b}, %fd{c};", "div.rn.f32 \t%f{a}, %f{b}, %f{c};"],
    "INT": ["add.s32 \t%r{a}, %r{b}, {o};", "mad.lo.s32 \t%r{a}, %r{b}, %r{c}, %r{d};", "mul.wide.s32 \t%rd{p}, %r{a}, 4;",
            "add.s64 \t%rd{p}, %rd{q}, %rd{p};", "sub.u32 \t%r{a}, %r{b}, %r{c};", "mul.lo.u64 \t%rd{p}, %rd{q}, 8;"],
    "SFU": ["ex2.approx.f32 \t%f{a}, %f{b};", "rcp.rn.f32 \t%f{a}, %f{b};", "rsqrt.approx.f32 \t%f{a}, %f{b};",
            "sqrt.approx.f32 \t%f{a}, %f{b};", "sin.approx.f32 \t%f{a}, %f{b};", "lg2.approx.f32 \t%f{a}, %f{b};"],
    "ALU": ["mov.u32 \t%r{a}, %r{b};", "shl.b32 \t%r{a}, %r{b}, 2;", "cvt.u64.u32 \t%rd{p}, %r{a};", "and.b32 \t%r{a}, %r{b}, 255;",
            "selp.f32 \t%f{a}, %f{b}, %f{c}, %p1;", "setp.gt.f32 \t%p2, %f{a}, %f{b};", "or.b32 \t%r{a}, %r{b}, %r{c};"],
    "Sync": ["bar.sync \t0;", "barrier.sync \t0;", "bar.arrive \t1, 64;", "redux.sync.add.s32 \t%r{a}, %r{b}, -1;"],
    "Other": ["cvta.to.global.u64 \t%rd{p}, %rd{q};", "xor.b32 \t%r{a}, %r{b}, %r{c};", "max.f32 \t%f{a}, %f{b}, %f{c};",
              "shfl.sync.bfly.b32 \t%r{a}, %r{b}, 16, 31, -1;", "neg.s32 \t%r{a}, %r{b};", "sqrt.rn.f32 \t%f{a}, %f{b};",
              "add.u16 \t%rs{a}, %rs{b}, %rs{c};", "lop3.b32 \t%r{a}, %r{b}, %r{c}, %r{d}, 150;",
              "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 \t{{%f{a}, %f{b}}}, {{%r{a}}}, {{%r{b}}}, {{%f{c}, %f{d}}};"],
}
_CLASSES = ("MemLoad", "MemStore", "FP32", "INT", "SFU", "ALU", "Sync", "Other")


def ptx_kernel(rng: np.random.Generator, name: str, n_instr: int, *, comments: bool = True) -> str:
    """One kernel of roughly ``n_instr`` statements."""
    mix = rng.dirichlet(np.full(len(_CLASSES), 0.7))
    n_loops = max(0, int(round(n_instr / 100.0 + rng.normal(0, 0.5))))
    lines = [f".visible .entry {name}(", f"\t.param .u64 {name}_param_0,", f"\t.param .u64 {name}_param_1,",
             f"\t.param .u32 {name}_param_2", ")", "{",
             "\t.reg .pred \t%p<8>;", "\t.reg .b16 \t%rs<16>;", "\t.reg .f32 \t%f<64>;", "\t.reg .b32 \t%r<64>;",
             "\t.reg .f64 \t%fd<16>;", "\t.reg .b64 \t%rd<32>;"]
    if rng.random() < 0.6:
        lines.append(f"\t.shared .align 4 .b8 {name}_tile[{int(rng.choice([256, 512, 1024, 4096, 8192]))}];")
    stride = int(rng.choice([4, 4, 4, 8, 16, 1]))
    lines += ["", f"\tld.param.u64 \t%rd1, [{name}_param_0];", f"\tld.param.u64 \t%rd2, [{name}_param_1];",
              f"\tld.param.u32 \t%r60, [{name}_param_2];", "\tcvta.to.global.u64 \t%rd3, %rd1;",
              "\tcvta.to.global.u64 \t%rd4, %rd2;", "\tmov.u32 \t%r1, %tid.x;", "\tmov.u32 \t%r2, %ctaid.x;",
              "\tmov.u32 \t%r3, %ntid.x;", "\tmad.lo.s32 \t%r4, %r2, %r3, %r1;",
              f"\tmul.wide.s32 \t%rd5, %r{int(rng.choice([1, 4]))}, {stride};", "\tadd.s64 \t%rd6, %rd3, %rd5;",
              "\tadd.s64 \t%rd7, %rd4, %rd5;", f"\tmov.u32 \t%r5, {name}_tile;" if False else "\tmov.u32 \t%r5, 0;",
              "\tcvt.u64.u32 \t%rd8, %r5;"]
    body_budget = max(1, n_instr - 16)
    loop_at = sorted(rng.choice(body_budget, size=min(n_loops, body_budget), replace=False).tolist()) if n_loops else []
    cls_idx = rng.choice(len(_CLASSES), size=body_budget, p=mix)
    regs = rng.integers(6, 60, size=(body_budget, 4))
    ptrs = rng.choice([6, 7, 6, 7, 9, 10], size=(body_budget, 2))
    offs = rng.choice([0, 4, 8, 16, 64, 128], size=body_budget)
    open_loop = None     # (label, counter, bound, remaining)
    loop_id = 0
    for i in range(body_budget):
        if loop_at and loop_at[0] == i and open_loop is None:
            loop_at.pop(0)
            loop_id += 1
            cnt = 40 + (loop_id % 20)
            kind = int(rng.integers(0, 5))
            init, bound, step, cmp_ = [(0, int(rng.integers(2, 200)), 1, "lt"), (int(rng.integers(8, 64)), 0, -1, "gt"),
                                       (0, int(rng.integers(4, 65)) * 4, 4, "ne"), (0, int(rng.integers(2, 100)), 2, "le"),
                                       (0, 0, 1, "dyn")][kind]
            lines.append(f"\tmov.u32 \t%r{cnt}, {init};")
            lines.append(f"$L__BB{name[-3:]}_{loop_id}:")
            open_loop = [f"$L__BB{name[-3:]}_{loop_id}", cnt, bound, step, cmp_, int(rng.integers(3, 30))]
        elif loop_at and loop_at[0] == i:
            loop_at.pop(0)
        c = _CLASSES[cls_idx[i]]
        pool = _POOLS[c]
        tmpl = pool[int(regs[i, 0]) % len(pool)]
        a, b, cc, d = (int(x) for x in regs[i])
        if open_loop is not None and a == open_loop[1]:
            a += 1
        text = tmpl.format(a=a, b=b, c=cc, d=d, p=int(ptrs[i, 0]), q=int(ptrs[i, 1]), o=int(offs[i]))
        if comments and i % 37 == 5:
            lines.append(f"\t.loc\t1 {10 + i % 90} {i % 7}")
        if comments and i % 53 == 7:
            text += " \t// inline note {}".format(i)
        lines.append("\t" + text)
        if open_loop is not None:
            open_loop[5] -= 1
            if open_loop[5] <= 0:
                lab, cnt, bound, step, cmp_, _ = open_loop
                if step >= 0:
                    lines.append(f"\tadd.s32 \t%r{cnt}, %r{cnt}, {step};")
                else:
                    lines.append(f"\tsub.s32 \t%r{cnt}, %r{cnt}, {-step};")
                if cmp_ == "dyn":
                    lines.append(f"\tsetp.lt.s32 \t%p3, %r{cnt}, %r60;")
                else:
                    lines.append(f"\tsetp.{cmp_}.s32 \t%p3, %r{cnt}, {bound};")
                lines.append(f"\t@%p3 bra \t{lab};")
                open_loop = None
    if open_loop is not None:
        lab, cnt, bound, step, cmp_, _ = open_loop
        lines.append(f"\tadd.s32 \t%r{cnt}, %r{cnt}, {abs(step) or 1};")
        lines.append(f"\tsetp.lt.s32 \t%p3, %r{cnt}, {max(bound, 2)};")
        lines.append(f"\t@%p3 bra \t{lab};")
    lines += ["\tst.global.f32 \t[%rd7], %f6;", "\tret;", "}", ""]
    return "\n".join(lines)


# one irregular construct for a kernel of the `irregular` share: text the fast lexer path hands to the exact walk
# (ptx.py:139-141 block comments, :257-270 statements that share or span lines, :232-236 label + statement)
_IRREGULAR = ("\t/* spilled: add.s32 %r9, %r9, 1;\n\t   ret; */ mov.u32 \t%r9, 1;", "\tmov.u32 \t%r9, 1; add.s32 \t%r9, %r9, 1;",
              "\tadd.s32 \t%r9,\n\t\t%r9,\n\t\t1;", "$L__note: mov.u32 \t%r9, 2;")


def ptx_corpus(seed: int, n_kernels: int, lo: int = 50, hi: int = 5000, *, comments: bool = True, irregular: float = 0.0,
               first: int = 0):
    """(text bytes, offsets int64[n_kernels+1]); kernel sizes log-uniform in [lo, hi] statements.
    ``irregular``: share of kernels that carry one construct outside the fast lexer path's grammar.
    ``first``: index of the first kernel (names stay unique when a corpus is generated in pieces)."""
    rng = np.random.default_rng(seed)
    sizes = np.exp(rng.uniform(np.log(lo), np.log(hi), size=n_kernels)).astype(int)
    odd = rng.random(n_kernels) < irregular if irregular > 0 else np.zeros(n_kernels, dtype=bool)
    parts, offs, pos = [], [0], 0
    head = "//\n// synthetic corpus segment\n//\n.version 8.7\n.target sm_100a\n.address_size 64\n\n"
    for k in range(n_kernels):
        txt = (head if comments else "") + ptx_kernel(rng, f"synk_{seed % 1000:03d}_{first + k:06d}", int(sizes[k]), comments=comments)
        if odd[k]:
            at = txt.index("\tcvt.u64.u32")
            txt = txt[:at] + _IRREGULAR[int(rng.integers(0, len(_IRREGULAR)))] + "\n" + txt[at:]
        b = txt.encode("ascii")
        parts.append(b)
        pos += len(b)
        offs.append(pos)
    return b"".join(parts), np.asarray(offs, dtype=np.int64)


def feature_rows(seed: int, n_kernels: int) -> tuple[np.ndarray, np.ndarray]:
    """(feat float64 [K, FEAT_WIDTH], res int64 [K, 2]) with both branches of every model
    conditional exercised (t_exec above and below tau_short, cap-limited or not)."""
    rng = np.random.default_rng(seed)
    feat = np.zeros((n_kernels, FEAT_WIDTH), dtype=np.float64)
    scale = np.exp(rng.uniform(np.log(10.0), np.log(2e6), size=n_kernels))
    mix = rng.dirichlet(np.full(6, 0.8), size=n_kernels)
    counts = np.floor(mix * scale[:, None])
    feat[:, 0] = counts[:, 0]                                  # n_mem
    feat[:, 1] = counts[:, 0] * rng.choice([4.0, 4.0, 8.0, 16.0], size=n_kernels)
    feat[:, 2:6] = counts[:, 1:5]                              # FP32 INT SFU ALU
    feat[:, 6] = np.floor(counts[:, 5] / 50.0)                 # n_sync
    feat[:, 7] = rng.choice([0.0, 0.25, 0.5, 0.75, 1.0, 1.0], size=n_kernels)
    feat[:, 8] = rng.choice([0, 0, 512, 4096, 16384], size=n_kernels)
    feat[:, 9] = rng.integers(16, 255, size=n_kernels)
    feat[:, 10] = np.floor(scale / 8.0)
    feat[rng.random(n_kernels) < 0.05, 0:2] = 0.0              # pure-compute kernels: ci = inf
    feat[:, F_OVR_TEXEC] = np.nan
    res = np.zeros((n_kernels, 2), dtype=np.int64)
    res[:, 0] = rng.choice([0, 0, 0, 1024, 8192, 32768], size=n_kernels)
    res[:, 1] = np.floor(np.exp(rng.uniform(0.0, np.log(65536.0), size=n_kernels))).astype(np.int64)
    return feat, res


def candidate_cloud(seed: int, n: int, kind: str = "uniform") -> tuple[np.ndarray, np.ndarray]:
    rng = np.random.default_rng(seed)
    if kind == "uniform":
        return rng.uniform(0.0, 10.0, n), rng.uniform(0.0, 10.0, n)
    if kind == "tied":          # clustered values force exact ties in both objectives
        return rng.integers(0, 40, n).astype(np.float64) / 4.0, rng.integers(0, 40, n).astype(np.float64) / 4.0
    if kind == "anticorrelated":
        e = rng.uniform(0.0, 10.0, n)
        return e, 10.0 - e + rng.normal(0.0, 0.5, n)
    raise ValueError(kind)
