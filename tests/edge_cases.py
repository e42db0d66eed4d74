"""Hand-written PTX edge cases (SURVEY Appendix B behaviours and lexer corner cases).
Inputs only; the expected outputs come from the reference (tests/golden/make_golden.py)."""

def _k(body: str, name: str = "k", header: str = "", params: str = "()") -> str:
    return f"{header}.visible .entry {name}{params}\n{{\n{body}\n}}\n"


EDGE_CASES = {
    "bar_only": _k("bar.sync 0;"),
    "block_comment_multi": _k("/* a; b;\n c; */ add.s32 %r1, %r2, 1;\n ret;"),
    "line_comment_brace": _k("add.s32 %r1, %r2, 1; // }\n ret;"),
    "entry_in_comment": "// .entry fake {\n/* .entry fake2 { */\n" + _k("ret;", name="real"),
    "multiline_call": _k("call.uni (r),\n foo,\n (a,\n b);\n ret;"),
    "two_on_line": _k("add.s32 %r1, %r2, 1; ret;"),
    "label_same_line": _k("L1: bra L1;"),
    "nested_scope": _k("{\n .reg .b32 t;\n mov.u32 %r1, %r2;\n}\n ret;"),
    "loc_no_semi": _k(".loc 1 5 0\n add.f32 %f1, %f2, %f3;\n .loc 1 6 0\n ret;"),
    "func_before": ".func foo()\n{\n add.s32 %r1, %r1, 1;\n ret;\n}\n" + _k("mov.u32 %r1, %r2;\n ret;"),
    "weak_entry": ".weak .entry w()\n{\n ret;\n}\n",
    "bare_entry": ".entry b()\n{\n exit;\n}\n",
    "maxntid": ".visible .entry m()\n.maxntid 256, 1, 1\n.minnctapersm 2\n{\n ret;\n}\n",
    "shared_decls": _k(".shared .align 16 .f32 a[64];\n .shared .b8 b[3];\n .shared .u64 c;\n .shared .f32 d[16][16];\n .shared .align 4 .weird e[5];\n ret;"),
    "module_shared": ".shared .f32 outside[64];\n.extern .shared .b8 dyn[];\n" + _k("ret;"),
    "dup_label": _k("L: add.s32 %r1, %r1, 1;\nL: sub.s32 %r1, %r1, 1;\n bra L;"),
    "label_at_end": _k("bra END;\n add.s32 %r1, %r1, 1;\nEND:"),
    "crlf": _k("add.s32 %r1, %r2, 1;\r\n ret;\r"),
    "vector_ld": _k("ld.global.v4.f32 {%f1,%f2,%f3,%f4}, [%rd1+16];\n st.global.v2.f64 [%rd2], {%fd1, %fd2};\n ret;"),
    "reg_decls": _k(".reg .pred %p<2>;\n .reg .f32 %f<4>;\n .reg .b32 %r<6>;\n .reg .b64 %rd<11>;\n .reg .b32 %r1<3>;\n .reg .b32 %x<2>, %y<2>;\n .reg .f32 %f<4>;\n ret;"),
    "pred_variants": _k("@%p1 bra L;\n @!%p2 add.s32 %r1, %r1, 1;\n @p3 mov.u32 %r1, 0;\n @%p4\tret;\nL: ret;"),
    "no_entry": ".version 7.0\n.func f() { ret; }\n",
    "no_body": ".visible .entry nb()\n",
    "unbalanced": ".visible .entry ub()\n{\n { add.s32 %r1, %r1, 1;\n ret;\n}\n",
    "empty_body": _k("\n // nothing\n"),
    "unterminated": _k("add.s32 %r1, %r2,\n 1"),
    "undefined_label": _k("bra NOWHERE;\n ret;"),
    "slash_star_in_line_comment": _k("add.s32 %r1, %r1, 1; // open /* here\n sub.s32 %r2, %r2, 1; */ mul.lo.s32 %r3, %r3, 2;\n ret;"),
    "slash_slash_star": _k("mov.u32 %r1, 1; //* tricky */ mov.u32 %r2, 2;\n ret;"),
    "block_closes_in_line": _k("mov.u32 %r1, 1; // a /* b */ c ; mov.u32 %r9, 9;\n ret;"),
    "star_slash_only": _k("mov.u32 %r1, 1; */ mov.u32 %r2, 2;\n ret;"),
    "slash_star_slash": _k("mov.u32 %r1, 1; /*/ mov.u32 %r2, 2; */ mov.u32 %r3, 3;\n ret;"),
    "unterminated_block_comment": _k("mov.u32 %r1, 1;\n ret;") + "/* trailing without close\n",
    "unterminated_block_in_body": _k("mov.u32 %r1, 1; /* never closed\n add.s32 %r2, %r2, 1; // x /* y\n ret;"),
    "unterminated_after_closed": _k("mov.u32 %r1, 1; /* ok */ mov.u32 %r2, 2; /* open\n sub.s32 %r3, %r3, 1;\n ret;"),
    "unterminated_star_slash_trick": _k("mov.u32 %r1, 1; /*/ add.s32 %r2, %r2, 1;\n ret;"),
    "semicolons": _k(";;; add.s32 %r1, %r1, 1;; ;\n ret;"),
    "label_colon_space": _k("L1:   add.s32 %r1, %r1, 1;\n$L__BB0_2:\n\tbra \t$L__BB0_2;"),
    "colon_opcode": _k("ld.global.L2::128B.f32 %f1, [%rd1];\n ret;"),
    "brace_statement": _k("{ .reg .b32 t; mov.u32 t, 1; }\n ret;"),
    "directive_multi": _k(".reg .b32 %r<4>; add.s32 %r1, %r2, 3; .pragma \"nounroll\";\n ret;"),
    "pending_then_directive": _k("add.s32 %r1,\n .reg .b32 %q<2>;\n ret;"),
    "pending_label_like": _k("add.s32 %r1, %r2,\nL9: 1;\n bra L0;\nL0: ret;"),
    "pending_brace": _k("mov.u32 %r1,\n{\n}\n 5;\n ret;"),
    "tabs_everywhere": _k("\t\tadd.s32\t%r1,\t%r2,\t1\t;\t\tret\t;"),
    "form_feed_ws": _k("add.s32 %r1,\x0c%r2,\x0b1;\n\x1cret\x1f;"),
    "body_same_line": ".visible .entry s() { mov.u32 %r1, 1; ret; }\n",
    "body_end_mid": ".visible .entry s()\n{\n mov.u32 %r1, 1; ret; } trailing garbage ; add.s32 %r1, %r1, 1;\n",
    "second_kernel_ignored": _k("ret;", name="first") + _k("add.s32 %r1, %r1, 1;\n ret;", name="second"),
    "entry_glued": "foo.entry glued()\n{\n ret;\n}\n",
    "entry_bad_then_good": ".entry 9bad() { ret; }\n.entry good()\n{\n exit;\n}\n",
    # capacities lifted in round 2: more than 12 operands (span record), more than 32 .reg declarations
    "many_operands": _k("call.uni (rv), fn, (" + ", ".join(f"p{i}" for i in range(9)) + ");\n"
                        " op.z %r1, " + ", ".join(f"%r{i}" for i in range(2, 22)) + ";\n"
                        " op.w %r1, {%r2, %r3}, [%rd1+4], " + ", ".join(str(i) for i in range(14)) + " ,\n  sym9 , // tail\n  (a, b) ;\n ret;"),
    "many_reg_decls": _k("\n".join(f" .reg .{('b32', 'f32', 'b64', 'pred')[i % 4]} %q{chr(97 + i % 26)}{chr(97 + i // 26)}<{i + 1}>;" for i in range(40)) + "\n .reg .f32 %f<5>;\n ret;"),
    "classes": _k("\n".join(f"{op} %r1, %r2;" for op in (
        "bar.arrive", "redux.sync.add.s32", "barrier.cta.sync", "vote.sync.ballot.b32", "shfl.sync.bfly.b32",
        "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32", "ldmatrix.sync.aligned.m8n8.x4.shared.b16",
        "ld.const.f32", "ld.f32", "ldu.global.f32", "st.param.f32", "st.local.u8", "mul.hi.u32", "add.cc.u32",
        "mad.lo.cc.u32", "addc.u32", "mul24.lo.s32", "rem.s32", "min.f32", "xor.b32", "not.pred", "lop3.b32",
        "cvta.to.global.u64", "add.u16", "fma.rn.f16x2", "fma.rn.bf16", "sqrt.rn.f32", "sqrt.approx.f32",
        "tanh.approx.f32", "brx.idx", "call.uni", "ret", "exit", "rcp.rn.f32", "sub.f64", "div.rn.f32", "div.s32",
        "cvt.rn.f32.s32", "selp.f32", "sync", "foo.sync.", "atom.global.add.u32", "red.global.add.f32",
        "membar.gl", "cp.async.ca.shared.global", "tcgen05.mma.cta_group::1.kind::f16", "bra.uni",
        "ld.global.v2.v4.f32.f64", "st.shared.global.u16", "setp.lt.and.s32", "mov.b64", "shr.u32", "and.pred"))
        + "\nT: ret;").replace("bra.uni %r1, %r2;", "bra.uni T;"),
    # `//` comments longer than a 4 KB tile (the lexer closes the line at the tile edge and carries the comment state):
    # a comment-only line, a comment behind a statement, one spanning three tiles, one holding "/*" and "*/"
    "long_line_comment": _k("add.s32 %r1, %r2, 1;\n // " + "x" * 5000 + "\n sub.s32 %r1, %r1, 2;\nL: bra L;\n ret;"),
    "long_trailing_comment": _k("add.s32 %r1, %r2, 1; // " + "y; " * 1700 + "\n @%p1 sub.s32 %r1, %r1, 2; // short\n ret;"),
    "huge_line_comment": "// " + "z{" * 6500 + "\n" + _k("ld.global.f32 %f1, [%rd1]; //" + "/" * 9000 + "\n st.global.f32 [%rd1], %f1;\n ret;"),
    "long_comment_with_block_marks": _k("mov.u32 %r1, 1; // " + "a" * 3000 + " /* " + "b" * 3000 + " */ " + "c" * 3000 + "\n mov.u32 %r2, 2;\n ret;"),
    # module-level lines longer than a tile in front of the kernel (initialiser lists are emitted on one line), a
    # one-line parameter list of 9 KB, a 6 KB block comment without a newline, `.entry` decoys inside the long lines
    "long_const_initialiser": ".version 8.0\n.const .align 4 .b8 table[16384] = {" + ", ".join(str(i % 251) for i in range(16384)) + "};\n"
                              + ".global .align 1 .b8 $str[9000] = {" + ", ".join("46" for _ in range(9000)) + "};\n" + _k("ld.const.u8 %rs1, [table+5];\n ret;"),
    "long_param_line": ".visible .entry wide(" + ", ".join(f".param .u64 wide_param_{i}" for i in range(400)) + ") { // {\n add.s32 %r1, %r1, 1;\n ret;\n}\n",
    "long_block_comment_before": "/* " + "no newline here .entry ghost { " * 200 + "*/ .version 8.0 /* " + "x" * 4200 + " */ " + _k("mov.u32 %r1, 7;\n ret;"),
    "long_line_then_entry_same_line": ".global .b32 g[3000] = {" + ", ".join("7" for _ in range(3000)) + "}; .visible .entry tail()\n{\n bar.sync 0;\n ret;\n}\n",
}
