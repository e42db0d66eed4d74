#!/usr/bin/env python
"""Executed-instruction mix per kernel from the ncu reports of a tag (ncu --page source --print-source sass):
warp instructions by SASS opcode, with the active threads per instruction.  usage: sass_mix.py <tag>"""
import collections
import csv
import io
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
tag = sys.argv[1]
out = [f"# executed SASS mix per kernel ({tag}); one launch each, ncu --set full --import-source on"]
for rep in sorted((ROOT / "gpurun_out").glob(f"prof_*_{tag}.ncu-rep")):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        continue
    name = rows[0][1] if rows[0] and rows[0][0] == "Kernel Name" else rep.name
    hdr = rows[1]
    ix, it, isrc = hdr.index("Instructions Executed"), hdr.index("Thread Instructions Executed"), hdr.index("Source")
    agg, tot, static = collections.defaultdict(lambda: [0.0, 0.0]), 0.0, 0
    for r in rows[2:]:
        if len(r) <= it:
            continue
        try:
            n, t = float(r[ix]), float(r[it])
        except ValueError:
            continue
        s = r[isrc].strip()
        if s.startswith("@"):
            s = s.split(None, 1)[1] if " " in s else s
        op = s.split()[0].split(".")[0] if s else "?"
        agg[op][0] += n; agg[op][1] += t; tot += n; static += 1
    out.append(f"\n## {rep.name}: {name[:90]}\nstatic instructions {static}, executed warp instructions {tot / 1e6:.1f} M")
    ctrl = sum(agg[o][0] for o in ("ISETP", "BRA", "BSSY", "BSYNC", "SEL", "PLOP3", "BREAK", "WARPSYNC", "BMOV", "EXIT", "CALL", "RET"))
    tma = sum(n for o, (n, _) in agg.items() if o.startswith(("UTMA", "UBLKCP", "TCGEN", "UTC")))
    out.append(f"control flow (ISETP BRA BSSY BSYNC SEL PLOP3 BREAK ...): {ctrl / max(tot, 1) * 100:.1f}%;  TMA / tcgen05 instructions: {tma:.0f} (none: byte / integer / fp64 stream kernels)")
    for op, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:16]:
        out.append(f"  {op:10s} {n / 1e6:9.1f} M {n / max(tot, 1) * 100:5.1f}%  threads/inst {t / max(n, 1):5.1f}")
(ROOT / "profiles" / f"sass_mix_{tag}.txt").write_text("\n".join(out) + "\n")
print("\n".join(out)[:2500])
