#!/usr/bin/env python
"""Top source lines of one .ncu-rep by stall samples and by executed instructions
(ncu --page source --print-source cuda,sass; needs -lineinfo).  usage: ncu_hot_lines.py rep [N]"""
import csv, io, subprocess, sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, hdr = [], "?", None
for r in csv.reader(io.StringIO(txt)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if r[0] in ("Function Name",) or hdr is None or not r[0].isdigit():
        continue
    d = dict(zip(hdr[4:], r[4:]))
    def num(k):
        try: return float(d.get(k, "0").replace(",", ""))
        except ValueError: return 0.0
    rows.append((fname, int(r[0]), r[1].strip()[:90], num("# Samples"), num("Instructions Executed"),
                 num("Thread Instructions Executed"), num("L1 Wavefronts Shared"), num("L1 Wavefronts Shared Ideal")))
# a line can appear several times (inlined at several places): merge
agg = {}
for f, ln, src, smp, ins, tins, wf, wfi in rows:
    a = agg.setdefault((f, ln), [src, 0, 0, 0, 0, 0]); a[1] += smp; a[2] += ins; a[3] += tins; a[4] += wf; a[5] += wfi
tot_s = sum(a[1] for a in agg.values()) or 1; tot_i = sum(a[2] for a in agg.values()) or 1
print(f"total samples {tot_s:.0f}  warp instructions {tot_i:.0f}  smem wavefronts {sum(a[4] for a in agg.values()):.0f} (ideal {sum(a[5] for a in agg.values()):.0f})")
for title, key in (("by stall samples", 1), ("by warp instructions", 2)):
    print(f"\n== {title}")
    for (f, ln), a in sorted(agg.items(), key=lambda kv: -kv[1][key])[:top]:
        print(f"{a[1]/tot_s*100:5.1f}%s {a[2]/tot_i*100:5.1f}%i thr/inst {a[3]/max(a[2],1):4.1f} wf {a[4]/max(a[5],1):4.1f}x  {f}:{ln}  {a[0]}")
