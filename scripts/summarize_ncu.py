#!/usr/bin/env python
"""Summarise gpurun_out/*.ncu-rep and the launch list into small text files under profiles/."""
import csv, io, subprocess, sys, json
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
OUT = ROOT / "profiles"
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__thread_inst_executed_per_inst_executed.ratio", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers", "launch__waves_per_multiprocessor",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum", "sm__inst_executed_pipe_fp64.sum",
        "smsp__inst_executed_pipe_fp64.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "lts__t_bytes.sum", "sm__cycles_elapsed.max"]


def raw(rep: Path):
    txt = subprocess.run(["ncu", "-i", str(rep), "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    if len(rows) < 3:
        return []
    hdr, units = rows[0], rows[1]
    return [{h: (v, u) for h, u, v in zip(hdr, units, vals)} for vals in rows[2:] if len(vals) == len(hdr)]   # one per captured launch


def main(tag: str):
    OUT.mkdir(exist_ok=True)
    lines = [f"# ncu --set full summaries ({tag}); one launch per kernel, cold cache, --clock-control none"]
    traffic = {}
    for rep in sorted((ROOT / "gpurun_out").glob(f"prof_*_{tag}.ncu-rep")):
      for m in raw(rep):
        name = m.get("Kernel Name", ("?", ""))[0]
        lines.append(f"\n## {rep.name}: {name}")
        for w in WANT:
            if w in m:
                lines.append(f"{w:70s} {m[w][0]:>16s} {m[w][1]}")
        def num(key):
            v, u = m.get(key, ("0", ""))
            f = float(v.replace(",", "")) if v else 0.0
            return f * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}.get(u, 1.0)
        tr = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        dur, du = m.get("gpu__time_duration.sum", ("0", "ns"))
        dur_s = float(dur.replace(",", "")) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}.get(du, 1e-9)
        lines.append(f"{'dram traffic (read+write)':70s} {tr/1e6:16.3f} MB  -> {tr/1e9/max(dur_s,1e-12):.1f} GB/s over {dur_s*1e3:.3f} ms")
        base = name.split('(')[0].split('::')[-1]
        key = base if base.startswith('flow_kernel<') else base.split('<')[0]          # flow_kernel<1> / <2> are two kernels
        traffic[key + ('_hist' if '_hist_' in rep.name else '')] = tr
    (OUT / f"ncu_full_{tag}.txt").write_text("\n".join(lines) + "\n")
    # launch list
    src = ROOT / "gpurun_out" / f"launches_{tag}.csv"
    if src.exists():
        body = [l for l in src.read_text().splitlines() if not l.startswith("==")]
        rows = list(csv.DictReader(body))
        agg = {}
        for r in rows:
            if r.get("Metric Name") != "gpu__time_duration.sum":
                continue
            k = r["Kernel Name"].split("(")[0][-70:]
            v = float(r["Metric Value"].replace(",", "")) * {"ns": 1e-9, "us": 1e-6, "ms": 1e-3}.get(r["Metric Unit"], 1e-9)
            a = agg.setdefault(k, [0, 0.0])
            a[0] += 1; a[1] += v
        tot = sum(a[1] for a in agg.values()) or 1.0
        out = [f"# ncu launch list ({tag}): gpu__time_duration.sum per kernel over the captured launches (cold-cache, serialised; compare SHARES)",
               f"{'kernel':72s} {'launches':>8s} {'total ms':>10s} {'avg us':>10s} {'share':>7s}"]
        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            out.append(f"{k:72s} {n:8d} {t*1e3:10.3f} {t/n*1e6:10.1f} {100*t/tot:6.1f}%")
        (OUT / f"launches_{tag}.txt").write_text("\n".join(out) + "\n")
    (OUT / f"traffic_{tag}.json").write_text(json.dumps(traffic, indent=1) + "\n")
    # bench.py reads profiles/traffic.json: keep the newest capture of every kernel, with the tag it came from
    latest = OUT / "traffic.json"
    merged = json.loads(latest.read_text()) if latest.exists() else {}
    for k, v in traffic.items():
        merged[k] = {"dram_bytes_per_launch": v, "capture": tag, "kernels_per_launch": int(sys.argv[2]) if len(sys.argv) > 2 else None}
    latest.write_text(json.dumps(merged, indent=1) + "\n")
    print((OUT / f"ncu_full_{tag}.txt").read_text()[:3000])


if __name__ == "__main__":
    main(sys.argv[1] if len(sys.argv) > 1 else "r1a")
