#!/bin/bash
# A/B of bench variants: usage gpu_ab.sh <tag> "<flagsA>" "<flagsB>" ...
cd "$(dirname "$0")/.."
TAG=$1; shift
mkdir -p gpurun_out
i=0
for f in "$@"; do
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $f > gpurun_out/ab_${TAG}_$i.json 2> gpurun_out/ab_${TAG}_$i.err || tail -5 gpurun_out/ab_${TAG}_$i.err
  python - <<PY
import json
d=json.load(open("gpurun_out/ab_${TAG}_$i.json"))
print("$f", {k:d[k] for k in ("ms_per_step","phases_ms","ptx_gb_per_s_lexer_only","ptx_gb_per_s_histogram_mode")}, "e2e ms", d["e2e"]["ms_per_step"])
PY
  i=$((i+1))
done
