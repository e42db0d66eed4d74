#!/bin/bash
# e2e pipeline experiments: streamed-analysis parity, then one bench run with extra e2e settings.  usage: gpu_e2e_sweep.sh <tag> <sweep> [bench args]
set -x
cd "$(dirname "$0")/.."
TAG=${1:-sweep}; SWEEP=$2; shift 2
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -k "streamed or grid or explore or extension" 2>&1 | tail -5
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 --e2e-sweep "$SWEEP" "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; grep "e2e sweep" gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; python - <<P
import json
d=json.loads(open("gpurun_out/bench_$TAG.json").read().strip().splitlines()[-1])
print(d["ms_per_step"], d["phases_ms"], d["e2e"]["ms_per_step"], d["e2e"]["timeline_ms"])
P
