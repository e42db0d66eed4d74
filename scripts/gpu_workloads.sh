#!/bin/bash
# every bench workload once (short runs).  usage: gpu_workloads.sh <tag>
set -x
cd "$(dirname "$0")/.."
TAG=${1:-wl}
mkdir -p gpurun_out
timeout 900 python bench.py --steps 6 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -5 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
for w in c1_latency grid_c3 front1e9 front1e9_3obj; do
  timeout 900 python bench.py --workload $w --steps 4 --warmup 3 > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err; tail -5 gpurun_out/bench_${w}_$TAG.err; cat gpurun_out/bench_${w}_$TAG.json
done
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -3 gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
