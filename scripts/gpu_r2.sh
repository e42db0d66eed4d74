#!/bin/bash
# round-2 GPU pass.  usage: gpu_r2.sh <tag> "<pytest -k expr or empty>" "<ncu kernel regexes>" [bench args]
set -x
cd "$(dirname "$0")/.."
TAG=${1:-r2}; KEXPR=$2; NCU_K=$3; shift; shift; shift
mkdir -p gpurun_out
if [ -n "$KEXPR" ]; then timeout 1500 python -m pytest tests -m gpu -x -q -k "$KEXPR" 2>&1 | tail -8; fi
timeout 900 python bench.py --steps 6 --warmup 3 "$@" > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
for k in $NCU_K; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline "$@" > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
