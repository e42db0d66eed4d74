#!/bin/bash
# ncu --set full of the step's kernels.  usage: gpu_prof.sh <tag> <kernels-per-rank> [kernel-regexes...]
cd "$(dirname "$0")/.."
TAG=$1; K=$2; shift; shift
mkdir -p gpurun_out
for k in "$@"; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels $K > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
