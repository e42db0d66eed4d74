#!/bin/bash
# quick GPU pass: parity tests + bench + launch list.  usage: gpu_quick.sh <tag> [pytest-args]
set -x
cd "$(dirname "$0")/.."
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_$TAG.log 2>&1; tail -2 gpurun_out/b_ncu_$TAG.log
for k in $NCU_FULL; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s ${NCU_SKIP:-2} -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
