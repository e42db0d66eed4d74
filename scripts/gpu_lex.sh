#!/bin/bash
# lexer-focused GPU pass: parity tests, bench, launch list, ncu full captures of the fast lexer in both modes.
# usage: gpu_lex.sh <tag> [full]
set -x
cd "$(dirname "$0")/.."
TAG=${1:-q}
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -8
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_$TAG.log 2>&1; tail -2 gpurun_out/b_ncu_$TAG.log
if [ "$2" = "full" ]; then
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:lex_fast -s 2 -c 1 -o gpurun_out/prof_lex_fast_rec_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_rec_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_rec_$TAG.log
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:lex_fast -s 10 -c 1 -o gpurun_out/prof_lex_fast_hist_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_hist_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_hist_$TAG.log
fi
