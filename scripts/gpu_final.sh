#!/bin/bash
# round-end GPU pass: parity tests, smoke, both bench arms, launch list of the bench command, ncu full captures at the bench size
# usage: gpu_final.sh <tag>
set -x
cd "$(dirname "$0")/.."
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -3 gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu_$TAG.log 2>&1; tail -2 gpurun_out/b_ncu_$TAG.log
for k in lex_fast flow_kernel skyline_group predict_grid; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
# histogram-mode lexer: the 4th..: launches after the record-mode ones of the e2e leg
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lex_fast_kernel.*0 -s 1 -c 1 -o gpurun_out/prof_lex_fast_hist_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu_hist_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_hist_$TAG.log
