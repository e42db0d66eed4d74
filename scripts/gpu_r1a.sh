#!/bin/bash
# round-1 first GPU pass: parity tests, smoke, bench, ncu launch list + full captures
set -x
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,memory.total --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -5 gpurun_out/bench_r1a.err; cat gpurun_out/bench_r1a.json
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu.log 2>&1; tail -3 gpurun_out/b_ncu.log
for k in predict_grid skyline_group lex_corpus flow_kernel; do
  timeout 400 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${k}_r1a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 9600 > gpurun_out/b_ncu_$k.log 2>&1; tail -2 gpurun_out/b_ncu_$k.log
done
ls -la gpurun_out
