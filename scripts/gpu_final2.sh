#!/bin/bash
# round-2 final pass: parity tests, smoke, every bench arm and workload, launch list, ncu captures at the bench size
# usage: gpu_final2.sh <tag>
set -x
cd "$(dirname "$0")/.."
TAG=${1:-final}
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q 2>&1 | tail -5
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 900 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err; tail -3 gpurun_out/bench_$TAG.err; cat gpurun_out/bench_$TAG.json
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err; tail -3 gpurun_out/bench_ref_$TAG.err; cat gpurun_out/bench_ref_$TAG.json
for w in c1_latency grid_c3 front1e9 front1e9_3obj; do
  timeout 900 python bench.py --workload $w --steps 6 --warmup 3 > gpurun_out/bench_${w}_$TAG.json 2> gpurun_out/bench_${w}_$TAG.err; tail -3 gpurun_out/bench_${w}_$TAG.err; cat gpurun_out/bench_${w}_$TAG.json
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 160 --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 > gpurun_out/b_ncu_$TAG.log 2>&1; tail -2 gpurun_out/b_ncu_$TAG.log
for k in lex_fast explore_groups; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
# the dataflow step is two launches (flow_kernel<1>, flow_kernel<2>): capture one of each
timeout 900 ncu --set full --clock-control none --import-source on -k regex:flow_kernel -s 2 -c 2 -o gpurun_out/prof_flow_kernel_$TAG python bench.py --steps 1 --warmup 1 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 > gpurun_out/b_ncu_flow_kernel_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_flow_kernel_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:lex_fast -s 2 -c 1 -o gpurun_out/prof_lex_fast_hist_$TAG python scripts/prof_hist.py > gpurun_out/b_ncu_hist_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_hist_$TAG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:predict_grid -s 4 -c 1 -o gpurun_out/prof_predict_grid_$TAG python bench.py --workload grid_c3 --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu_grid_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_grid_$TAG.log
for k in pre_min pre_filter; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s 1 -c 1 -o gpurun_out/prof_${k}_$TAG python bench.py --workload front1e9 --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/b_ncu_${k}_$TAG.log 2>&1; tail -1 gpurun_out/b_ncu_${k}_$TAG.log
done
