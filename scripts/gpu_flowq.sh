#!/bin/bash
# quick look at the dataflow kernels: resident bench phases + per-launch times
cd "$(dirname "$0")/.."
timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 --e2e-sweep "" > gpurun_out/bench_fq.json 2>gpurun_out/bench_fq.err; python -c "
import json
d=json.loads(open('gpurun_out/bench_fq.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['phases_ms'], d['e2e']['ms_per_step'])"
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:flow_kernel -c 4 --csv --log-file gpurun_out/launches_fq.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 > /dev/null 2>&1; grep flow_kernel gpurun_out/launches_fq.csv | awk -F'","' '{print $5, $NF}' | tail -4
