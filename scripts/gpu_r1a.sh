set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -15
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -5
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r1a.json 2> gpurun_out/bench_r1a.err; tail -3 gpurun_out/bench_r1a.err; cat gpurun_out/bench_r1a.json
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_r1a.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --kernels 8192 > gpurun_out/b_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:predict_grid -s 1 -c 1 -o gpurun_out/prof_grid_r1a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 8192 > gpurun_out/b_ncu2.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:skyline_group -s 1 -c 1 -o gpurun_out/prof_sky_r1a python bench.py --steps 1 --warmup 1 --no-cpu-baseline --kernels 8192 > gpurun_out/b_ncu3.log 2>&1
ls -la gpurun_out
