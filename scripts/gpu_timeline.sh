for cfg in "384 64 2" "192 0 2" "384 0 1"; do set -- $cfg
timeout 600 python bench.py --steps 4 --warmup 3 --no-cpu-baseline --nvcc-mb 0 --irregular-leg 0 --e2e-chunk-mb $1 --e2e-tail-mb $2 --e2e-pipelines $3 > gpurun_out/tl.json 2>gpurun_out/tl.err; python - <<P
import json
d=json.loads(open("gpurun_out/tl.json").read().strip().splitlines()[-1])
print("$cfg", d["e2e"]["ms_per_step"], d["e2e"]["timeline_ms"])
P
done
