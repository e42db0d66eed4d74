#!/usr/bin/env python
"""cProfile of the configs[0] session (one PTX file through the drop-in API)."""
import cProfile, pstats, sys, io
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch
import bench_extra
from paper_2601_13345_b200 import api
src, kern = bench_extra._c1_source()
a, p = api.default_architecture(), api.default_calibration()
res = api.compute_input_resources(128, 4, 16, 64, 4, a, rule="generic")
def session():
    m = api.parse_ptx(src, kern)
    cfg = api.estimate_trip_counts(api.build_cfg(m), m)
    return api.pareto_explore(m, cfg, a, p, res, bench_extra.DIMS, bench_extra.CAPS, rho=0.95)
for _ in range(3): session()
pr = cProfile.Profile(); pr.enable()
for _ in range(5): session()
torch.cuda.synchronize(); pr.disable()
s = io.StringIO(); pstats.Stats(pr, stream=s).sort_stats("cumulative").print_stats(32); print(s.getvalue()[:6000])
