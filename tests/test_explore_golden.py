"""BASELINE configs[0] and configs[1] end to end against the reference itself (tests/golden/ref_explore.json,
written by tests/golden/make_golden_explore.py from /root/reference): nvcc tiled-matmul / conv2d / MHA PTX
(and the mha_like fixture) x dims 1..1024 (464 shapes) x 7 caps x every modelled spec x seq_len sweeps.
Three routes, all bit-exact: the drop-in api (parse -> cfg -> trips -> evaluate_configs / pareto_explore),
the batched engine path (score_grid -> skyline_groups), and the one-launch sweep (pareto_explore_sweep)."""
from __future__ import annotations

import hashlib
import json
from pathlib import Path

import numpy as np
import pytest
import torch

from paper_2601_13345_b200 import api, engine, native, specs
from paper_2601_13345_b200 import errors as E

G = Path(__file__).parent / "golden"
EXP = json.loads((G / "ref_explore.json").read_text())
PARSE = json.loads((G / "ref_parse.json").read_text())
MODEL = json.loads((G / "ref_model.json").read_text())
FIXT = json.loads((G / "ref_fixtures.json").read_text())
DIMS = list(range(1, 1025))
CAPS = EXP["caps"]
hx = float.hex


def _spec(name):
    if name == "alt":
        return specs.architecture_from_dict(MODEL["alt_spec"]["arch"]), specs.calibration_from_dict(MODEL["alt_spec"]["calibration"])
    return specs.load_profile(specs.SPEC_DIR / name.split(":", 1)[1])


def _source(key):
    kind, name = key.split(":")
    return (PARSE[name]["source"], PARSE[name]["kernel"]) if kind == "parse" else (FIXT["sources"][name], None)


def _row_text(p) -> str:
    c = p.config
    return f"{c.block_x},{c.block_y},{hx(c.p_cap)},{hx(p.time.t_exec)},{hx(p.power.p_dyn)},{hx(p.e_pred)},{int(p.power.cap_limited)}"


def _front_rows(entries):
    return [f"{e.config.block_x},{e.config.block_y},{hx(e.config.p_cap)}" for e in entries]


def _check_front(case, entries, t_peak):
    rows = _front_rows(entries)
    assert len(rows) == case["front_n"]
    if "front" in case:
        assert [[e.config.block_x, e.config.block_y, e.config.p_cap] for e in entries] == case["front"]
    else:
        for i, want in case["front_sample"].items():
            assert rows[int(i)] == want
    assert hashlib.sha256("\n".join(rows).encode()).hexdigest() == case["front_sha256"]
    assert hx(t_peak) == case["t_peak"]


def _cases(backend):
    cases = [c for c in EXP["cases"] if "error" not in c]
    if backend == "emul":            # emulated kernels: one case per kernel family
        keep, seen = [], set()
        for c in cases:
            key = (c["kernel"], c["spec"] == "file:synthetic-48sm.json")
            if key not in seen and (c["seq_len"] in (128, 2048)):
                seen.add(key)
                keep.append(c)
        cases = keep[:6]
    return cases


def test_dropin_api_reproduces_reference_explore(backend):
    modules = {}
    for case in _cases(backend):
        if case["source"] not in modules:
            src, kern = _source(case["source"])
            m = api.parse_ptx(src, kern)
            modules[case["source"]] = (m, api.estimate_trip_counts(api.build_cfg(m), m))
        m, cfg = modules[case["source"]]
        a, p = _spec(case["spec"])
        res = api.compute_input_resources(case["seq_len"], 4, 16, 64, 4, a, rule=case["rule"])
        assert [res.shared_mem_bytes, res.grid_x, res.grid_y, res.grid_z] == case["resources"]
        cfgs = api.generate_valid_configs(a, res, DIMS, CAPS)
        assert len(cfgs) == case["n_configs"] and len({(c.block_x, c.block_y) for c in cfgs}) == case["n_shapes"]
        preds = api.evaluate_configs(m, cfg, a, p, res, cfgs)
        rows = [_row_text(q) for q in preds]
        for i, want in case["sample"].items():
            assert rows[int(i)] == want, (case["kernel"], case["spec"], case["seq_len"], i)
        assert hashlib.sha256("\n".join(rows).encode()).hexdigest() == case["sha256"]
        ps = api.pareto_explore(m, cfg, a, p, res, DIMS, CAPS, rho=case["rho"])
        _check_front(case, ps.entries, ps.t_peak)


def test_sweep_gives_every_front_from_one_launch(backend):
    """f-4: all specs x all sequence lengths of one kernel in ONE grid launch + ONE skyline launch."""
    by_kernel = {}
    for c in _cases(backend) if backend == "emul" else [c for c in EXP["cases"] if "error" not in c]:
        by_kernel.setdefault((c["kernel"], c["source"], c["rule"]), []).append(c)
    for (kname, source, rule), cases in by_kernel.items():
        src, kern = _source(source)
        m = api.parse_ptx(src, kern)
        cfg = api.estimate_trip_counts(api.build_cfg(m), m)
        spec_names = sorted({c["spec"] for c in cases})
        seqs = sorted({c["seq_len"] for c in cases})
        pairs = [_spec(n) for n in spec_names]
        # resources are spec-independent for these workloads (the rule only reads max_shared for its overflow check)
        resources = [api.compute_input_resources(s, 4, 16, 64, 4, pairs[0][0], rule=rule) for s in seqs]
        rt = native.get_runtime()
        before = rt.launches()
        fronts = api.pareto_explore_sweep(m, cfg, pairs, resources, DIMS, CAPS, rho=0.95)
        assert rt.launches() - before == 3            # prepare + grid + skyline
        for c in cases:
            ps = fronts[(spec_names.index(c["spec"]), seqs.index(c["seq_len"]))]
            _check_front(c, ps.entries, ps.t_peak)


def test_resource_rule_errors_match_reference(backend):
    for c in EXP["cases"]:
        if "error" not in c:
            continue
        a, _ = _spec(c["spec"])
        with pytest.raises(getattr(E, c["error"])):
            api.compute_input_resources(c["seq_len"], 4, 16, 64, 4, a, rule=c["rule"])
