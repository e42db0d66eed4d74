#!/usr/bin/env python
"""Generates the golden vectors under tests/golden/ by RUNNING THE REFERENCE
(/root/reference/pkg/src/ptxwatt, imported in place in the build container; it does not
exist on the GPU box, which is why its outputs are committed here).

    python tests/golden/make_golden.py

Outputs
  ref_fixtures.json   the reference's own 5 PTX fixtures (inputs, as test data) + its manifest.json
                      hand counts (pkg/tests/fixtures/manifest.json:1-75)
  ref_parse.json      reference outputs for: those fixtures, tests/edge_cases.py, seeded synthetic
                      kernels, nvcc-generated kernels (tiled matmul, conv2d, MHA): module fields,
                      CFG, trips, aligned fraction, dynamic counts, or the exception class
  ref_classify.json   classify_opcode / access_bytes over an opcode table (ptx.py:99-136, 64-76;
                      known-answer list of pkg/tests/test_ptx_parser.py:120-134 included)
  ref_model.json      generate_valid_configs, evaluate_configs (hex floats), pareto_explore for the
                      fixtures x several resource / spec settings; model helper known answers
                      (pkg/tests/test_power_model.py:52-126, test_time_model.py:15-54)
  ref_pareto.json     pareto_front / pareto_front_bruteforce on seeded random and tied clouds
                      (seeds 19, 202 as in pkg/tests/test_explorer.py:199, test_acceptance.py:109)
"""
from __future__ import annotations

import json
import math
import subprocess
import sys
import tempfile
from dataclasses import replace
from pathlib import Path

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
REF = Path("/root/reference/pkg")
sys.path.insert(0, str(REF / "src"))
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

import numpy as np  # noqa: E402
import ptxwatt as ref  # noqa: E402
from ptxwatt import explorer as rex, power_model as rpm, time_model as rtm  # noqa: E402
from ptxwatt.errors import PtxWattError  # noqa: E402
from ptxwatt.features import dynamic_instruction_counts  # noqa: E402
from ptxwatt.ptx import classify_opcode  # noqa: E402

from edge_cases import EDGE_CASES  # noqa: E402
from paper_2601_13345_b200 import synth  # noqa: E402

FIX = ("straight_line", "vecadd", "diamond", "counted_loop", "mha_like")
hx = float.hex

NVCC_KERNELS = r'''
#define T 16
extern "C" __global__ void tiled_matmul(const float* A, const float* B, float* C, int N) {
  __shared__ float As[T][T]; __shared__ float Bs[T][T];
  int row = blockIdx.y * T + threadIdx.y, col = blockIdx.x * T + threadIdx.x; float acc = 0.f;
  for (int t = 0; t < N / T; ++t) {
    As[threadIdx.y][threadIdx.x] = A[row * N + t * T + threadIdx.x];
    Bs[threadIdx.y][threadIdx.x] = B[(t * T + threadIdx.y) * N + col];
    __syncthreads();
    for (int k = 0; k < T; ++k) acc += As[threadIdx.y][k] * Bs[k][threadIdx.x];
    __syncthreads();
  }
  C[row * N + col] = acc;
}
extern "C" __global__ void conv2d_3x3(const float* in, const float* w, float* out, int H, int W) {
  int x = blockIdx.x * blockDim.x + threadIdx.x, y = blockIdx.y * blockDim.y + threadIdx.y;
  if (x < 1 || y < 1 || x >= W - 1 || y >= H - 1) return;
  float s = 0.f;
  for (int dy = -1; dy <= 1; ++dy) for (int dx = -1; dx <= 1; ++dx) s += in[(y + dy) * W + x + dx] * w[(dy + 1) * 3 + dx + 1];
  out[y * W + x] = s;
}
extern "C" __global__ void mha_scores(const float* q, const float* k, float* p, int L, int D) {
  extern __shared__ float row[];
  int h = blockIdx.x, i = blockIdx.y; const float* qi = q + (h * L + i) * D; float mx = -1e30f;
  for (int j = threadIdx.x; j < L; j += blockDim.x) {
    float s = 0.f; for (int d = 0; d < 64; ++d) s += qi[d] * k[(h * L + j) * D + d];
    row[j] = s; mx = fmaxf(mx, s);
  }
  __syncthreads();
  for (int j = threadIdx.x; j < L; j += blockDim.x) p[(h * L + i) * L + j] = __expf(row[j] - mx);
}
'''


def nvcc_ptx() -> dict[str, str]:
    out = {}
    with tempfile.TemporaryDirectory() as td:
        src = Path(td) / "k.cu"
        src.write_text(NVCC_KERNELS)
        for arch in ("sm_70", "sm_100a"):
            ptx = Path(td) / f"k_{arch}.ptx"
            subprocess.run(["nvcc", "-ptx", f"-arch={arch}", "-lineinfo", str(src), "-o", str(ptx)], check=True,
                           capture_output=True)
            text = ptx.read_text()
            for name in ("tiled_matmul", "conv2d_3x3", "mha_scores"):
                out[f"nvcc_{arch}_{name}"] = (text, name)
    return out


def describe(src: str, kernel=None, default_trip=32.0) -> dict:
    try:
        m = ref.parse_ptx(src, kernel)
    except PtxWattError as ex:
        return {"error": type(ex).__name__}
    cfg0 = ref.build_cfg(m)
    cfg = ref.estimate_trip_counts(cfg0, m, default_trip=default_trip)
    n_mem, mem_bytes, by_unit, n_sync = dynamic_instruction_counts(m, cfg)
    hist = [0] * 9
    for ins in m.instructions:
        hist[ref.ptx.OPCODE_CLASSES.index(ins.opcode_class)] += 1
    return {
        "kernel_name": m.kernel_name, "parameters": [list(p) for p in m.parameters],
        "registers_declared": m.registers_declared, "static_shared_bytes": m.static_shared_bytes,
        "instructions": [[i.opcode, i.opcode_class, i.state_space, list(i.operands), i.predicate, i.source_line]
                         for i in m.instructions],
        "labels": m.labels, "class_hist": hist,
        "blocks": [list(b) for b in cfg.blocks], "edges": [list(e) for e in cfg.edges],
        "loops": [[l.header, sorted(l.body), l.header_label, hx(l.trip)] for l in cfg.loops],
        "default_trip": default_trip,
        "aligned_fraction": hx(ref.analyze_memory_alignment(m, cfg)),
        "dynamic": {"n_mem": hx(n_mem), "mem_bytes": hx(mem_bytes), "n_sync": hx(n_sync),
                    **{u: hx(v) for u, v in by_unit.items()}},
    }


def main():
    fixtures = {n: (REF / "tests" / "fixtures" / f"{n}.ptx").read_text() for n in FIX}
    manifest = json.loads((REF / "tests" / "fixtures" / "manifest.json").read_text())
    (HERE / "ref_fixtures.json").write_text(json.dumps({"sources": fixtures, "manifest": manifest}, indent=1))

    cases = {}
    for n, src in fixtures.items():
        cases[f"fixture_{n}"] = {"source": src, "kernel": None, "expect": describe(src),
                                 "expect_trip5": describe(src, default_trip=5.0)}
    for n, src in EDGE_CASES.items():
        cases[f"edge_{n}"] = {"source": src, "kernel": None, "expect": describe(src)}
    text, offs = synth.ptx_corpus(seed=11, n_kernels=10, lo=20, hi=260)
    for i in range(10):
        src = text[offs[i]:offs[i + 1]].decode()
        cases[f"synth_{i}"] = {"source": src, "kernel": None, "expect": describe(src), "expect_trip5": describe(src, default_trip=5.0)}
    for n, (src, kern) in nvcc_ptx().items():
        cases[n] = {"source": src, "kernel": kern, "expect": describe(src, kern)}
    (HERE / "ref_parse.json").write_text(json.dumps(cases, indent=0))

    ops = sorted({i[0] for c in cases.values() if "instructions" in c["expect"] for i in c["expect"]["instructions"]} | {
        "bar.sync", "ld.global.f32", "ld.shared.v4.f32", "ld.param.u64", "st.global.v2.f64", "bra", "add.s32", "add.f32",
        "mul.wide.s32", "mad.lo.s32", "fma.rn.f32", "div.rn.f32", "ex2.approx.f32", "sqrt.approx.f32", "sqrt.rn.f32",
        "mov.u32", "setp.lt.s32", "cvta.to.global.u64", "shfl.sync.bfly.b32", "bar.arrive", "redux.sync.add.s32",
        "ld.const.f32", "ldu.global.f32", "brx.idx", "ret", "exit", "add.u16", "selp.f32", "cvt.rn.f32.s32", "ld.f32"})
    (HERE / "ref_classify.json").write_text(json.dumps(
        {op: [*classify_opcode(op), ref.Instruction(op, "Other", "none", (), None, 0).access_bytes] for op in ops}, indent=0))

    arch, prof = ref.default_architecture(), ref.default_calibration()
    arch2 = replace(arch, name="alt-84sm", sm_count=84, max_warps_per_sm=64, max_shared_per_sm=102400, bw_max=936e9,
                    p_tdp=350.0, p_static=55.0, p_cap_min=120.0, dvfs_exponent_k=2, tau_short=5e-6, f_base=1.7e9)
    prof2 = replace(prof, l_mem_coal=350.0, l_mem_uncoal=900.0, sm_power_beta=0.81, kappa=0.2, t_base=1e-6,
                    time_weights=(0.9, 1.1, 1.0), transient_ratio_r=0.9)
    model = {"cases": [], "alt_spec": {"arch": ref.calibration.architecture_to_dict(arch2),
                                       "calibration": ref.calibration.calibration_to_dict(prof2)}}
    dims = [1, 2, 3, 4, 8, 16, 32, 48, 128, 256, 1024]
    caps = [90.0, 100.0, 150.0, 200.0, 250.0, 300.0, 350.0]
    for n, src in fixtures.items():
        if n in ('straight_line', 'diamond'):
            continue
        m = ref.parse_ptx(src)
        cfg = ref.estimate_trip_counts(ref.build_cfg(m), m)
        for spec_name, (a, p) in {"default": (arch, prof), "alt": (arch2, prof2)}.items():
            for res in (ref.InputResources(0, 16, 4, 1), ref.InputResources(4096, 300, 40, 1)):
                cfgs = rex.generate_valid_configs(a, res, dims, caps)
                preds = rex.evaluate_configs(m, cfg, a, p, res, cfgs)
                fronts = {}
                for rho in (0.95, 1.0, 0.6):
                    ps = rex.pareto_explore(m, cfg, a, p, res, dims, caps, rho=rho)
                    fronts[str(rho)] = {"t_peak": hx(ps.t_peak),
                                        "entries": [[e.config.block_x, e.config.block_y, e.config.p_cap] for e in ps.entries]}
                model["cases"].append({
                    "fixture": n, "spec": spec_name, "resources": [res.shared_mem_bytes, res.grid_x, res.grid_y, res.grid_z],
                    "dims": dims, "caps": caps,
                    "configs": [[c.block_x, c.block_y, c.p_cap] for c in cfgs],
                    "pred": [[hx(p_.time.t_exec), hx(p_.power.p_dyn), hx(p_.e_pred), p_.power.cap_limited] for p_ in preds],
                    "detail": [[hx(p_.time.t_mem), hx(p_.time.t_comp), hx(p_.time.t_sync), hx(p_.time.mwp), hx(p_.time.cwp),
                                hx(p_.time.bw_eff), hx(p_.power.p_units), hx(p_.power.p_shape), hx(p_.power.p_mem),
                                hx(p_.power.p_sm), hx(p_.power.f_adj), hx(p_.power.ci), p_.power.active_sms] for p_ in preds[:24]],
                    "fronts": fronts})
    model["kats"] = {
        "shape_power(10,0.1,2,32,1)": hx(rpm.shape_power(10.0, 0.1, 2, 32, 1.0)),
        "shape_power(10,0.1,16,16,1)": hx(rpm.shape_power(10.0, 0.1, 16, 16, 1.0)),
        "sm_concurrency_power(16,2,0.8,30)": hx(rpm.sm_concurrency_power(16, 2.0, 0.8, 30.0)),
        "sm_concurrency_power(0,2,0.8,30)": hx(rpm.sm_concurrency_power(0, 2.0, 0.8, 30.0)),
        "dvfs_frequency(1,125,250,3)": hx(rpm.dvfs_frequency(1.0, 125.0, 250.0, 3)),
        "dvfs_frequency(1,100,250,3)": hx(rpm.dvfs_frequency(1.0, 100.0, 250.0, 3)),
        "memory_power(20,0.25,0.6)": hx(rpm.memory_power(20.0, 0.25, 0.6)),
        "transient_correction(100,5e-6,1e-5,0.833)": hx(rpm.transient_correction(100.0, 5e-6, 1e-5, 0.833)),
        "activity_rate(100,8,4,1)": hx(rpm.activity_rate(100.0, 8.0, 4.0, 1.0)),
        "mwp(400,40)": hx(rtm.mwp(400.0, 40.0)), "mwp(20,40)": hx(rtm.mwp(20.0, 40.0)),
        "cwp(300,100)": hx(rtm.cwp(300.0, 100.0)), "cwp(0,100)": hx(rtm.cwp(0.0, 100.0)),
    }
    (HERE / "ref_model.json").write_text(json.dumps(model, indent=0))

    def synth_pred(e, t, i):
        tb = ref.TimeBreakdown(1.0, 1.0, 1.0, 0.0, 0.0, 0.0, float(t))
        pb = ref.PowerBreakdown(0.0, 0.0, 0.0, 0.0, 0.0, 1.0, 0.0, 1, False)
        return ref.Prediction(ref.LaunchConfig(32 * (1 + i % 7), 1 + i // 7, 100.0 + (i % 3)), tb, pb, float(e))
    clouds = []
    rng = np.random.default_rng(19)
    for trial in range(40):
        n = int(rng.integers(1, 400))
        if trial % 2 == 0:
            e, t = rng.uniform(0, 10, n), rng.uniform(0, 10, n)
        else:
            e, t = rng.integers(0, 6, n).astype(float), rng.integers(0, 6, n).astype(float)
        preds = [synth_pred(e[i], t[i], i) for i in range(n)]
        front = rex.pareto_front(preds)
        brute = rex.pareto_front_bruteforce(preds)
        assert [id(p) for p in front] == [id(p) for p in brute.entries]
        idx = {id(p): i for i, p in enumerate(preds)}
        clouds.append({"e": [hx(float(x)) for x in e], "t": [hx(float(x)) for x in t],
                       "cfg": [[p.config.block_x, p.config.block_y, p.config.p_cap] for p in preds],
                       "front": [idx[id(p)] for p in front], "t_peak": hx(brute.t_peak)})
    (HERE / "ref_pareto.json").write_text(json.dumps(clouds, indent=0))
    # CLI reports of the reference (pkg/src/ptxwatt/cli.py) for byte-identity checks
    from ptxwatt import cli as rcli
    import contextlib, io
    cli_cases = []
    with tempfile.TemporaryDirectory() as td:
        for fx in ("vecadd", "mha_like"):
            ptx = Path(td) / f"{fx}.ptx"
            ptx.write_text(fixtures[fx])
            for argv in (["analyze", str(ptx), "--block-x", "64", "--block-y", "2", "--shared-mem-bytes", "1024"],
                         ["predict", str(ptx), "--block-x", "32", "--block-y", "4", "--p-cap", "180", "--seq-len", "256"],
                         ["explore", str(ptx), "--caps", "100,150,200,250", "--rho", "0.9"],
                         ["explore", str(ptx), "--dims", "1,2,4,8,16,32,64,128", "--format", "json", "--resource-rule", "generic"],
                         ["predict", str(ptx), "--block-x", "5", "--block-y", "5"],
                         ["explore", str(ptx), "--seq-len", "100000"]):
                out, err = io.StringIO(), io.StringIO()
                with contextlib.redirect_stdout(out), contextlib.redirect_stderr(err):
                    rc = rcli.main(list(argv))
                cli_cases.append({"fixture": fx, "argv": argv[:1] + ["@PTX@"] + argv[2:], "rc": rc,
                                  "stdout": out.getvalue(), "stderr": err.getvalue().replace(str(ptx), "@PTX@")})
    (HERE / "ref_cli.json").write_text(json.dumps(cli_cases, indent=0))
    print("golden vectors written:", sorted(p.name for p in HERE.glob("*.json")))


if __name__ == "__main__":
    main()
