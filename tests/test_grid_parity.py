"""K2+K3 (ffb_predict_grid) against the oracle: bit-exact t_exec / e_pred / occupancy."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import flipflop_oracle as orc
from paper_2601_13345_b200 import engine, native, specs, synth


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def _alt_spec():
    a = specs.default_architecture()
    p = specs.default_calibration()
    from dataclasses import replace
    a2 = replace(a, name="alt-84sm", sm_count=84, max_warps_per_sm=64, max_shared_per_sm=102400, bw_max=936e9,
                 p_tdp=350.0, p_static=55.0, p_cap_min=120.0, dvfs_exponent_k=2, tau_short=5e-6, f_base=1.7e9)
    p2 = replace(p, l_mem_coal=350.0, l_mem_uncoal=900.0, sm_power_beta=0.81, kappa=0.2, t_base=1e-6,
                 time_weights=(0.9, 1.1, 1.0), transient_ratio_r=0.9)
    return a2, p2


@pytest.mark.parametrize("axes", ["xy", "xyz_regs"])
def test_streaming_grid_with_factored_model_equals_the_full_chain(backend, axes):
    """t / e only (no flags, no status: the streaming configuration) takes the kernel that evaluates the group's
    (threads, regs) and clipped-block_x class rows once and two divides per shape; every bit must equal the
    per-shape chain of the general kernel, which the test above pins to the oracle.  Odd J x C sizes exercise
    both write-out forms."""
    K = 5 if backend == "emul" else 300
    feat, res = synth.feature_rows(seed=17, n_kernels=K)
    pairs = [(specs.default_architecture(), specs.default_calibration(), 65536 if axes == "xyz_regs" else 0), _alt_spec()]
    sp = engine.spec_rows(pairs)
    if axes == "xy":
        shp = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, list(range(1, 1025)))][: (121 if backend == "emul" else 464)])
    else:
        pw = [1, 2, 4, 8, 16, 32, 64, 128]
        shp = engine.shape_rows([(bx, by, bz, rg) for bx in pw for by in pw for bz in (1, 2, 3) for rg in (16, 64, 255)][: (275 if backend == "emul" else 10**6)])
    caps = np.array([100.0, 125.0, 150.0, 200.0, 249.0, 250.0, 400.0])
    d_feat, d_res = engine.features_tensor(feat), engine.resources_tensor(res)
    full = engine.score_grid(d_feat, d_res, sp, shp, caps, want=("t", "e", "flags"))
    lean = engine.score_grid(d_feat, d_res, sp, shp, caps, want=("t", "e"), check=False)
    assert np.array_equal(_bits(full.t.cpu().numpy()), _bits(lean.t.cpu().numpy()))
    assert np.array_equal(_bits(full.e.cpu().numpy()), _bits(lean.e.cpu().numpy()))
    assert np.isfinite(lean.t.cpu().numpy()).any() and np.isinf(lean.t.cpu().numpy()).any()


@pytest.mark.parametrize("case", ["default", "two_specs"])
def test_grid_matches_oracle_bitwise(backend, case):
    K = 6 if backend == "emul" else 64
    feat, res = synth.feature_rows(seed=7, n_kernels=K)
    pairs = [(specs.default_architecture(), specs.default_calibration())]
    if case == "two_specs":
        pairs.append(_alt_spec())
    sp = engine.spec_rows(pairs)
    dims = [1, 2, 3, 4, 8, 16, 32, 64, 96, 128, 256, 512, 1024]
    caps = np.array([90.0, 100.0, 125.0, 150.0, 175.0, 200.0, 225.0, 250.0, 300.0, 400.0])
    # shape axis: union over specs of shapes valid for shared_dyn = 0 (validity is masked per point)
    shp = engine.enumerate_shapes(sp[-1], 0, dims)
    r = engine.score_grid(engine.features_tensor(feat), engine.resources_tensor(res), sp,
                          engine.shape_rows([tuple(x) for x in shp]), caps, want=("t", "e", "flags", "occ"))
    t, e, fl, occ = (x.cpu().numpy() for x in (r.t, r.e, r.flags, r.occ))
    for s, (a, p) in enumerate(pairs):
        ad, cd = orc.arch_dict(a), orc.cal_dict(p)
        for k in range(K):
            want_valid = {(bx, by, c) for bx, by, c in orc.enumerate_configs(ad, int(res[k, 0]), dims, caps.tolist())}
            f = dict(zip(("n_mem", "mem_bytes", "FP32", "INT", "SFU", "ALU", "n_sync", "aligned", "static_shared"),
                         feat[k, :9]))
            for j, (bx, by) in enumerate(shp):
                for c, cap in enumerate(caps):
                    valid = (int(bx), int(by), float(cap)) in want_valid
                    assert bool(fl[k, s, j, c] & native.PT_VALID) == valid
                    if not valid:
                        assert np.isinf(t[k, s, j, c]) and np.isinf(e[k, s, j, c])
                        continue
                    w = orc.score_point(f, ad, cd, int(bx), int(by), float(cap), int(res[k, 0]), int(res[k, 1]))
                    assert _bits(t[k, s, j, c]) == _bits(w["t_exec"])
                    assert _bits(e[k, s, j, c]) == _bits(w["e_pred"])
                    assert bool(fl[k, s, j, c] & native.PT_CAP_LIMITED) == w["cap_limited"]
                    assert _bits(occ[k, s, j]) == _bits(w["blocks_per_sm"])


def test_grid_matches_vectorised_oracle_large(backend):
    """Bigger slice through the numpy oracle (same IEEE ops, vectorised)."""
    K = 16 if backend == "emul" else 2048
    feat, res = synth.feature_rows(seed=11, n_kernels=K)
    a, p = specs.default_architecture(), specs.default_calibration()
    sp = engine.spec_rows([(a, p)])
    dims = [2 ** i for i in range(11)]
    caps = np.array([100.0, 125.0, 150.0, 175.0, 200.0, 225.0, 250.0])
    shp = engine.enumerate_shapes(sp[0], 0, dims)
    r = engine.score_grid(engine.features_tensor(feat), engine.resources_tensor(res), sp,
                          engine.shape_rows([tuple(x) for x in shp]), caps, want=("t", "e", "flags"))
    wt, we = orc.score_grid_numpy(feat, res, orc.arch_dict(a), orc.cal_dict(p), shp, caps)
    valid = (r.flags.cpu().numpy()[:, 0] & 1).astype(bool)
    # dynamic shared above the SM limit invalidates the whole kernel (explorer.py:85-88)
    assert np.array_equal(valid.all(axis=(1, 2)), res[:, 0] <= a.max_shared_per_sm)
    got_t, got_e = r.t.cpu().numpy()[:, 0], r.e.cpu().numpy()[:, 0]
    assert np.array_equal(_bits(got_t[valid]), _bits(wt[valid]))
    assert np.array_equal(_bits(got_e[valid]), _bits(we[valid]))
    assert np.isinf(got_t[~valid]).all()


def test_detail_rows_and_strict_errors(backend):
    from paper_2601_13345_b200.errors import InvalidConfig, EmptyGrid
    a, p = specs.default_architecture(), specs.default_calibration()
    sp = engine.spec_rows([(a, p)])
    feat, res = synth.feature_rows(seed=3, n_kernels=2)
    shp = engine.shape_rows([(32, 4), (16, 8)])
    r = engine.score_grid(engine.features_tensor(feat), engine.resources_tensor(res), sp, shp,
                          np.array([150.0, 250.0]), want=("detail", "e", "t"), strict=True)
    d = r.detail.cpu().numpy()
    assert np.array_equal(_bits(d[..., native.D_T_EXEC]), _bits(r.t.cpu().numpy()))
    assert np.array_equal(_bits(d[..., native.D_E_PRED]), _bits(r.e.cpu().numpy()))
    assert (d[..., native.D_WARPS] == 4.0).all()
    with pytest.raises(InvalidConfig):
        engine.score_grid(engine.features_tensor(feat), engine.resources_tensor(res), sp,
                          engine.shape_rows([(5, 5)]), np.array([150.0]), strict=True)
    res0 = res.copy()
    res0[:, 1] = 0
    with pytest.raises(EmptyGrid):
        engine.score_grid(engine.features_tensor(feat), engine.resources_tensor(res0), sp, shp,
                          np.array([150.0]), strict=True)


def test_lean_streaming_path_matches_checked_path(backend):
    """check=False + (t, e) only selects the lean kernel variant (vector stores, no status)."""
    K = 5 if backend == "emul" else 1500
    feat, res = synth.feature_rows(seed=21, n_kernels=K)
    sp = engine.spec_rows([(specs.default_architecture(), specs.default_calibration()), _alt_spec()])
    shp = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, [1, 2, 4, 8, 16, 32, 64, 128, 256, 512, 1024])])
    for caps in (np.array([100.0, 150.0, 200.0, 250.0, 275.0]), np.array([125.0, 225.0])):
        f, r_ = engine.features_tensor(feat), engine.resources_tensor(res)
        full = engine.score_grid(f, r_, sp, shp, caps, want=("t", "e", "flags"))
        lean = engine.score_grid(f, r_, sp, shp, caps, want=("t", "e"), check=False)
        assert torch.equal(full.t.view(torch.int64), lean.t.view(torch.int64))
        assert torch.equal(full.e.view(torch.int64), lean.e.view(torch.int64))
