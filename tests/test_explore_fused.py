"""K2 + K3 + K4 fused (ffb_explore_groups) against (a) the two-call route ffb_predict_grid ->
ffb_skyline_groups and (b) the oracle: same fronts, same order, same t_peak, bit-identical (e, t)."""
from __future__ import annotations

import json
from pathlib import Path

import numpy as np
import pytest
import torch

import flipflop_oracle as orc
from paper_2601_13345_b200 import engine, errors, native, specs, synth

G_DIR = Path(__file__).parent / "golden"


def _tie(shapes, n_caps, caps):
    J = len(shapes)
    order = sorted(range(J), key=lambda j: (tuple(int(v) for v in shapes[j]), j))
    rank = np.empty(J, dtype=np.int64)
    rank[order] = np.arange(J)
    corder = sorted(range(n_caps), key=lambda c: (float(caps[c]), c))
    crank = np.empty(n_caps, dtype=np.int64)
    crank[corder] = np.arange(n_caps)
    return (rank[:, None] * n_caps + crank[None, :]).reshape(-1).astype(np.int32)


def _alt():
    model = json.loads((G_DIR / "ref_model.json").read_text())
    return specs.architecture_from_dict(model["alt_spec"]["arch"]), specs.calibration_from_dict(model["alt_spec"]["calibration"])


@pytest.mark.parametrize("case", ["pow2", "all_dims", "unsorted_caps_zregs", "one_cap", "no_floor"])
def test_fused_equals_two_call_route_and_oracle(backend, case):
    a, p = specs.default_architecture(), specs.default_calibration()
    pairs = [(a, p), _alt()]
    sp = engine.spec_rows(pairs)
    K = 3 if backend == "emul" else 96
    rho = 0.95
    caps = np.array([100.0, 125.0, 150.0, 175.0, 200.0, 225.0, 250.0])
    if case == "pow2":
        shapes = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[1], 0, [2 ** i for i in range(11)])])
    elif case == "all_dims":
        dims = list(range(1, 1025)) if backend != "emul" else [1, 2, 3, 4, 6, 8, 12, 16, 24, 32, 48, 64, 96, 128, 256, 512, 1024]
        shapes = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[1], 0, dims)])
    elif case == "unsorted_caps_zregs":
        caps = np.array([250.0, 90.0, 180.0, 120.0, 300.0, 150.0, 150.0])          # unsorted, a duplicate, out-of-range values
        shapes = np.array([(bx, by, bz, rg) for bx in (1, 4, 16, 32, 64, 256) for by in (1, 2, 8, 32) for bz in (1, 2, 4)
                           for rg in (32, 128)], dtype=np.int32)
        sp = engine.spec_rows([(a, p, 65536), (*_alt(), 131072)])
    elif case == "one_cap":
        caps = np.array([200.0])
        shapes = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, [1, 2, 4, 8, 16, 32, 64, 128, 256, 512])])
    else:
        rho = 0.0
        shapes = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, [1, 2, 4, 8, 16, 32, 64, 128])])
    feat, res = synth.feature_rows(seed=17, n_kernels=K)
    res[:, 0] = np.array([0, 0, 2048, 70000, 0, 16384])[np.arange(K) % 6]           # incl. one above the default SM's shared memory
    S, J, C = sp.shape[0], shapes.shape[0], caps.size
    G = J * C
    d_feat, d_res = engine.features_tensor(feat), engine.resources_tensor(res)
    rt = native.get_runtime()
    fi, fn, tp, fe, ft = engine.explore_groups(d_feat, d_res, sp, shapes, caps, rho=rho, want_values=True)
    r = engine.score_grid(d_feat, d_res, sp, shapes, caps, want=("t", "e"))
    tie = _tie(shapes, C, caps)
    gi, gn, gtp = engine.skyline_groups(r.e.view(-1), r.t.view(-1), K * S, G, tie=rt.to_device(torch.from_numpy(tie)), rho=rho)
    assert torch.equal(fn, gn)
    assert torch.equal(tp.view(torch.int64), gtp.view(torch.int64))
    fi_h, gi_h, fn_h = fi.cpu().numpy(), gi.cpu().numpy(), fn.cpu().numpy()
    e_h, t_h = r.e.cpu().numpy().reshape(K * S, G), r.t.cpu().numpy().reshape(K * S, G)
    fe_h, ft_h = fe.cpu().numpy(), ft.cpu().numpy()
    for g in range(K * S):
        n = int(fn_h[g])
        assert np.array_equal(fi_h[g, :n], gi_h[g, :n]), (case, g)
        assert np.array_equal(fe_h[g, :n].view(np.uint64), e_h[g][fi_h[g, :n]].view(np.uint64))
        assert np.array_equal(ft_h[g, :n].view(np.uint64), t_h[g][fi_h[g, :n]].view(np.uint64))
    # oracle on a sample of groups (the grid itself is oracle-checked in test_grid_parity / test_extension_axes)
    for g in list(range(0, K * S, max(1, (K * S) // 12)))[:12]:
        want, wtp = orc.pareto_indices(e_h[g], t_h[g], tie=tie, rho=rho)
        assert fi_h[g, : int(fn_h[g])].tolist() == want
        assert (np.isinf(wtp) and np.isinf(float(tp[g]))) or float(tp[g]) == wtp
    # compact layout holds the same runs
    ci, cn, ctp, coff = engine.explore_groups(d_feat, d_res, sp, shapes, caps, rho=rho, compact=True, cap_front=int(fn_h.sum()) + 8)
    ci_h, coff_h = ci.cpu().numpy(), coff.cpu().numpy()
    assert torch.equal(cn, fn)
    for g in range(K * S):
        n = int(fn_h[g])
        assert np.array_equal(ci_h[coff_h[g]: coff_h[g] + n], fi_h[g, :n])
    order = np.lexsort((fn_h, coff_h))                                # runs tile the buffer without gaps or overlap
    assert np.array_equal(coff_h[order], np.concatenate([[0], np.cumsum(fn_h[order])[:-1]]))


def test_fused_heavy_ties(backend):
    """Every candidate of a group can carry the same (e, t) - e.g. a kernel without instructions, where nothing
    depends on the shape except eta: all ties stay on the front, in (bx, by, cap) order."""
    a, p = specs.default_architecture(), specs.default_calibration()
    sp = engine.spec_rows([(a, p)])
    feat, res = synth.feature_rows(seed=1, n_kernels=2)
    feat[0, :] = 0.0
    feat[0, native.F_ALIGNED] = 1.0
    feat[0, native.F_OVR_TEXEC] = np.nan
    shapes = engine.shape_rows([tuple(x) for x in engine.enumerate_shapes(sp[0], 0, [32, 64, 128, 256, 512, 1024, 1, 2, 4, 8])])
    caps = np.array([150.0, 200.0])
    d_feat, d_res = engine.features_tensor(feat), engine.resources_tensor(res)
    fi, fn, tp = engine.explore_groups(d_feat, d_res, sp, shapes, caps, rho=0.95)
    r = engine.score_grid(d_feat, d_res, sp, shapes, caps, want=("t", "e"))
    tie = _tie(shapes, caps.size, caps)
    for g in range(2):
        want, _ = orc.pareto_indices(r.e[g].cpu().numpy().reshape(-1), r.t[g].cpu().numpy().reshape(-1), tie=tie, rho=0.95)
        assert fi[g, : int(fn[g])].cpu().tolist() == want
    assert int(fn[0]) > shapes.shape[0] // 4          # the tie-heavy group keeps a large front


def test_fused_capacity_is_reported(backend):
    a, p = specs.default_architecture(), specs.default_calibration()
    sp = engine.spec_rows([(a, p)])
    feat, res = synth.feature_rows(seed=1, n_kernels=1)
    shapes = engine.shape_rows([(32, 1)] * 700)
    caps = np.linspace(100.0, 250.0, 50)                 # 35 000 candidates in one group
    with pytest.raises(errors.CapacityExceeded):
        engine.explore_groups(engine.features_tensor(feat), engine.resources_tensor(res), sp, shapes, caps)
    fi, fn, tp = engine.explore_groups(engine.features_tensor(feat), engine.resources_tensor(res), sp, shapes[:40], caps[:7])
    with pytest.raises(errors.CapacityExceeded):         # dense front buffer too small
        engine.explore_groups(engine.features_tensor(feat), engine.resources_tensor(res), sp, shapes[:40], caps[:7], cap_front=3)
