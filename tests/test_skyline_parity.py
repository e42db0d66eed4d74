"""K4 (ffb_skyline_groups / ffb_skyline) against the oracle: membership AND order exact."""
from __future__ import annotations

import numpy as np
import pytest
import torch

import flipflop_oracle as orc
from paper_2601_13345_b200 import engine, native, synth
from paper_2601_13345_b200.errors import CapacityExceeded


def _dev(x):
    rt = native.get_runtime()
    return rt.to_device(torch.from_numpy(np.ascontiguousarray(x)))


@pytest.mark.parametrize("kind", ["uniform", "tied", "anticorrelated"])
@pytest.mark.parametrize("rho", [0.95, 1.0, 0.0])
def test_groups_match_oracle(backend, kind, rho):
    ng, G = (3, 300) if backend == "emul" else (64, 3248)
    e, t = synth.candidate_cloud(seed=202, n=ng * G, kind=kind)
    if kind == "anticorrelated" and backend != "emul":
        t = 10.0 - e + np.random.default_rng(1).normal(0.0, 2.0, e.size)   # keep the front below the survivor cap
    fi, fn, tp = engine.skyline_groups(_dev(e), _dev(t), ng, G, rho=rho)
    fi, fn, tp = fi.cpu().numpy(), fn.cpu().numpy(), tp.cpu().numpy()
    for g in range(ng):
        want, wtp = orc.pareto_indices(e[g * G:(g + 1) * G], t[g * G:(g + 1) * G], rho=rho)
        assert fi[g, :fn[g]].tolist() == want
        assert tp[g] == wtp


def test_ties_all_survive_and_bruteforce_agrees(backend):
    rng = np.random.default_rng(19)
    for _ in range(4):
        n = int(rng.integers(1, 400))
        e = rng.integers(0, 5, n).astype(np.float64)
        t = rng.integers(0, 5, n).astype(np.float64)
        fi, fn, _ = engine.skyline_groups(_dev(e), _dev(t), 1, n, rho=0.0)
        got = fi.cpu().numpy()[0, :int(fn[0])].tolist()
        assert set(got) == orc.pareto_bruteforce(e, t)
        key = [(e[i], t[i], i) for i in got]
        assert key == sorted(key)


def test_tie_key_orders_equal_points(backend):
    e = np.array([1.0, 1.0, 1.0, 2.0])
    t = np.array([3.0, 3.0, 3.0, 1.0])
    tie = torch.tensor([2, 0, 1, 0], dtype=torch.int32)
    fi, fn, _ = engine.skyline_groups(_dev(e), _dev(t), 1, 4, tie=native.get_runtime().to_device(tie), rho=0.0)
    assert fi.cpu().numpy()[0, :int(fn[0])].tolist() == [1, 2, 0, 3]


def test_invalid_points_never_on_front(backend):
    e = np.array([np.inf, 1.0, np.inf, 0.5])
    t = np.array([np.inf, 2.0, np.inf, 3.0])
    fi, fn, tp = engine.skyline_groups(_dev(e), _dev(t), 1, 4, rho=0.0)
    assert fi.cpu().numpy()[0, :int(fn[0])].tolist() == [3, 1] and tp[0].item() == 2.0
    fi, fn, tp = engine.skyline_groups(_dev(np.full(4, np.inf)), _dev(np.full(4, np.inf)), 1, 4, rho=0.95)
    assert int(fn[0]) == 0 and np.isinf(tp[0].item())


def test_front_capacity_is_reported(backend):
    n = 64
    e = np.arange(n, dtype=np.float64)
    t = e[::-1].copy()
    with pytest.raises(CapacityExceeded):
        engine.skyline_groups(_dev(e), _dev(t), 1, n, rho=0.0, cap_front=8)


@pytest.mark.parametrize("kind", ["uniform", "tied"])
def test_large_set_hierarchical(backend, kind):
    n = 30_000 if backend == "emul" else (5_000_000 if kind == "uniform" else 100_000)
    e, t = synth.candidate_cloud(seed=5, n=n, kind=kind)
    cap = 1 << 13
    ids, fe, ft, tpk = engine.skyline(_dev(e), _dev(t), rho=0.0, cap_front=cap)
    want, wtp = orc.pareto_indices(e, t, rho=0.0)
    assert ids.cpu().numpy().tolist() == want
    assert np.array_equal(fe.cpu().numpy(), e[want]) and np.array_equal(ft.cpu().numpy(), t[want])
    assert tpk == wtp
    # idempotence: the front of the front is the front
    ids2, *_ = engine.skyline(fe.contiguous(), ft.contiguous(), ids=ids.contiguous(), rho=0.0, cap_front=cap)
    assert ids2.cpu().numpy().tolist() == want


@pytest.mark.parametrize("kind", ["uniform", "tied", "anticorrelated", "specials", "constant_e"])
def test_streaming_prefilter_keeps_the_front(backend, kind, monkeypatch):
    """Sets of 2^20 candidates and more first go through the two-pass bucket pre-filter of ffb_skyline; the
    threshold is lowered here so that the CPU suite covers it too: same front, same order, same t_peak,
    with ties, NaNs, infinities and a degenerate e range."""
    monkeypatch.setenv("FFB_SKYLINE_PREFILTER_MIN", "1000")
    n = 20_000 if backend == "emul" else 3_000_000
    if kind == "specials":
        e, t = synth.candidate_cloud(seed=8, n=n, kind="uniform")
        rng = np.random.default_rng(8)
        e[rng.integers(0, n, 50)] = np.inf
        t[rng.integers(0, n, 50)] = np.inf
        e[rng.integers(0, n, 20)] = -1e300                          # far below the sampled range
        e[:3] = 1e300
    elif kind == "constant_e":
        e, t = np.full(n, 2.5), np.random.default_rng(3).integers(0, 50, n).astype(np.float64)
    else:
        e, t = synth.candidate_cloud(seed=6, n=n, kind=kind)
    rho = 0.9 if kind == "uniform" else 0.0
    want, wtp = orc.pareto_indices(e, t, rho=rho)
    ids, fe, ft, tpk = engine.skyline(_dev(e), _dev(t), rho=rho, cap_front=max(1 << 15, len(want) + 8))
    assert ids.cpu().numpy().tolist() == want
    assert np.array_equal(fe.cpu().numpy(), e[want]) and np.array_equal(ft.cpu().numpy(), t[want])
    assert tpk == wtp


@pytest.mark.parametrize("kind", ["all_on_front", "tied", "tied_floor"])
def test_front_larger_than_one_cta(backend, kind):
    """Fronts that hold a constant fraction of the set (ties, anti-correlated clouds) are finished by the
    device-wide sort of ffb_bigfront.cu: membership, reference order (e, t, id) and t_peak as the oracle."""
    n = 30_000 if backend == "emul" else 2_000_000
    rng = np.random.default_rng(12)
    if kind == "all_on_front":
        e = np.arange(n, dtype=np.float64) // 3                      # triples of equal e ...
        t = (n - np.arange(n, dtype=np.float64)) // 3 + rng.integers(0, 2, n)      # ... t falls as e grows: nearly all stay
    else:
        e, t = synth.candidate_cloud(seed=13, n=n, kind="tied")     # pkg/tests/test_acceptance.py:114-115 distribution
    rho = 0.5 if kind == "tied_floor" else 0.0
    want, wtp = orc.pareto_indices(e, t, rho=rho)
    assert len(want) > (65535 if backend == "gpu" and rho == 0.0 else (8192 if kind == "all_on_front" else 500))
    ids, fe, ft, tpk = engine.skyline(_dev(e), _dev(t), rho=rho, cap_front=len(want) + 5)
    assert ids.cpu().numpy().tolist() == want
    assert np.array_equal(fe.cpu().numpy(), e[want]) and np.array_equal(ft.cpu().numpy(), t[want])
    assert tpk == wtp
    with pytest.raises(CapacityExceeded):
        engine.skyline(_dev(e), _dev(t), rho=rho, cap_front=len(want) - 1)


@pytest.mark.parametrize("levels,rho", [(1, 0.0), (4, 0.0), (9, 0.9), (64, 0.0)])
def test_three_objective_groups_match_oracle(backend, levels, rho):
    """Extension (occupancy as a third objective): groups against the O(n^2) definition in the oracle;
    one occupancy level reduces to the two-objective front."""
    rng = np.random.default_rng(100 + levels)
    n_groups, G = (4, 300) if backend == "emul" else (40, 3248)
    e = np.round(rng.uniform(0.0, 10.0, n_groups * G), 1)            # rounded: plenty of ties in e and t
    t = np.round(rng.uniform(1.0, 10.0, n_groups * G), 1)
    occ = rng.integers(0, levels, n_groups * G).astype(np.float64) / max(levels, 1)
    tie = rng.permutation(G).astype(np.int32)
    fi, fn, tp = engine.skyline_groups(_dev(e), _dev(t), n_groups, G, tie=_dev(tie), rho=rho, occ=_dev(occ))
    fi, fn = fi.cpu().numpy(), fn.cpu().numpy()
    for g in range(n_groups):
        sl = slice(g * G, (g + 1) * G)
        want, wtp = orc.pareto_indices3(e[sl], t[sl], occ[sl], tie=tie, rho=rho)
        assert fi[g, : int(fn[g])].tolist() == want, (g, levels)
        assert float(tp[g]) == wtp
        if levels == 1:
            assert want == orc.pareto_indices(e[sl], t[sl], tie=tie, rho=rho)[0]


@pytest.mark.parametrize("prefilter", [False, True])
def test_three_objective_large_set_and_capacity(backend, prefilter, monkeypatch):
    # with the pre-filter: one table column per distinct occupancy value (8 here), also with the rho floor below
    monkeypatch.setenv("FFB_SKYLINE_PREFILTER_MIN", "1000" if prefilter else str(1 << 40))
    n = 20_000 if backend == "emul" else 2_000_000
    rng = np.random.default_rng(77)
    e, t = rng.uniform(0.0, 10.0, n), rng.uniform(0.0, 10.0, n)
    occ = rng.integers(1, 9, n).astype(np.float64) / 8.0
    ids, fe, ft, tpk = engine.skyline(_dev(e), _dev(t), occ=_dev(occ), rho=0.0, cap_front=1 << 14)
    want, wtp = [], float(t.min())
    # reference answer without the O(n^2) scan over everything: a 3-objective front member is a
    # 2-objective front member of the points whose occupancy is at least its own
    cand = set()
    for lv in np.unique(occ):
        sub = np.nonzero(occ >= lv)[0]
        cand.update(int(sub[i]) for i in orc.pareto_indices(e[sub], t[sub], rho=0.0)[0])
    cand = np.asarray(sorted(cand))
    keep = [int(i) for i in cand if not np.any((e[cand] < e[i]) & (t[cand] < t[i]) & (occ[cand] >= occ[i]))]
    keep = np.asarray(keep)
    want = keep[np.lexsort((keep, t[keep], e[keep]))].tolist()
    assert ids.cpu().numpy().tolist() == want and tpk == wtp
    with pytest.raises(CapacityExceeded):                  # more than 64 occupancy levels in one group
        engine.skyline_groups(_dev(e[:4096].copy()), _dev(t[:4096].copy()), 1, 4096, rho=0.0, occ=_dev(rng.uniform(0, 1, 4096)))
