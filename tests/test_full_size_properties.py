"""BASELINE.json's full sizes on one B200, checked through size-independent properties
(the oracle cannot run at these sizes): replica invariance and checksums for the corpus,
sampled oracle rows for the 10^8-point grid, dominance / idempotence / sortedness for the
10^9-candidate front.  GPU only; the whole file takes about a minute."""
from __future__ import annotations

import dataclasses

import numpy as np
import pytest
import torch

import flipflop_oracle as orc
from paper_2601_13345_b200 import corpus, engine, native, specs, synth

pytestmark = pytest.mark.gpu


def test_corpus_1_4_gb_replica_invariance(gpu_only):
    """configs[3] per-GPU share (1.44 GB, 38 400 kernels): the corpus is 32 tilings of 1 200 generated
    kernels, so every replica of a kernel (another address, another alignment against the 16-byte
    loads and the 4 KB tiles, other neighbours in the work queue) must give the same histogram,
    declarations and feature row; the first replica is checked against the oracle on a sample."""
    rt = gpu_only
    corp = corpus.bench_corpus(seed=4, target_bytes=0, n_kernels=38_400, rt=rt)
    assert corp.n_bytes > 1.4e9
    lex, fl = corpus.analyze_corpus(corp, rt=rt)
    torch.cuda.synchronize()
    K, base = corp.n_segs, 1200
    reps = K // base
    assert int((fl.status != 0).sum()) == 0
    assert lex.path_counts.cpu().tolist()[:2] == [K, 0]            # compiler-shaped text: all on the fast path
    hist = lex.hist.view(reps, base, -1)
    assert bool((hist == hist[0:1]).all())
    info = lex.info_i32().view(reps, base, 12)
    assert bool((info[:, :, :8] == info[0:1, :, :8]).all())        # status, counts, declarations (offsets differ per replica? no: relative)
    feat = fl.feat.view(reps, base, -1)[:, :, :11]
    assert bool((feat.view(torch.int64) == feat[0:1].view(torch.int64)).all())
    assert int(lex.hist.sum()) == int(lex.info_i32()[:, 1].sum())  # checksum: classes partition the instructions
    text, offs = corp.host_sample()
    for k in range(0, base, 97):
        src = text[offs[k]:offs[k + 1]].decode("ascii")
        want = np.asarray(orc.kernel_feature_row(src), dtype=np.float64)
        assert fl.feat[k, :11].cpu().numpy().tobytes() == want.tobytes()


def test_grid_1e8_points_sampled_against_oracle(gpu_only):
    """configs[2] folded into the axes the kernel has: 256 kernels x 18 spec rows x 464 shapes x 47 caps
    (the cap tile's capacity) = 1.005e8 grid points.  Every point of 20 sampled (kernel, spec) rows equals
    the oracle bit for bit; t_exec is monotone along the cap axis (a higher cap never lowers the DVFS
    frequency)."""
    rt = gpu_only
    a, p = specs.default_architecture(), specs.default_calibration()
    sp_rows = []
    n_specs = 18
    for i in range(n_specs):                             # modeled specs: the shipped one and scaled variants
        ai = a if i == 0 else dataclasses.replace(a, name=f"spec{i}", sm_count=a.sm_count + 12 * i,
                                                  f_base=a.f_base * (1.0 + 0.05 * i), bw_max=a.bw_max * (1.0 + 0.1 * i))
        sp_rows.append((ai, p))
    sp = engine.spec_rows(sp_rows)
    shp_xy = engine.enumerate_shapes(sp[0], 0, list(range(1, 1025)), rt=rt)
    shp = engine.shape_rows([tuple(x) for x in shp_xy])
    caps = np.linspace(a.p_cap_min, a.p_tdp, 47)
    feat_np, res_np = synth.feature_rows(seed=3, n_kernels=256)
    res_np[:, 0] = 0
    r = engine.score_grid(engine.features_tensor(feat_np, rt=rt), engine.resources_tensor(res_np, rt=rt), sp, shp, caps,
                          want=("t", "e"), check=False, rt=rt)
    torch.cuda.synchronize()
    assert r.t.numel() >= 1.0e8
    rng = np.random.default_rng(7)
    for k, s in zip(rng.integers(0, 256, 20), rng.integers(0, n_specs, 20)):
        ai = sp_rows[int(s)][0]
        wt, we = orc.score_grid_numpy(feat_np[k:k + 1], res_np[k:k + 1], orc.arch_dict(ai), orc.cal_dict(p), shp_xy, caps)
        gt, ge = r.t[k, s].cpu().numpy(), r.e[k, s].cpu().numpy()
        ok = np.isfinite(wt[0])
        assert np.array_equal(np.isfinite(gt), ok)
        assert np.array_equal(gt[ok].view(np.uint64), wt[0][ok].view(np.uint64))
        assert np.array_equal(ge[ok].view(np.uint64), we[0][ok].view(np.uint64))
    t = r.t.view(-1, caps.size)
    fin = torch.isfinite(t).all(dim=1)
    assert bool((t[fin][:, 1:] <= t[fin][:, :-1]).all())          # more power never makes a kernel slower


@pytest.mark.parametrize("kind", ["uniform", "anticorrelated"])
def test_front_of_1e9_candidates(gpu_only, kind):
    """configs[4], one GPU's worth done whole: 10^9 candidates (16 GB of e, t).  The front is sorted by
    (e, t), strictly decreasing in t along increasing e, no input point dominates a front point (sampled),
    the front of the front is the front, and every front id points at its own (e, t)."""
    rt = gpu_only
    n = 1_000_000_000
    g = torch.Generator(device=rt.device).manual_seed(5)
    e = torch.empty(n, dtype=torch.float64, device=rt.device)
    t = torch.empty(n, dtype=torch.float64, device=rt.device)
    step = 1 << 27
    for lo in range(0, n, step):                        # generated in pieces: torch.rand temporaries stay small
        hi = min(n, lo + step)
        e[lo:hi] = torch.rand(hi - lo, generator=g, dtype=torch.float64, device=rt.device) * 10.0
        if kind == "uniform":
            t[lo:hi] = torch.rand(hi - lo, generator=g, dtype=torch.float64, device=rt.device) * 10.0
        else:
            t[lo:hi] = 10.0 - e[lo:hi] + torch.randn(hi - lo, generator=g, dtype=torch.float64, device=rt.device) * 0.5
    cap = 1 << 16
    ids, fe, ft, tpk = engine.skyline(e, t, rho=0.0, cap_front=cap, rt=rt)
    torch.cuda.synchronize()
    m = ids.numel()
    assert 1 <= m < cap
    assert tpk == float(t.min())
    assert bool((e[ids] == fe).all()) and bool((t[ids] == ft).all())
    assert bool((fe[1:] >= fe[:-1]).all())
    strictly = fe[1:] > fe[:-1]
    assert bool((ft[1:][strictly] < ft[:-1][strictly]).all())      # lower t is the only reason to stay at a higher e
    # no candidate dominates a front member: for a sample of 2e6 inputs, look up the front's min t below their e
    idx = torch.randint(0, n, (2_000_000,), generator=g, device=rt.device)
    pos = torch.searchsorted(fe, e[idx], right=False)               # front members with e strictly below
    best_t_below = torch.where(pos > 0, ft[(pos - 1).clamp(min=0)], torch.full_like(ft[:1], float("inf")).expand(pos.shape))
    on_front_or_dominated = (t[idx] >= best_t_below) | (torch.isin(idx, ids))
    not_dominated = t[idx] < best_t_below
    # a sampled point that nothing on the front dominates must itself be on the front (ties aside)
    cand = idx[not_dominated]
    pe, pt = e[cand], t[cand]
    p2 = torch.searchsorted(fe, pe, right=False)
    hit = (p2 < m) & (fe[p2.clamp(max=m - 1)] == pe)
    assert bool(hit.all()) and bool(on_front_or_dominated.all())
    ids2, fe2, ft2, _ = engine.skyline(fe.contiguous(), ft.contiguous(), ids=ids.contiguous(), rho=0.0, cap_front=cap, rt=rt)
    assert torch.equal(ids2, ids) and torch.equal(fe2, fe) and torch.equal(ft2, ft)


def test_tied_front_of_1e9_candidates(gpu_only):
    """configs[4] with the clustered / tied distribution of pkg/tests/test_acceptance.py:114-115 at 10^9: every
    candidate with the lowest e or the lowest t is on the front (5% of the set, all exact ties), far beyond what
    one CTA can sort - the streaming pre-filter leaves exactly those, the device-wide sort orders them."""
    rt = gpu_only
    n = 1_000_000_000
    g = torch.Generator(device=rt.device).manual_seed(11)
    e = torch.empty(n, dtype=torch.float64, device=rt.device)
    t = torch.empty(n, dtype=torch.float64, device=rt.device)
    step = 1 << 27
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        e[lo:hi] = torch.randint(0, 40, (hi - lo,), generator=g, device=rt.device).to(torch.float64) / 4.0
        t[lo:hi] = torch.randint(0, 40, (hi - lo,), generator=g, device=rt.device).to(torch.float64) / 4.0
    on_front = (e == 0.0) | (t == 0.0)
    m = int(on_front.sum().item())
    assert m > 40_000_000
    ids, fe, ft, tpk = engine.skyline(e, t, rho=0.0, cap_front=m + 16, rt=rt)
    torch.cuda.synchronize()
    assert ids.numel() == m and tpk == 0.0
    assert bool(on_front[ids].all())
    assert bool((e[ids] == fe).all()) and bool((t[ids] == ft).all())
    # reference order: (e, t, id) ascending
    same_e = fe[1:] == fe[:-1]
    assert bool((fe[1:] >= fe[:-1]).all())
    assert bool((ft[1:][same_e] >= ft[:-1][same_e]).all())
    same_et = same_e & (ft[1:] == ft[:-1])
    assert bool((ids[1:][same_et] > ids[:-1][same_et]).all())


def test_three_objective_front_of_1e9_candidates(gpu_only):
    """configs[4], "+occupancy" (extension): 10^9 candidates with 8 occupancy levels.  The 2-objective front is
    a subset of the 3-objective one (3-objective dominance implies 2-objective dominance), no front member is
    dominated by another front member, and the front of the front is the front."""
    rt = gpu_only
    n = 1_000_000_000
    g = torch.Generator(device=rt.device).manual_seed(9)
    e = torch.empty(n, dtype=torch.float64, device=rt.device)
    t = torch.empty(n, dtype=torch.float64, device=rt.device)
    occ = torch.empty(n, dtype=torch.float64, device=rt.device)
    step = 1 << 27
    for lo in range(0, n, step):
        hi = min(n, lo + step)
        e[lo:hi] = torch.rand(hi - lo, generator=g, dtype=torch.float64, device=rt.device) * 10.0
        t[lo:hi] = torch.rand(hi - lo, generator=g, dtype=torch.float64, device=rt.device) * 10.0
        occ[lo:hi] = torch.randint(1, 9, (hi - lo,), generator=g, device=rt.device).to(torch.float64) / 8.0
    cap = 1 << 16
    ids3, fe3, ft3, _ = engine.skyline(e, t, occ=occ, rho=0.0, cap_front=cap, rt=rt)
    ids2, fe2, ft2, _ = engine.skyline(e, t, rho=0.0, cap_front=cap, rt=rt)
    torch.cuda.synchronize()
    assert 1 <= ids2.numel() <= ids3.numel() < cap
    assert bool(torch.isin(ids2, ids3).all())
    fo3 = occ[ids3]
    dom = (fe3[None, :] < fe3[:, None]) & (ft3[None, :] < ft3[:, None]) & (fo3[None, :] >= fo3[:, None])
    assert not bool(dom.any())
    again, *_ = engine.skyline(fe3.contiguous(), ft3.contiguous(), occ=fo3.contiguous(), ids=ids3.contiguous(), rho=0.0, cap_front=cap, rt=rt)
    assert torch.equal(again, ids3)
