"""Host-side multi-rank logic on CPU: world_size-2 gloo, emulated kernels on each rank."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _worker(rank: int, world: int, port: int, kind: str, rho: float, out_dir: str):
    for p in (ROOT, ROOT / "tests" / "simt", ROOT / "oracle"):
        sys.path.insert(0, str(p))
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from build_emul import build_emul
    from paper_2601_13345_b200 import dist as ffd, native, synth
    rt = native.Runtime(native.bind(build_emul()), torch.device("cpu"))
    native.install_runtime_for_tests(rt)
    n = 6000
    three = kind.endswith("+occ")
    e, t = synth.candidate_cloud(seed=5, n=n, kind=kind.replace("+occ", ""))
    occ = (np.random.default_rng(6).integers(1, 6, n) / 5.0) if three else None
    lo, hi = ffd.shard_range(n, rank, world)
    ids, fe, ft, tp = ffd.sharded_skyline(torch.from_numpy(e[lo:hi].copy()), torch.from_numpy(t[lo:hi].copy()), lo,
                                          rho=rho, cap_front=2048,
                                          occ=torch.from_numpy(occ[lo:hi].copy()) if three else None)
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), ids=ids.numpy(), e=fe.numpy(), t=ft.numpy(), tp=tp)
    dist.destroy_process_group()


@pytest.mark.parametrize("kind,rho", [("uniform", 0.0), ("tied", 0.9), ("uniform+occ", 0.0)])
def test_sharded_front_equals_global_front(tmp_path, kind, rho):
    sys.path.insert(0, str(ROOT / "oracle"))
    import flipflop_oracle as orc
    from paper_2601_13345_b200 import synth
    from build_emul import build_emul
    build_emul()                      # compile once, before the ranks race for it
    port = 29500 + (os.getpid() % 500)
    mp.spawn(_worker, args=(2, port, kind, rho, str(tmp_path)), nprocs=2, join=True)
    e, t = synth.candidate_cloud(seed=5, n=6000, kind=kind.replace("+occ", ""))
    if kind.endswith("+occ"):
        occ = np.random.default_rng(6).integers(1, 6, 6000) / 5.0
        want, wtp = orc.pareto_indices3(e, t, occ, rho=rho)
    else:
        want, wtp = orc.pareto_indices(e, t, rho=rho)
    for r in range(2):
        got = np.load(tmp_path / f"r{r}.npz")
        assert got["ids"].tolist() == want
        assert np.array_equal(got["e"], e[want]) and np.array_equal(got["t"], t[want])
        assert float(got["tp"]) == wtp


def test_shard_helpers():
    from paper_2601_13345_b200 import dist as ffd
    for n in (0, 1, 7, 8, 1001):
        for w in (1, 2, 3, 8):
            spans = [ffd.shard_range(n, r, w) for r in range(w)]
            assert spans[0][0] == 0 and spans[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            assert max(b - a for a, b in spans) - min(b - a for a, b in spans) <= 1
    off = np.array([0, 10, 1000, 1010, 1020, 5000, 5001, 9000])
    for w in (1, 2, 3, 4, 8):
        spans = [ffd.shard_segments(off, r, w) for r in range(w)]
        assert spans[0][0] == 0 and spans[-1][1] == len(off) - 1
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
