"""bench.py's CPU legs and the extra workloads BASELINE.json names besides the headline one.

CPU legs: the reference's own implementation (oracle/_ref/ptxwatt, the unmodified package copied
there by __graft_entry__.build() while /root/reference exists; `kind: "reference"`) on all host
cores, one process per core; the oracle port (`kind: "port"`) only when that copy is absent.
Both are CHECKERS / baselines: nothing here is on the product path.

Workloads (bench.py --workload ...):
  front1e9        BASELINE configs[4]: Pareto front of 10^9 (e, t) candidates, sharded by index range over the ranks,
                  local fronts merged with one all-gather (dist.sharded_skyline);
  front1e9_3obj   the same with the occupancy objective (extension, "parity unpinned");
  grid_c3         BASELINE configs[2]: 256 kernels x 4 specs x blockDim x/y/z x regs x smem x caps ~ 10^8 points scored;
  c1_latency      BASELINE configs[0]: one tiled-matmul PTX file through the drop-in API
                  (parse_ptx -> build_cfg -> estimate_trip_counts -> pareto_explore), latency per session.
"""
from __future__ import annotations

import json
import os
import sys
import time
from pathlib import Path
from types import SimpleNamespace

import numpy as np

ROOT = Path(__file__).resolve().parent
REF_DIR = ROOT / "oracle" / "_ref"
DIMS = list(range(1, 1025))
CAPS = [100.0, 125.0, 150.0, 175.0, 200.0, 225.0, 250.0]
RHO = 0.95


def cpu_kind() -> str:
    return "reference" if (REF_DIR / "ptxwatt" / "__init__.py").exists() else "port"


def _import_reference():
    if str(REF_DIR) not in sys.path:
        sys.path.insert(0, str(REF_DIR))
    import ptxwatt  # noqa: F401  (the unmodified reference package)
    return ptxwatt


def _import_oracle():
    if str(ROOT / "oracle") not in sys.path:
        sys.path.insert(0, str(ROOT / "oracle"))
    import flipflop_oracle
    return flipflop_oracle


# --------------------------------------------------------------------------- full analysis of kernels (headline workload)
def _analysis_worker(args):
    """One process: the whole path for a list of kernels - lex/classify, CFG + trips, features, 464 shapes x 7 caps
    scored, front at rho.  Returns (points, bytes, [front as [(bx, by, cap)]])."""
    kind, srcs, blocks = args
    fronts, points, nbytes = [], 0, 0
    if kind == "reference":
        ref = _import_reference()
        from ptxwatt import explorer as rex
        a, p = ref.default_architecture(), ref.default_calibration()
        for src, tb in zip(srcs, blocks):
            m = ref.parse_ptx(src)
            cfg = ref.estimate_trip_counts(ref.build_cfg(m), m)
            res = ref.InputResources(shared_mem_bytes=0, grid_x=int(tb))
            points += len(rex.generate_valid_configs(a, res, DIMS, CAPS))
            ps = ref.pareto_explore(m, cfg, a, p, res, DIMS, CAPS, rho=RHO)
            fronts.append([(e.config.block_x, e.config.block_y, e.config.p_cap) for e in ps.entries])
            nbytes += len(src)
    else:
        orc = _import_oracle()
        from paper_2601_13345_b200 import specs
        a, p = specs.default_architecture(), specs.default_calibration()
        ad, cd = orc.arch_dict(a), orc.cal_dict(p)
        cfgs = orc.enumerate_configs(ad, 0, DIMS, None)
        shp = np.array([(bx, by) for bx, by, _ in cfgs], dtype=np.int32)
        order = np.lexsort((shp[:, 1], shp[:, 0]))
        rank_of = np.empty(len(shp), dtype=np.int64)
        rank_of[order] = np.arange(len(shp))
        caps = np.asarray(CAPS)
        tie = (rank_of[:, None] * caps.size + np.arange(caps.size)[None, :]).reshape(-1).astype(np.int32)
        for src, tb in zip(srcs, blocks):
            row = np.zeros((1, 18))
            row[0, :11] = orc.kernel_feature_row(src)
            t, e = orc.score_grid_numpy(row, np.array([[0, int(tb)]], dtype=np.int64), ad, cd, shp, caps)
            idx, _ = orc.pareto_indices(e[0].reshape(-1), t[0].reshape(-1), tie=tie, rho=RHO)
            fronts.append([(int(shp[i // caps.size, 0]), int(shp[i // caps.size, 1]), float(caps[i % caps.size])) for i in idx])
            points += shp.shape[0] * caps.size
            nbytes += len(src)
    return points, nbytes, fronts


def cpu_analysis(srcs, blocks, workers: int):
    """Times the CPU implementation of the full path on `srcs` (text) with all `workers` processes.
    Returns dict(points, bytes, seconds, fronts, kind)."""
    import multiprocessing as mp
    kind = cpu_kind()
    workers = max(1, min(workers, len(srcs)))
    parts = [list(range(i, len(srcs), workers)) for i in range(workers)]
    jobs = [(kind, [srcs[j] for j in part], [blocks[j] for j in part]) for part in parts]
    with mp.get_context("fork").Pool(workers) as pool:
        pool.map(_noop, range(workers))                       # processes are up before the clock starts
        t0 = time.perf_counter()
        res = pool.map(_analysis_worker, jobs)
        dt = time.perf_counter() - t0
    fronts = [None] * len(srcs)
    for part, (_, _, fr) in zip(parts, res):
        for j, f in zip(part, fr):
            fronts[j] = f
    return {"points": sum(r[0] for r in res), "bytes": sum(r[1] for r in res), "seconds": dt, "fronts": fronts,
            "kind": kind, "workers": workers}


def _noop(_):
    return 0


# The reference re-derives the dynamic counts for every config (features.py:62-81 inside extract_features), so one
# pareto_explore over 3248 configs costs it about 30 ms per statement of the kernel: 35 s for the corpus' average kernel
# (1150 statements), 150 s for the largest.  To keep a step within seconds the CPU sample takes ONE kernel per process
# from the kernels of at most 20 KB (about 600 statements); that flatters the CPU (its configs/s fall with kernel size).
SAMPLE_MAX_BYTES = 20_000
SAMPLE_NOTE = "one kernel per process, drawn from the kernels of <= 20 KB - the reference's cost per config grows with kernel size, so this flatters it"


def cpu_sample_kernels(offs, workers: int, step: int):
    sizes = np.diff(np.asarray(offs, dtype=np.int64))
    small = np.flatnonzero(sizes <= SAMPLE_MAX_BYTES)
    if small.size == 0:
        small = np.argsort(sizes)[: max(workers, 1)]
    start = (step * workers * 7) % small.size
    return [int(small[(start + 7 * j) % small.size]) for j in range(min(workers, small.size))]


# --------------------------------------------------------------------------- front of a candidate cloud (CPU)
def _front_worker(args):
    kind, seed, n, three = args
    rng = np.random.default_rng(seed)
    e, t = rng.uniform(0.0, 10.0, n), rng.uniform(0.0, 10.0, n)
    occ = rng.integers(1, 9, n).astype(np.float64) / 8.0
    if kind == "reference" and not three:
        ref = _import_reference()
        from ptxwatt import explorer as rex
        # explorer.pareto_front reads .e_pred, .time.t_exec and .config.{block_x, block_y, p_cap} only; the stand-in
        # objects are built outside the clock
        preds = [SimpleNamespace(e_pred=float(e[i]), time=SimpleNamespace(t_exec=float(t[i])),
                                 config=SimpleNamespace(block_x=i, block_y=1, p_cap=100.0)) for i in range(n)]
        t0 = time.perf_counter()
        front = rex.pareto_front(preds)
        return n, time.perf_counter() - t0, len(front)
    orc = _import_oracle()
    t0 = time.perf_counter()
    idx = orc.pareto_indices3(e, t, occ)[0] if three else orc.pareto_indices(e, t)[0]
    return n, time.perf_counter() - t0, len(idx)


def cpu_front(n_per_worker: int, workers: int, three: bool):
    import multiprocessing as mp
    kind = "port" if three else cpu_kind()          # the reference has no 3-objective rule
    with mp.get_context("fork").Pool(workers) as pool:
        res = pool.map(_front_worker, [(kind, 100 + w, n_per_worker, three) for w in range(workers)])
    secs = max(r[1] for r in res)
    return {"candidates": sum(r[0] for r in res), "seconds": secs, "kind": kind, "workers": workers}


# --------------------------------------------------------------------------- shared bits of the GPU legs
def _peak():
    try:
        peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        return float(peaks["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback 6.65 TB/s"


def _dist_env():
    return int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")), int(os.environ.get("LOCAL_RANK", "0"))


def _max_over_ranks(ms, world, dev):
    if world == 1:
        return ms
    import torch
    import torch.distributed as dist
    tms = torch.tensor([ms], dtype=torch.float64, device=dev)
    dist.all_reduce(tms, op=dist.ReduceOp.MAX)
    return float(tms.item())


def _timed(fn, steps, warmup, world, dev):
    """W untimed + K timed calls, barrier + synchronize on both sides, CUDA events, max over ranks. Returns ms total."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    return _max_over_ranks(e0.elapsed_time(e1), world, dev)


def _base_line(args, metric, unit, value, ms_total, world, workload, config, clocks, launches, higher=True):
    return {"metric": metric, "value": value, "unit": unit, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms_total / args.steps, "higher_is_better": higher, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": {"workload": workload, **config}, "clocks": clocks,
            "gpu_launches": launches}


# --------------------------------------------------------------------------- front1e9 / front1e9_3obj
def run_front(args, three: bool, ClockSampler):
    import torch
    import torch.distributed as dist
    from paper_2601_13345_b200 import dist as fdist, engine, native
    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rt = native.get_runtime(local)
    dev = rt.device
    n_total = int(args.candidates)
    lo, hi = fdist.shard_range(n_total, rank, world)            # strong split of ONE candidate set (configs[4]) ...
    if args.weak_front:                                         # ... or 10^9 per GPU (weak) on request
        lo, hi = rank * n_total, (rank + 1) * n_total
    n = hi - lo
    g = torch.Generator(device=dev).manual_seed(5 + rank)
    e = torch.empty(n, dtype=torch.float64, device=dev)
    t = torch.empty(n, dtype=torch.float64, device=dev)
    occ = torch.empty(n, dtype=torch.float64, device=dev) if three else None
    piece = 1 << 27
    for a0 in range(0, n, piece):
        b0 = min(n, a0 + piece)
        e[a0:b0] = torch.rand(b0 - a0, generator=g, dtype=torch.float64, device=dev) * 10.0
        t[a0:b0] = torch.rand(b0 - a0, generator=g, dtype=torch.float64, device=dev) * 10.0
        if three:
            occ[a0:b0] = torch.randint(1, 9, (b0 - a0,), generator=g, device=dev).to(torch.float64) / 8.0
    cap = 1 << 16
    state = {}

    def step():
        state["front"] = fdist.sharded_skyline(e, t, lo, rho=0.0, cap_front=cap, rt=rt, occ=occ)

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    l0 = rt.launches()
    ms = _timed(step, args.steps, args.warmup, world, dev)
    launches = (rt.launches() - l0) * args.steps // (args.steps + args.warmup)
    clocks = sampler.stop() if rank == 0 else None
    ids, fe, ft, tpk = state["front"]
    # every rank holds the same merged front (byte-compared through a checksum all-reduce)
    chk = torch.stack([ids.to(torch.float64).sum(), fe.sum(), ft.sum(), torch.tensor(float(ids.numel()), device=dev, dtype=torch.float64)])
    if world > 1:
        mx, mn = chk.clone(), chk.clone()
        dist.all_reduce(mx, op=dist.ReduceOp.MAX)
        dist.all_reduce(mn, op=dist.ReduceOp.MIN)
        assert torch.equal(mx, mn), "ranks disagree on the merged front"
    # e2e: candidates in pinned host memory -> front on the host; the upload runs in 2^26-candidate chunks on a copy
    # stream, every chunk is reduced to its front while the next one uploads, the chunk fronts are merged at the end
    chunk = 1 << 26
    e2e_n = min(n, int(args.e2e_candidates))
    h_e = torch.empty(e2e_n, dtype=torch.float64).pin_memory()
    h_t = torch.empty(e2e_n, dtype=torch.float64).pin_memory()
    h_e.copy_(e[:e2e_n]); h_t.copy_(t[:e2e_n])
    h_o = None
    if three:
        h_o = torch.empty(e2e_n, dtype=torch.float64).pin_memory()
        h_o.copy_(occ[:e2e_n])
    copy_stream = torch.cuda.Stream(device=dev)
    bufs = [[torch.empty(chunk, dtype=torch.float64, device=dev) for _ in range(3 if three else 2)] for _ in range(2)]
    evs = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    host_front = {}

    def e2e_step():
        main = torch.cuda.current_stream(dev)
        parts = []
        n_chunks = (e2e_n + chunk - 1) // chunk
        for c in range(n_chunks):
            a0, b0 = c * chunk, min(e2e_n, (c + 1) * chunk)
            bset = bufs[c & 1]
            with torch.cuda.stream(copy_stream):
                if c >= 2:
                    copy_stream.wait_event(done[c & 1])       # the chunk that used this buffer has been reduced
                bset[0][: b0 - a0].copy_(h_e[a0:b0], non_blocking=True)
                bset[1][: b0 - a0].copy_(h_t[a0:b0], non_blocking=True)
                if three:
                    bset[2][: b0 - a0].copy_(h_o[a0:b0], non_blocking=True)
                evs[c & 1].record(copy_stream)
            main.wait_event(evs[c & 1])
            cid = torch.arange(lo + a0, lo + b0, dtype=torch.int64, device=dev)
            fid, fe_, ft_, _ = engine.skyline(bset[0][: b0 - a0], bset[1][: b0 - a0], ids=cid, rho=0.0, cap_front=cap, rt=rt,
                                              occ=bset[2][: b0 - a0] if three else None)
            done[c & 1].record(main)
            parts.append((fid, fe_, ft_, (bset[2][fid - (lo + a0)] if three else None)))
        ids_ = torch.cat([p_[0] for p_ in parts]); fe_ = torch.cat([p_[1] for p_ in parts]); ft_ = torch.cat([p_[2] for p_ in parts])
        fo_ = torch.cat([p_[3] for p_ in parts]).contiguous() if three else None
        lid, le, lt, _ = engine.skyline(fe_.contiguous(), ft_.contiguous(), ids=ids_.contiguous(), rho=0.0, cap_front=cap, rt=rt, occ=fo_)
        locc = None
        if three:                                             # occupancy of the surviving members, from the chunk fronts
            pos = torch.searchsorted(ids_sorted := torch.sort(ids_)[0], lid)
            locc = fo_[torch.sort(ids_)[1][pos]].contiguous()
        res = fdist.merge_fronts(lid, le, lt, rho=0.0, cap_front=cap, rt=rt, occ=locc)
        host_front["ids"] = res[0].cpu()                      # device -> host read of the result (synchronises)

    e2e_steps = max(2, args.steps // 3)
    ms_e2e = _timed(e2e_step, e2e_steps, 1, world, dev)
    if e2e_n == n:
        assert torch.equal(host_front["ids"], ids.cpu()), "streamed e2e front differs from the resident one"
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    total = n * world if args.weak_front else n_total
    peak, peak_src = _peak()
    per_step_ms = ms / args.steps
    bytes_per = 24.0 if three else 16.0
    achieved = bytes_per * n / (per_step_ms / 1e3) / 1e9
    out = _base_line(args, "pareto_candidates_per_sec", "candidates/s", total / (per_step_ms / 1e3), ms, world,
                     f"BASELINE configs[4]: Pareto front of {total:.3g} uniform (e, t{', occupancy' if three else ''}) candidates, "
                     f"{n} per GPU, local fronts merged with one all-gather + final skyline pass",
                     {"candidates_per_gpu": n, "objectives": 3 if three else 2, "front_size": int(ids.numel()),
                      "l2": "inputs (>= 16 GB per GPU) far above the 126 MB L2"}, clocks, launches)
    out["scaling"] = "weak" if args.weak_front else "strong"
    out["roofline"] = {"bound": "hbm", "kernel": "skyline (ffb_skyline, hierarchical chunk fronts)", "achieved": achieved, "peak": peak,
                       "unit": "GB/s", "frac": achieved / peak, "traffic": None, "peak_source": peak_src,
                       "algorithmic_bytes": f"{int(bytes_per)} B read per candidate"}
    out["e2e"] = {"value": (e2e_n * world) / (ms_e2e / e2e_steps / 1e3), "unit": "candidates/s",
                  "h2d_bytes_per_step": int(bytes_per) * e2e_n * world, "d2h_bytes_per_step": int(host_front["ids"].numel()) * 8 * world,
                  "ms_per_step": ms_e2e / e2e_steps, "steps": e2e_steps, "candidates_per_gpu": e2e_n,
                  "pipeline": "2^26-candidate chunks: upload on a copy stream, chunk front on the compute stream, chunk fronts merged at the end"}
    if not args.no_cpu_baseline:
        workers = os.cpu_count() or 1
        # the three-objective definition in the oracle is the O(n^2) scan: a small set per process
        c = cpu_front(40_000 if three else (200_000 if cpu_kind() == "reference" else 2_000_000), workers, three)
        out["cpu_baseline"] = {"value": c["candidates"] / c["seconds"], "unit": "candidates/s", "cores": c["workers"], "kind": c["kind"],
                               "sample": f"{c['candidates']} uniform candidates, one independent set of {c['candidates'] // c['workers']} per process "
                                         f"({'explorer.pareto_front of the reference' if c['kind'] == 'reference' else ('oracle O(n^2) definition' if three else 'oracle sort-sweep')}), {c['seconds']:.1f} s"}
    else:
        out["cpu_baseline"] = None
    if world > 1:
        dist.destroy_process_group()
    return out


# --------------------------------------------------------------------------- grid_c3
def run_grid_c3(args, ClockSampler):
    import dataclasses
    import torch
    import torch.distributed as dist
    from paper_2601_13345_b200 import engine, native, specs, synth
    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rt = native.get_runtime(local)
    dev = rt.device
    a, p = specs.default_architecture(), specs.default_calibration()
    sp_list = [(dataclasses.replace(a, name=f"spec{i}", sm_count=a.sm_count + 16 * i, f_base=a.f_base * (1.0 + 0.1 * i),
                                    bw_max=a.bw_max * (1.0 + 0.15 * i)) if i else a, p, 65536) for i in range(4)]
    sp = engine.spec_rows(sp_list)
    pow2 = [2 ** i for i in range(11)]
    shapes = [(bx, by, bz, regs) for bx in pow2 for by in pow2 for bz in (1, 2, 4) for regs in (16, 32, 64, 128, 255)]
    shp = engine.shape_rows(shapes)
    caps = np.linspace(a.p_cap_min, a.p_tdp, 11)
    feat_np, res_np = synth.feature_rows(seed=3 + rank, n_kernels=256)
    smem = np.array([0, 1024, 4096, 16384, 49152], dtype=np.int64)
    feat5 = np.repeat(feat_np, smem.size, axis=0)                      # the smem axis rides on the kernel rows (d_res)
    res5 = np.repeat(res_np, smem.size, axis=0)
    res5[:, 0] = np.tile(smem, 256)
    K, S, J, C = feat5.shape[0], sp.shape[0], shp.shape[0], caps.size
    points = K * S * J * C
    h_feat, h_res = torch.from_numpy(feat5).pin_memory(), torch.from_numpy(res5).pin_memory()
    d_feat, d_res = h_feat.to(dev), h_res.to(dev)
    bufs = {"t": torch.empty((K, S, J, C), dtype=torch.float64, device=dev), "e": torch.empty((K, S, J, C), dtype=torch.float64, device=dev)}
    fn_h = torch.empty((K * S,), dtype=torch.int32).pin_memory()

    def step():
        engine.score_grid(d_feat, d_res, sp, shp, caps, want=("t", "e"), out=bufs, check=False, rt=rt)

    def e2e_step():
        f, r_ = h_feat.to(dev, non_blocking=True), h_res.to(dev, non_blocking=True)
        r = engine.score_grid(f, r_, sp, shp, caps, want=("t", "e"), out=bufs, check=False, rt=rt)
        _, fn, _ = engine.skyline_groups(r.e.view(-1), r.t.view(-1), K * S, J * C, rho=RHO, rt=rt)[:3]
        fn_h.copy_(fn, non_blocking=True)                              # the result a caller reads: one front size per (kernel, spec)
        torch.cuda.current_stream(dev).synchronize()

    sampler = ClockSampler(local)
    if rank == 0:
        sampler.start()
    l0 = rt.launches()
    ms = _timed(step, args.steps, args.warmup, world, dev)
    launches = (rt.launches() - l0) * args.steps // (args.steps + args.warmup)
    clocks = sampler.stop() if rank == 0 else None
    e2e_steps = max(2, args.steps // 2)
    ms_e2e = _timed(e2e_step, e2e_steps, 1, world, dev)
    valid = int(torch.isfinite(bufs["t"]).sum().item())
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return None
    peak, peak_src = _peak()
    per = ms / args.steps
    achieved = 16.0 * points / (per / 1e3) / 1e9
    out = _base_line(args, "configs_scored_per_sec", "configs/s", points * world / (per / 1e3), ms, world,
                     f"BASELINE configs[2]: per GPU 256 kernels x {smem.size} dynamic-smem sizes x {S} specs x {J} block shapes "
                     f"(blockDim x, y in 2^0..2^10, z in 1/2/4, regs in 16..255) x {C} caps = {points} grid points scored (t_exec, e_pred)",
                     {"points_per_gpu": points, "valid_points_per_gpu": valid, "kernels": 256, "specs": S, "shapes": J, "caps": C,
                      "l2": "each step writes 1.6 GB, far above the 126 MB L2"}, clocks, launches)
    out["roofline"] = {"bound": "hbm", "kernel": "predict_grid_kernel", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                       "traffic": None, "peak_source": peak_src, "algorithmic_bytes": "16 B written per grid point (t_exec, e_pred f64)"}
    out["e2e"] = {"value": points * world / (ms_e2e / e2e_steps / 1e3), "unit": "configs/s",
                  "h2d_bytes_per_step": int(h_feat.numel() * 8 + h_res.numel() * 8) * world, "d2h_bytes_per_step": int(fn_h.numel() * 4) * world,
                  "ms_per_step": ms_e2e / e2e_steps, "steps": e2e_steps, "result": "one front per (kernel, spec) group, sizes read back"}
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_grid(feat5, res5, sp_list, shp, caps)
    else:
        out["cpu_baseline"] = None
    if world > 1:
        dist.destroy_process_group()
    return out


def _grid_worker(args):
    feat, res, ad, cd, shp, caps, rps = args
    orc = _import_oracle()
    t0 = time.perf_counter()
    orc.score_grid_numpy(feat, res, ad, cd, shp, caps, regs_per_sm=rps)
    return feat.shape[0] * shp.shape[0] * caps.size, time.perf_counter() - t0


def _cpu_grid(feat5, res5, sp_list, shp, caps):
    """The reference has no block_z / register axes: the oracle's vectorised definition (numpy) is the CPU baseline."""
    import multiprocessing as mp
    orc = _import_oracle()
    workers = os.cpu_count() or 1
    a, p, rps = sp_list[0]
    rows = min(feat5.shape[0], 8 * workers)
    jobs = [(feat5[i::workers][: rows // workers + 1], res5[i::workers][: rows // workers + 1], orc.arch_dict(a), orc.cal_dict(p), shp, caps, rps)
            for i in range(workers)]
    with mp.get_context("fork").Pool(workers) as pool:
        pool.map(_noop, range(workers))
        t0 = time.perf_counter()
        res = pool.map(_grid_worker, jobs)
        dt = time.perf_counter() - t0
    pts = sum(r[0] for r in res)
    return {"value": pts / dt, "unit": "configs/s", "cores": workers, "kind": "port",
            "sample": f"oracle score_grid_numpy (extension axes have no reference implementation) on {pts} points of spec 0, {workers} processes, {dt:.1f} s"}


# --------------------------------------------------------------------------- c1_latency
def _c1_source():
    parse = json.loads((ROOT / "tests" / "golden" / "ref_parse.json").read_text())
    key = "nvcc_sm_100a_tiled_matmul"
    return parse[key]["source"], parse[key]["kernel"]


def run_c1_latency(args, ClockSampler):
    import torch
    from paper_2601_13345_b200 import api, native
    rank, world, local = _dist_env()
    if rank != 0:
        return None                                      # one file, one session: replicas only
    torch.cuda.set_device(local)
    rt = native.get_runtime(local)
    src, kern = _c1_source()
    a, p = api.default_architecture(), api.default_calibration()
    res = api.compute_input_resources(128, 4, 16, 64, 4, a, rule="generic")

    def session():
        m = api.parse_ptx(src, kern)
        cfg = api.estimate_trip_counts(api.build_cfg(m), m)
        return api.pareto_explore(m, cfg, a, p, res, DIMS, CAPS, rho=RHO)

    for _ in range(args.warmup):
        ps = session()
    torch.cuda.synchronize()
    sampler = ClockSampler(local)
    sampler.start()
    l0 = rt.launches()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        ps = session()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    clocks = sampler.stop()
    launches = rt.launches() - l0
    ms = dt * 1e3 / args.steps
    n_cfg = len(api.generate_valid_configs(a, res, DIMS, CAPS))
    out = _base_line(args, "analysis_latency_ms", "ms", ms, dt * 1e3, 1,
                     f"BASELINE configs[0]: one nvcc tiled-matmul PTX file ({len(src)} bytes) through the drop-in API "
                     f"(parse_ptx, build_cfg, estimate_trip_counts, pareto_explore over {n_cfg} configs), one session per step, host wall clock",
                     {"configs": n_cfg, "front_size": len(ps.entries), "l2": "latency workload: KB-sized inputs, nothing to flush"},
                     clocks, launches, higher=False)
    out["scaling"] = "replicas only"
    out["roofline"] = {"bound": "hbm", "kernel": "launch-latency bound (KB-sized inputs; about %d launches + host object construction per session)" % (launches // max(args.steps, 1)),
                       "achieved": len(src) / (ms / 1e3) / 1e9, "peak": _peak()[0], "unit": "GB/s", "frac": len(src) / (ms / 1e3) / 1e9 / _peak()[0],
                       "traffic": None, "peak_source": _peak()[1], "algorithmic_bytes": "1 B per PTX byte + 16 B per config"}
    out["e2e"] = {"value": ms, "unit": "ms", "h2d_bytes_per_step": len(src) + 4096, "d2h_bytes_per_step": n_cfg * 16,
                  "note": "the session above IS the end-to-end call: host string in, ParetoSet of frozen dataclasses out"}
    if not args.no_cpu_baseline:
        out["cpu_baseline"] = _cpu_c1(src, kern, max(3, args.steps // 3))
        if out["cpu_baseline"].get("front") is not None:
            mine = [(e.config.block_x, e.config.block_y, e.config.p_cap) for e in ps.entries]
            assert mine == out["cpu_baseline"].pop("front"), "GPU front differs from the CPU implementation's"
            out["cpu_baseline"]["front_identical"] = True
    else:
        out["cpu_baseline"] = None
    return out


def _cpu_c1(src, kern, reps):
    kind = cpu_kind()
    if kind == "reference":
        ref = _import_reference()
        a, p = ref.default_architecture(), ref.default_calibration()
        res = ref.compute_input_resources(128, 4, 16, 64, 4, a, rule="generic")
        t0 = time.perf_counter()
        for _ in range(reps):
            m = ref.parse_ptx(src, kern)
            cfg = ref.estimate_trip_counts(ref.build_cfg(m), m)
            ps = ref.pareto_explore(m, cfg, a, p, res, DIMS, CAPS, rho=RHO)
        dt = time.perf_counter() - t0
        front = [(e.config.block_x, e.config.block_y, e.config.p_cap) for e in ps.entries]
        return {"value": dt * 1e3 / reps, "unit": "ms", "cores": 1, "kind": kind, "front": front,
                "sample": f"{reps} sessions of the reference's own parse_ptx .. pareto_explore on the same file (single-threaded, as the reference runs it)"}
    r = cpu_analysis([src], [64], 1)
    return {"value": r["seconds"] * 1e3, "unit": "ms", "cores": 1, "kind": kind, "front": None, "sample": "oracle port, one session"}


# --------------------------------------------------------------------------- reference arms of the extra workloads
def reference_arm_extra(args):
    rank, world, _ = _dist_env()
    if rank != 0:
        return None
    workers = os.cpu_count() or 1
    wl = args.workload
    if wl in ("front1e9", "front1e9_3obj"):
        three = wl.endswith("3obj")
        n_per = 30_000 if three else (100_000 if cpu_kind() == "reference" else 1_000_000)
        tot_c, tot_s = 0, 0.0
        for i in range(args.warmup + args.steps):
            c = cpu_front(n_per, workers, three)
            if i >= args.warmup:
                tot_c += c["candidates"]; tot_s += c["seconds"]
        value, unit, metric = tot_c / tot_s, "candidates/s", "pareto_candidates_per_sec"
        sample = f"{n_per} uniform candidates per process, {workers} processes, per step"
        kind = c["kind"]
        workload = f"BASELINE configs[4] on the host cores, bounded sample per step: {sample}"
        higher = True
    elif wl == "c1_latency":
        src, kern = _c1_source()
        c = _cpu_c1(src, kern, args.warmup + args.steps)
        value, unit, metric, kind, sample = c["value"], "ms", "analysis_latency_ms", c["kind"], c["sample"]
        workload = "BASELINE configs[0] on the host: " + sample
        workers, higher = 1, False
        tot_s = value * args.steps / 1e3
    elif wl == "grid_c3":
        import dataclasses
        from paper_2601_13345_b200 import engine, specs, synth
        a, p = specs.default_architecture(), specs.default_calibration()
        pow2 = [2 ** i for i in range(11)]
        shp = engine.shape_rows([(bx, by, bz, regs) for bx in pow2 for by in pow2 for bz in (1, 2, 4) for regs in (16, 32, 64, 128, 255)])
        caps = np.linspace(a.p_cap_min, a.p_tdp, 11)
        feat_np, res_np = synth.feature_rows(seed=3, n_kernels=256)
        tot_p, tot_s = 0, 0.0
        for i in range(args.warmup + args.steps):
            c = _cpu_grid(feat_np, res_np, [(a, p, 65536)], shp, caps)
            if i >= args.warmup:
                tot_p += 1; tot_s += 1.0 / c["value"]
        value, unit, metric, kind, sample = tot_p / tot_s, "configs/s", "configs_scored_per_sec", c["kind"], c["sample"]
        workload = "BASELINE configs[2] on the host cores, bounded sample per step: " + sample
        higher = True
        tot_s = args.steps * 1.0
    else:
        raise SystemExit(f"--impl reference has no arm for workload {wl}")
    return {"impl": "reference", "metric": metric, "value": value, "unit": unit, "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": tot_s / max(args.steps, 1) * 1e3, "higher_is_better": higher, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": {"workload": workload},
            "cpu_baseline": {"value": value, "unit": unit, "cores": workers, "kind": kind, "sample": sample},
            "e2e": {"value": value, "unit": unit, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
