"""Multi-GPU sharding of the analysis path (one process per GPU, torch.distributed).

What shards how:
  * corpus lexing / dataflow, grid scoring, per-kernel fronts: kernels are independent units;
    every rank takes a contiguous run of kernels — NO data-path collective;
  * one large candidate set sharded by index range (BASELINE config 5): every rank reduces its
    shard to a local front, the fixed-capacity front buffers are exchanged with ONE all-gather
    (NCCL over NVLink on GPUs), and every rank runs the final skyline pass on the gathered
    buffer in place.  Exact because strict dominance is transitive (a globally dominated point
    is dominated by a global-front member, and global-front members survive their local pass)
    and because the throughput floor commutes with the front (explorer.py:137,209-211: a
    dominator has strictly smaller t, so it is itself eligible); the global min-t point is never
    dominated, hence t_peak can be read off the merged front.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from . import engine, native


def shard_range(n: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous [start, stop) of n units for this rank; sizes differ by at most one."""
    base, extra = divmod(n, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_segments(seg_off: np.ndarray, rank: int, world: int) -> tuple[int, int]:
    """Contiguous run of corpus segments with about 1/world of the BYTES (kernels differ in size)."""
    seg_off = np.asarray(seg_off, dtype=np.int64)
    total = int(seg_off[-1] - seg_off[0])
    cuts = [int(np.searchsorted(seg_off, seg_off[0] + total * r // world, side="left")) for r in range(world + 1)]
    cuts[0], cuts[-1] = 0, len(seg_off) - 1
    for r in range(1, world + 1):
        cuts[r] = max(cuts[r], cuts[r - 1])
    return cuts[rank], cuts[rank + 1]


def merge_fronts(ids: torch.Tensor, e: torch.Tensor, t: torch.Tensor, *, rho: float = 0.0, cap_front: int = 1 << 14,
                 group=None, rt: native.Runtime | None = None, occ: torch.Tensor | None = None):
    """All-gather local fronts (padded to ``cap_front``) and run the final skyline pass.
    Returns (ids, e, t, t_peak) of the global front, identical on every rank.  ``occ`` (occupancy of
    the local front members) switches to the three-objective rule (engine.skyline)."""
    rt = rt or native.get_runtime()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    k = int(ids.numel())
    if k > cap_front:
        from .errors import CapacityExceeded
        raise CapacityExceeded(f"local front of {k} points exceeds the exchange capacity {cap_front}")
    inf = float("inf")
    # one buffer, one collective: [cap, 3 or 4] = (e, t, id-as-f64-bits[, occ])
    width = 3 if occ is None else 4
    pack = torch.full((cap_front, width), inf, dtype=torch.float64, device=rt.device)
    pack[:k, 0], pack[:k, 1] = e, t
    pack[:k, 2] = ids.view(torch.float64) if ids.dtype == torch.int64 else ids.to(torch.int64).view(torch.float64)
    if occ is not None:
        pack[:, 3] = 0.0                                  # padding rows have e = t = inf and never enter the front
        pack[:k, 3] = occ
    if world > 1:
        gathered = torch.empty((world * cap_front, width), dtype=torch.float64, device=rt.device)
        dist.all_gather_into_tensor(gathered, pack, group=group)
    else:
        gathered = pack
    ge, gt = gathered[:, 0].contiguous(), gathered[:, 1].contiguous()
    gid = gathered[:, 2].contiguous().view(torch.int64)
    gocc = gathered[:, 3].contiguous() if occ is not None else None
    return engine.skyline(ge, gt, ids=gid, rho=rho, cap_front=cap_front, rt=rt, occ=gocc)


def sharded_skyline(e: torch.Tensor, t: torch.Tensor, first_id: int, *, rho: float = 0.0, cap_front: int = 1 << 14,
                    group=None, rt: native.Runtime | None = None, occ: torch.Tensor | None = None):
    """Front of a candidate set whose shard [first_id, first_id + len(e)) lives on this rank
    (two objectives, or three with ``occ``)."""
    rt = rt or native.get_runtime()
    # ids are positions in the shard (no id array for 10^9 candidates); the global id is first_id + position
    lpos, le, lt, _ = engine.skyline(e, t, rho=0.0, cap_front=cap_front, rt=rt, occ=occ)   # floor only at the end
    locc = occ[lpos].contiguous() if occ is not None else None
    lid = lpos + first_id
    return merge_fronts(lid, le, lt, rho=rho, cap_front=cap_front, group=group, rt=rt, occ=locc)
