"""Tensor-level entry points over libffb: the batched calls the reference lacks.

These are what bench.py and the corpus pipeline use; the drop-in functions in ``api``
are thin wrappers that re-materialise the reference's dataclasses from these tensors.
All tensors live on the runtime's device; host-side arguments (specs, shapes, caps) are
small and go through the C-ABI as host arrays.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from . import native
from .errors import raise_for_status
from .model_types import ArchitectureSpec, CalibrationProfile
from .specs import pack_spec


def spec_rows(specs) -> np.ndarray:
    """[(arch, profile) | (arch, profile, regs_per_sm)] -> float64 [S, SPEC_WIDTH]."""
    rows = []
    for item in specs:
        arch, prof, *rest = item
        rows.append(pack_spec(arch, prof, int(rest[0]) if rest else 0))
    return np.ascontiguousarray(np.asarray(rows, dtype=np.float64).reshape(len(rows), native.SPEC_WIDTH))


def shape_rows(shapes) -> np.ndarray:
    """[(bx, by) | (bx, by, bz) | (bx, by, bz, regs)] -> int32 [J, 4]."""
    out = np.ones((len(shapes), 4), dtype=np.int32)
    out[:, 3] = 0
    for i, sh in enumerate(shapes):
        out[i, : len(sh)] = sh
    return out


@dataclass
class GridResult:
    t: torch.Tensor | None        # [K,S,J,C] f64
    e: torch.Tensor | None
    pdyn: torch.Tensor | None
    flags: torch.Tensor | None    # u8
    occ: torch.Tensor | None      # [K,S,J]
    detail: torch.Tensor | None   # [K,S,J,C,DETAIL_WIDTH]
    status: int = 0


def score_grid(feat: torch.Tensor, res: torch.Tensor, spec: np.ndarray, shape: np.ndarray,
               cap: np.ndarray, *, want=("t", "e"), strict: bool = False, out: dict | None = None,
               check: bool = True, rt: native.Runtime | None = None) -> GridResult:
    """K2+K3 over kernel x spec x shape x cap (ffb_predict_grid).

    ``want`` selects outputs among t, e, pdyn, flags, occ, detail.  ``out`` may hold
    preallocated tensors under the same names (bench.py reuses its buffers).
    ``check=False`` skips the device->host read of the status word (no sync).
    """
    rt = rt or native.get_runtime()
    K, S, J, Cn = feat.shape[0], spec.shape[0], shape.shape[0], cap.shape[0]
    assert feat.dtype == torch.float64 and feat.shape[1] == native.FEAT_WIDTH and feat.is_contiguous()
    assert res.dtype == torch.int64 and tuple(res.shape) == (K, 2) and res.is_contiguous()
    spec = np.ascontiguousarray(spec, dtype=np.float64)
    shape = np.ascontiguousarray(shape, dtype=np.int32)
    cap = np.ascontiguousarray(cap, dtype=np.float64)
    out = dict(out or {})
    full = (K, S, J, Cn)

    def buf(name, shp, dtype):
        if name not in want:
            return None
        t = out.get(name)
        if t is None:
            t = rt.empty(shp, dtype)
        assert tuple(t.shape) == tuple(shp) and t.dtype == dtype and t.is_contiguous()
        return t

    r = GridResult(
        t=buf("t", full, torch.float64), e=buf("e", full, torch.float64),
        pdyn=buf("pdyn", full, torch.float64), flags=buf("flags", full, torch.uint8),
        occ=buf("occ", (K, S, J), torch.float64),
        detail=buf("detail", (*full, native.DETAIL_WIDTH), torch.float64),
    )
    status = torch.zeros(1, dtype=torch.int32, device=rt.device) if check else None
    g = native.GridDesc(
        n_kernels=K, n_specs=S, n_shapes=J, n_caps=Cn,
        d_feat=native.ptr(feat), d_res=native.ptr(res),
        h_spec=spec.ctypes.data, h_shape=shape.ctypes.data, h_cap=cap.ctypes.data,
        d_t=native.ptr(r.t), d_e=native.ptr(r.e), d_pdyn=native.ptr(r.pdyn), d_flags=native.ptr(r.flags),
        d_occ=native.ptr(r.occ), d_detail=native.ptr(r.detail), d_status=native.ptr(status),
        strict=1 if strict else 0,
    )
    rc = rt.lib.ffb_predict_grid(rt.ctx, C.byref(g), rt.stream())
    rt.check(rc, "ffb_predict_grid")
    if check:
        r.status = int(status.item()) & 0xFFFFFFFF
        if strict and r.status:
            for code in range(1, 32):
                if r.status & (1 << code):
                    raise_for_status(code, "model check failed on the device")
    return r


def score_grid_sweep(feat: torch.Tensor, res_axis: torch.Tensor, spec: np.ndarray, shape: np.ndarray, cap: np.ndarray,
                     **kw) -> GridResult:
    """Workload sweep in ONE launch: every kernel is scored under R resource rows
    (e.g. one per sequence length, launch.py:44-82).  ``res_axis`` is int64 [R, 2] (the same rows for
    every kernel) or [K, R, 2]; the kernel rows are replicated R times on the device and the grid
    kernel runs once over K*R rows.  Outputs gain an axis: t / e / ... [K, R, S, J, C], occ [K, R, S, J]."""
    K = feat.shape[0]
    if res_axis.dim() == 2:
        res_axis = res_axis.unsqueeze(0).expand(K, -1, -1)
    assert res_axis.dtype == torch.int64 and res_axis.shape[0] == K and res_axis.shape[2] == 2
    R = res_axis.shape[1]
    feat_r = feat.repeat_interleave(R, dim=0).contiguous()
    res_r = res_axis.reshape(K * R, 2).contiguous()
    r = score_grid(feat_r, res_r, spec, shape, cap, **kw)
    for name in ("t", "e", "pdyn", "flags", "occ", "detail"):
        v = getattr(r, name)
        if v is not None:
            setattr(r, name, v.view(K, R, *v.shape[1:]))
    return r


def enumerate_shapes(spec_row: np.ndarray, shared_dyn: int, dims, rt: native.Runtime | None = None) -> np.ndarray:
    """Valid (bx, by) pairs in canonical (threads, bx, by) order — explorer.py:76-88,93."""
    lib = (rt or native.get_runtime()).lib
    dims = np.ascontiguousarray(np.asarray(list(dims), dtype=np.int64))
    if dims.size and (dims.max() > 2**31 - 1 or dims.min() < -(2**31)):
        raise ValueError("block dimension candidates must fit int32")
    d32 = np.ascontiguousarray(dims.astype(np.int32))
    n = C.c_int64(0)
    cap = int(d32.size) * int(d32.size)
    outxy = np.empty((max(cap, 1), 2), dtype=np.int32)
    row = np.ascontiguousarray(spec_row, dtype=np.float64)
    rc = lib.ffb_enumerate_shapes(row.ctypes.data, int(shared_dyn), d32.ctypes.data, int(d32.size),
                                  outxy.ctypes.data, cap, C.byref(n))
    raise_for_status(rc, "ffb_enumerate_shapes")
    return outxy[: n.value].copy()


def skyline_groups(e: torch.Tensor, t: torch.Tensor, n_groups: int, group_size: int, *,
                   tie: torch.Tensor | None = None, rho: float = 0.95, cap_front: int | None = None,
                   compact: bool = False, out: tuple | None = None, check: bool = True,
                   rt: native.Runtime | None = None, occ: torch.Tensor | None = None):
    """K4 on n_groups consecutive groups.  ``occ`` adds the occupancy objective (extension: a
    candidate is dropped iff another has strictly lower e and t and occupancy at least as high).

    Dense (default): returns (front_idx [n_groups, cap_front], front_n, t_peak).
    ``compact=True``: returns (front_idx [cap_front] flat, front_n, t_peak, front_off) where group
    g's front is front_idx[front_off[g] : front_off[g] + front_n[g]]; cap_front is the TOTAL capacity.
    """
    rt = rt or native.get_runtime()
    assert e.dtype == torch.float64 and t.dtype == torch.float64 and e.is_contiguous() and t.is_contiguous()
    assert e.numel() == n_groups * group_size == t.numel()
    cap_front = int(cap_front if cap_front is not None else group_size)
    if out is not None:
        front_idx, front_n, tpeak, front_off = out
    else:
        front_idx = rt.empty((cap_front,) if compact else (n_groups, cap_front), torch.int32)
        front_n = rt.empty((n_groups,), torch.int32)
        tpeak = rt.empty((n_groups,), torch.float64)
        front_off = rt.empty((n_groups,), torch.int64) if compact else None
    status = torch.zeros(1, dtype=torch.int32, device=rt.device) if check else None
    if tie is not None:
        assert tie.dtype == torch.int32 and tie.numel() == group_size and tie.is_contiguous()
    if occ is not None:
        assert occ.dtype == torch.float64 and occ.numel() == e.numel() and occ.is_contiguous()
    rc = rt.lib.ffb_skyline_groups3(rt.ctx, native.ptr(e), native.ptr(t), native.ptr(occ), n_groups, group_size,
                                    native.ptr(tie), float(rho), native.ptr(front_idx), native.ptr(front_n),
                                    native.ptr(tpeak), cap_front, native.ptr(front_off), native.ptr(status), rt.stream())
    rt.check(rc, "ffb_skyline_groups")
    if check:
        st = int(status.item()) & 0xFFFFFFFF
        for code in range(1, 32):
            if st & (1 << code):
                raise_for_status(code, "skyline capacity exceeded (front or survivor buffer)")
    if compact:
        return front_idx, front_n, tpeak, front_off
    return front_idx, front_n, tpeak


def explore_groups(feat: torch.Tensor, res: torch.Tensor, spec: np.ndarray, shape: np.ndarray, cap: np.ndarray, *,
                   rho: float = 0.95, cap_front: int | None = None, compact: bool = False, want_values: bool = False,
                   out: tuple | None = None, check: bool = True, rt: native.Runtime | None = None):
    """K2 + K3 + K4 fused (ffb_explore_groups): the front of every (kernel, spec) group, grid never materialised.

    Same result as ``score_grid`` followed by ``skyline_groups`` with the reference tie key; group
    g = k * S + s, candidate index j * C + c.  Dense: (front_idx [K*S, cap_front], front_n, t_peak);
    ``compact=True``: (front_idx [cap_front], front_n, t_peak, front_off).  ``want_values`` appends
    (front_e, front_t) laid out like front_idx.  ``out`` = preallocated (front_idx, front_n, t_peak, front_off)."""
    rt = rt or native.get_runtime()
    K, S, J, Cn = feat.shape[0], spec.shape[0], shape.shape[0], cap.shape[0]
    assert feat.dtype == torch.float64 and feat.shape[1] == native.FEAT_WIDTH and feat.is_contiguous()
    assert res.dtype == torch.int64 and tuple(res.shape) == (K, 2) and res.is_contiguous()
    spec = np.ascontiguousarray(spec, dtype=np.float64)
    shape = np.ascontiguousarray(shape, dtype=np.int32)
    cap = np.ascontiguousarray(cap, dtype=np.float64)
    n_groups = K * S
    cap_front = int(cap_front if cap_front is not None else J * Cn)
    if out is not None:
        front_idx, front_n, tpeak, front_off = out
    else:
        front_idx = rt.empty((cap_front,) if compact else (n_groups, cap_front), torch.int32)
        front_n = rt.empty((n_groups,), torch.int32)
        tpeak = rt.empty((n_groups,), torch.float64)
        front_off = rt.empty((n_groups,), torch.int64) if compact else None
    fe = rt.empty(tuple(front_idx.shape), torch.float64) if want_values else None
    ft = rt.empty(tuple(front_idx.shape), torch.float64) if want_values else None
    status = torch.zeros(1, dtype=torch.int32, device=rt.device) if check else None
    d = native.ExploreDesc(
        n_kernels=K, n_specs=S, n_shapes=J, n_caps=Cn, d_feat=native.ptr(feat), d_res=native.ptr(res),
        h_spec=spec.ctypes.data, h_shape=shape.ctypes.data, h_cap=cap.ctypes.data, rho=float(rho),
        d_front_idx=native.ptr(front_idx), d_front_n=native.ptr(front_n), d_tpeak=native.ptr(tpeak), cap_front=cap_front,
        d_front_off=native.ptr(front_off), d_front_e=native.ptr(fe), d_front_t=native.ptr(ft), d_status=native.ptr(status))
    rc = rt.lib.ffb_explore_groups(rt.ctx, C.byref(d), rt.stream())
    rt.check(rc, "ffb_explore_groups")
    if check:
        st = int(status.item()) & 0xFFFFFFFF
        for code in range(1, 32):
            if st & (1 << code):
                raise_for_status(code, "explore: front buffer too small")
    res_t = (front_idx, front_n, tpeak, front_off) if compact else (front_idx, front_n, tpeak)
    return res_t + ((fe, ft) if want_values else ())


def skyline(e: torch.Tensor, t: torch.Tensor, *, ids: torch.Tensor | None = None, rho: float = 0.0,
            cap_front: int = 1 << 16, rt: native.Runtime | None = None, occ: torch.Tensor | None = None):
    """K4 on one large candidate set.  Returns (ids, e, t, t_peak) of the front in (e, t, id) order."""
    rt = rt or native.get_runtime()
    assert e.dtype == torch.float64 and t.dtype == torch.float64 and e.is_contiguous() and t.is_contiguous()
    n = e.numel()
    assert t.numel() == n
    out_id = rt.empty((cap_front,), torch.int64)
    out_e = rt.empty((cap_front,), torch.float64)
    out_t = rt.empty((cap_front,), torch.float64)
    n_out, tpeak = C.c_int64(0), C.c_double(float("inf"))
    if ids is not None:
        assert ids.dtype == torch.int64 and ids.numel() == n and ids.is_contiguous()
    if occ is not None:
        assert occ.dtype == torch.float64 and occ.numel() == n and occ.is_contiguous()
    rc = rt.lib.ffb_skyline(rt.ctx, native.ptr(e), native.ptr(t), native.ptr(occ), native.ptr(ids), n, float(rho),
                            native.ptr(out_id), native.ptr(out_e), native.ptr(out_t), cap_front,
                            C.byref(n_out), C.byref(tpeak), rt.stream())
    rt.check(rc, "ffb_skyline")
    k = n_out.value
    return out_id[:k], out_e[:k], out_t[:k], tpeak.value


def features_tensor(rows, rt: native.Runtime | None = None) -> torch.Tensor:
    rt = rt or native.get_runtime()
    arr = np.asarray(rows, dtype=np.float64).reshape(-1, native.FEAT_WIDTH)
    return rt.to_device(torch.from_numpy(np.ascontiguousarray(arr)))


def resources_tensor(rows, rt: native.Runtime | None = None) -> torch.Tensor:
    rt = rt or native.get_runtime()
    arr = np.asarray(rows, dtype=np.int64).reshape(-1, 2)
    return rt.to_device(torch.from_numpy(np.ascontiguousarray(arr)))
