"""ctypes binding of libffb.so (include/ffb.h) and the per-device runtime object.

There is deliberately no CPU implementation behind these calls: if the shared object
or a CUDA device is missing, ``get_runtime`` raises ``NativeLibraryMissing``.

The CPU test-suite exercises the same kernels through a SIMT-emulated build of the very
same sources (tests/simt); it installs that build explicitly with
``install_runtime_for_tests`` — the package never looks for it on its own.
"""
from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

import torch

from .errors import NativeLibraryMissing, raise_for_status

FEAT_WIDTH = 18
(F_N_MEM, F_MEM_BYTES, F_FP32, F_INT, F_SFU, F_ALU, F_N_SYNC, F_ALIGNED, F_STATIC_SHARED,
 F_REGS_DECLARED, F_N_INSTR, F_RESERVED, F_OVR, F_OVR_WARPS, F_OVR_BPS, F_OVR_ETA, F_OVR_NCOMP,
 F_OVR_TEXEC) = range(18)
SPEC_WIDTH = 48
DETAIL_WIDTH = 21
N_CLASSES = 9
PT_VALID, PT_CAP_LIMITED = 1, 2

(D_MWP, D_CWP, D_BW_EFF, D_T_MEM, D_T_COMP, D_T_SYNC, D_T_EXEC, D_P_UNITS, D_P_SHAPE, D_P_MEM,
 D_P_SM, D_P_DYN, D_F_ADJ, D_CI, D_ACTIVE_SMS, D_CAP_LIMITED, D_E_PRED, D_WARPS, D_BLOCKS_PER_SM,
 D_ETA, D_WAVES) = range(DETAIL_WIDTH)

_vp, _i64, _i32, _f64 = C.c_void_p, C.c_int64, C.c_int32, C.c_double


class GridDesc(C.Structure):
    _fields_ = [
        ("n_kernels", _i64), ("n_specs", _i64), ("n_shapes", _i64), ("n_caps", _i64),
        ("d_feat", _vp), ("d_res", _vp), ("h_spec", _vp), ("h_shape", _vp), ("h_cap", _vp),
        ("d_t", _vp), ("d_e", _vp), ("d_pdyn", _vp), ("d_flags", _vp), ("d_occ", _vp),
        ("d_detail", _vp), ("d_status", _vp), ("strict", _i32),
    ]


class ExploreDesc(C.Structure):
    _fields_ = [
        ("n_kernels", _i64), ("n_specs", _i64), ("n_shapes", _i64), ("n_caps", _i64),
        ("d_feat", _vp), ("d_res", _vp), ("h_spec", _vp), ("h_shape", _vp), ("h_cap", _vp),
        ("rho", _f64), ("d_front_idx", _vp), ("d_front_n", _vp), ("d_tpeak", _vp), ("cap_front", _i64),
        ("d_front_off", _vp), ("d_front_e", _vp), ("d_front_t", _vp), ("d_status", _vp),
    ]


_SIGNATURES = {
    "ffb_abi_version": (_i32, []),
    "ffb_create": (_i32, [_i32, C.POINTER(_vp)]),
    "ffb_destroy": (_i32, [_vp]),
    "ffb_last_error": (C.c_char_p, [_vp]),
    "ffb_launch_count": (_i64, [_vp]),
    "ffb_predict_grid": (_i32, [_vp, C.POINTER(GridDesc), _vp]),
    "ffb_explore_groups": (_i32, [_vp, C.POINTER(ExploreDesc), _vp]),
    "ffb_enumerate_shapes": (_i32, [_vp, _i64, _vp, _i64, _vp, _i64, C.POINTER(_i64)]),
    "ffb_skyline_groups": (_i32, [_vp, _vp, _vp, _i64, _i64, _vp, _f64, _vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "ffb_skyline_groups3": (_i32, [_vp, _vp, _vp, _vp, _i64, _i64, _vp, _f64, _vp, _vp, _vp, _i64, _vp, _vp, _vp]),
    "ffb_lex_corpus": (_i32, [_vp, _vp, _vp]),
    "ffb_kernel_features": (_i32, [_vp, _vp, _vp]),
    "ffb_classify_opcodes": (_i32, [_vp, _vp, _vp, _i64, _vp, _vp]),
    "ffb_name_hash": (C.c_uint64, [C.c_char_p, _i64]),
    "ffb_skyline": (_i32, [_vp, _vp, _vp, _vp, _vp, _i64, _f64, _vp, _vp, _vp, _i64,
                           C.POINTER(_i64), C.POINTER(_f64), _vp]),
}

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "libffb.so"


def bind(path: str | Path) -> C.CDLL:
    lib = C.CDLL(str(path))
    for name, (res, args) in _SIGNATURES.items():
        fn = getattr(lib, name)        # AttributeError if the .so lacks a declared symbol
        fn.restype = res
        fn.argtypes = args
    return lib


def declared_symbols() -> tuple[str, ...]:
    return tuple(_SIGNATURES)


class _LockedLib:
    """The context is not thread-safe by itself (include/ffb.h): its host staging buffer, table
    shadow and scratch reservations are per context.  Every ffb_* call made through a Runtime
    therefore holds the runtime's lock, so Python threads sharing the per-device runtime
    (the reference's ``evaluate_configs(jobs>1)`` is reentrant, explorer.py:177-179) cannot
    interleave inside a call.  Ordering on the device is the stream's; a context serves one
    stream at a time unless the caller orders the streams itself (corpus.StreamedAnalysis does)."""

    def __init__(self, lib: C.CDLL, lock: threading.RLock):
        self._lib, self._lock = lib, lock

    def __getattr__(self, name):
        fn = getattr(self._lib, name)
        lock = self._lock

        def call(*args):
            with lock:
                return fn(*args)
        call.__name__ = name
        setattr(self, name, call)
        return call


class Runtime:
    """One libffb context on one device plus tensor helpers."""

    def __init__(self, lib: C.CDLL, device: torch.device, device_index: int = 0):
        self.lock = threading.RLock()
        self.raw_lib = lib
        self.lib = _LockedLib(lib, self.lock)
        self.device = device
        handle = _vp()
        rc = self.lib.ffb_create(device_index, C.byref(handle))
        if rc != 0 or not handle.value:
            raise NativeLibraryMissing(f"ffb_create failed on device {device_index} (status {rc})")
        self.ctx = handle
        self._status = torch.zeros(1, dtype=torch.int32, device=device)

    # -- helpers
    def stream(self) -> int:
        if self.device.type == "cuda":
            return torch.cuda.current_stream(self.device).cuda_stream
        return 0

    def check(self, rc: int, what: str) -> None:
        if rc != 0:
            msg = self.lib.ffb_last_error(self.ctx)
            raise_for_status(rc, f"{what}: {msg.decode() if msg else ''}")

    def launches(self) -> int:
        return int(self.lib.ffb_launch_count(self.ctx))

    def empty(self, shape, dtype) -> torch.Tensor:
        return torch.empty(shape, dtype=dtype, device=self.device)

    def to_device(self, t: torch.Tensor, dtype=None) -> torch.Tensor:
        if dtype is not None and t.dtype != dtype:
            t = t.to(dtype)
        return t.to(self.device, non_blocking=True).contiguous()

    def close(self) -> None:
        if getattr(self, "ctx", None) is not None and self.ctx.value:
            self.lib.ffb_destroy(self.ctx)
            self.ctx = _vp()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_lock = threading.Lock()
_runtimes: dict[int, Runtime] = {}
_test_runtime: Runtime | None = None
_lib: C.CDLL | None = None


def load_library() -> C.CDLL:
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise NativeLibraryMissing(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(needs nvcc). This package has no CPU path.")
        _lib = bind(LIB_PATH)
        if _lib.ffb_abi_version() != 1:
            raise NativeLibraryMissing("libffb.so ABI version mismatch; rebuild")
    return _lib


def get_runtime(device: int | None = None) -> Runtime:
    if _test_runtime is not None:
        return _test_runtime
    if not torch.cuda.is_available():
        raise NativeLibraryMissing("no CUDA device visible; this package has no CPU path")
    idx = torch.cuda.current_device() if device is None else int(device)
    with _lock:
        rt = _runtimes.get(idx)
        if rt is None:
            rt = Runtime(load_library(), torch.device("cuda", idx), idx)
            _runtimes[idx] = rt
    return rt


def install_runtime_for_tests(rt: Runtime | None) -> None:
    """Test hook (tests/conftest.py): route calls to a SIMT-emulated build on host memory."""
    global _test_runtime
    _test_runtime = rt


def ptr(t: torch.Tensor | None) -> int | None:
    if t is None:
        return None
    assert t.is_contiguous()
    return t.data_ptr()
