"""ctypes binding of libmoba_b200.so (the C ABI in include/moba_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA
device is present, every op raises. Status codes map onto the reference's
exception classes (src/core.py:17-38).
"""

from __future__ import annotations

import ctypes
import os

from .core import ConfigError, MobaError, PlanValidationError, ShapeError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MOBA_LIB") or os.path.join(_HERE, "libmoba_b200.so")

MOBA_OK = 0
MOBA_ERR_SHAPE = 1
MOBA_ERR_CONFIG = 2
MOBA_ERR_PLAN = 3
MOBA_ERR_CUDA = 4
MOBA_ERR_UNSUPPORTED = 5
MOBA_ERR_WORKSPACE = 6

MOBA_ROUTE_FP32 = 0
MOBA_ROUTE_TC = 1

_p = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_f32 = ctypes.c_float
_sz = ctypes.c_size_t

# name -> (restype, argtypes); every symbol declared in include/moba_b200.h
SIGNATURES = {
    "moba_version": (ctypes.c_char_p, []),
    "moba_status_string": (ctypes.c_char_p, [_i32]),
    "moba_last_error": (ctypes.c_char_p, []),
    "moba_centroids": (_i32, [_p, _p, _i32, _i64, _i64, _i32, _i32, _p, _p, _p]),
    "moba_centroids_f32": (_i32, [_p, _p, _i32, _i64, _i64, _i32, _i32, _p, _p, _p]),
    "moba_route_workspace_size": (_sz, [_i64, _i64, _i32, _i32]),
    "moba_route": (_i32, [_p, _p, _i64, _i64, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "moba_varlen": (_i32, [_p, _i64, _i64, _i32, _i32, _p, _p, _p, _p, _p, _sz, _p]),
    "moba_plan_row_pos": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _i32, _p, _p]),
    "moba_validate_plan": (_i32, [_p, _p, _p, _p, _i64, _i64, _i32, _i32, _p, _sz, _p]),
    "moba_fwd_workspace_size": (_sz, [_i64, _i64, _i32, _i32, _i32]),
    "moba_bwd_workspace_size": (_sz, [_i64, _i64, _i32, _i32, _i32, _i32]),
    "moba_fwd": (_i32, [_p, _p, _p, _i64, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _f32, _p, _p, _p, _sz, _p]),
    "moba_bwd": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _i32,
                        _f32, _p, _p, _p, _p, _sz, _p]),
    "moba_route_gqa": (_i32, [_p, _p, _i64, _i32, _i64, _i32, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "moba_route_f32": (_i32, [_p, _p, _i64, _i32, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _p, _p, _sz, _p]),
    "moba_fwd_gqa": (_i32, [_p, _p, _p, _i64, _i32, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _f32, _p, _p, _p, _sz,
                            _p]),
    "moba_bwd_gqa_workspace_size": (_sz, [_i64, _i32, _i64, _i32, _i32, _i32, _i32]),
    "moba_bwd_gqa": (_i32, [_p, _p, _p, _p, _p, _p, _i64, _i32, _i64, _i32, _i32, _i32, _p, _p, _p, _p, _i32,
                            _f32, _p, _p, _p, _p, _sz, _p]),
    "moba_conv_bwd_workspace_size": (_sz, [_i64, _i64, _i32, _i32]),
    "moba_conv_bwd": (_i32, [_p, _p, _i32, _p, _i64, _i64, _i32, _p, _p, _p, _sz, _p]),
    "moba_launch_count": (ctypes.c_ulonglong, []),
    "moba_timing_enable": (None, [_i32]),
    "moba_timing_enabled": (_i32, []),
    "moba_timing_reset": (None, []),
    "moba_timing_read": (_i32, [ctypes.c_char_p, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_longlong)]),
}

STAGES = ("centroid", "route", "varlen", "fwd", "combine", "bwd_pre", "bwd", "bwd_post", "conv_bwd")


def timing_read() -> dict:
    """{stage: (total_ms, launches)} from the library's event timers."""
    lib = load()
    out = {}
    for st in STAGES:
        ms = ctypes.c_double()
        n = ctypes.c_longlong()
        check(lib.moba_timing_read(st.encode(), ctypes.byref(ms), ctypes.byref(n)), "moba_timing_read")
        out[st] = (ms.value, n.value)
    return out

_lib = None


def load():
    """Load and type the library (idempotent). Raises if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise MobaError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(or `make -C paper_2511_11571_b200/csrc`). There is no CPU fallback.")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def check(status: int, what: str) -> None:
    if status == MOBA_OK:
        return
    lib = load()
    msg = f"{what}: {lib.moba_status_string(status).decode()}"
    detail = lib.moba_last_error().decode()
    if detail:
        msg += f" ({detail})"
    if status == MOBA_ERR_SHAPE:
        raise ShapeError(msg)
    if status in (MOBA_ERR_CONFIG, MOBA_ERR_UNSUPPORTED):
        raise ConfigError(msg)
    if status == MOBA_ERR_PLAN:
        raise PlanValidationError(msg)
    raise MobaError(msg)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None -> NULL)."""
    return None if t is None else t.data_ptr()


def stream_ptr(device=None) -> int:
    import torch
    return torch.cuda.current_stream(device).cuda_stream
