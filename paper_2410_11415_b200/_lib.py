"""ctypes binding of ``libklay.so`` (the C ABI declared in ``include/klay.h``).

This is the binding a maintainer of the reference would add:
the reference engine is pure Python + numpy, so its natural FFI is ctypes.
There is no fallback: if the library is missing, every entry point raises.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libklay.so")

KLAY_OK, KLAY_EINVAL, KLAY_EFORMAT, KLAY_ECUDA, KLAY_EUNSUPPORTED = range(5)
KLAY_REAL, KLAY_LOG, KLAY_BOOL, KLAY_MAXPROD = range(4)
KLAY_F32, KLAY_F64, KLAY_U1 = 0, 1, 2
KLAY_RETAIN_BACKWARD = 2

_c_i64 = ctypes.c_int64
_c_i32 = ctypes.c_int32
_vp = ctypes.c_void_p

# name -> (restype, argtypes); must match include/klay.h exactly
SIGNATURES = {
    "klay_version": (ctypes.c_char_p, []),
    "klay_last_error": (ctypes.c_char_p, []),
    "klay_plan_create": (ctypes.c_int, [_c_i64, _c_i32, _vp, _vp, _vp, _vp, _c_i32, _vp, _vp,
                                        _c_i32, ctypes.POINTER(_vp)]),
    "klay_plan_destroy": (ctypes.c_int, [_vp]),
    "klay_plan_num_nodes": (_c_i64, [_vp]),
    "klay_plan_max_width": (_c_i64, [_vp]),
    "klay_plan_schedule": (ctypes.c_int, [_vp, _vp]),
    "klay_plan_layer_offset": (_c_i64, [_vp, _c_i32]),
    "klay_row_stride": (_c_i64, [_c_i64, _c_i32]),
    "klay_forward": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _c_i32, _vp, _c_i64, _c_i32, _vp,
                                    _c_i64, ctypes.c_double, _vp, _vp]),
    "klay_forward_workspace": (ctypes.c_size_t, [_vp, _c_i32, _c_i64]),
    "klay_backward": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _c_i64, _vp, _vp, _vp, _c_i64,
                                      ctypes.c_double, _c_i32, _vp]),
    "klay_backward_workspace": (ctypes.c_size_t, [_vp, _c_i32, _c_i64]),
    "klay_fill_trace": (ctypes.c_int, [_vp, _c_i32, _c_i32, _vp, _c_i64, _c_i64, ctypes.c_double,
                                        _vp]),
    "klay_read_klay": (ctypes.c_int, [ctypes.c_char_p, _c_i64, ctypes.POINTER(_vp)]),
    "klay_read_klay_error": (ctypes.c_char_p, []),
    "klay_file_info": (ctypes.c_int, [_vp, _vp]),
    "klay_file_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "klay_file_destroy": (None, [_vp]),
    "klay_layerize": (ctypes.c_int, [_c_i32, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp,
                                     ctypes.POINTER(_vp)]),
    "klay_layered_info": (_c_i64, [_vp, _c_i32]),
    "klay_layered_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "klay_layered_destroy": (None, [_vp]),
    "klay_layerize_error": (ctypes.c_char_p, []),
    "klay_launch_count": (_c_i64, []),
    "klay_set_launch_filter": (ctypes.c_uint32, [ctypes.c_uint32]),
    "klay_profiler_begin": (ctypes.c_int, []),
    "klay_profiler_end": (ctypes.c_int, [_c_i32, _vp, _vp, _vp, _vp]),
}


class KlayLibError(RuntimeError):
    """libklay missing or a call failed (non-shape failures)."""


_lib = None


def load(path: str | None = None):
    """Load libklay.so (once). Raises KlayLibError when it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("KLAY_LIB", LIB_PATH)
    if not os.path.exists(path):
        raise KlayLibError(
            f"libklay.so not found at {path}; build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (there is no CPU fallback)")
    lib = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    return load().klay_last_error().decode("utf-8", "replace")


def check(rc: int, what: str) -> None:
    if rc == KLAY_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc in (KLAY_EINVAL, KLAY_EUNSUPPORTED):
        from .engine import EvalError
        raise EvalError(msg)
    if rc == KLAY_EFORMAT:
        from .tensorized import KlayFormatError
        raise KlayFormatError(msg)
    raise KlayLibError(msg)
