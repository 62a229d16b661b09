"""ctypes binding of the C ABI in include/askv.h (libaskv.so, sm_100a).

There is deliberately no fallback: if the library is missing or fails to load
every operation raises (north star: "no CPU fallback").
"""

from __future__ import annotations

import ctypes as C
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "libaskv.so"

ASKV_OK = 0
ASKV_EINVAL = -1
ASKV_ECUDA = -2
ASKV_EUNSUPPORTED = -3

_vp, _i32, _i64, _f32, _f64, _sz = C.c_void_p, C.c_int, C.c_int64, C.c_float, C.c_double, C.c_size_t
_pi64 = C.POINTER(C.c_int64)

# name -> (restype, argtypes); must match include/askv.h exactly
SIGNATURES = {
    "askv_version": (_i32, []),
    "askv_last_error": (C.c_char_p, []),
    "askv_rope_table": (_i32, [_vp, _i32, _i32, _f64, _vp]),
    "askv_reembed": (_i32, [_vp, _vp, _i32, _i64, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _i32,
                            _vp, _i64, _vp]),
    "askv_rotate_rows": (_i32, [_vp, _i64, _i32, _i32, _i32, _vp, _i32, _vp, _i32, _vp, _i64,
                                _vp]),
    "askv_rope_new": (_i32, [_vp, _i64, _i32, _i32, _i32, _i32, _vp, _i32, _i32, _vp, _vp, _i64,
                             _vp, _vp]),
    "askv_prefill_attn": (_i32, [_vp, _vp, _i64, _i32, _i32, _i32, _i32, _i32, _f32, _vp, _vp,
                                 _sz, _i32, _vp]),
    "askv_attn_workspace_bytes": (_sz, [_i32, _i32, _i32, _i32, _i32]),
    "askv_attn_num_splits": (_i32, [_i32, _i32, _i32, _i32]),
    "askv_preload_layer": (_i32, [_vp, _vp, _pi64, _i32, _i64, _i64, _i64, _i64, _vp, _vp]),
    "askv_save_layer": (_i32, [_vp, _pi64, _i32, _i64, _i64, _i32, _i64, _i64, _i32, _vp, _vp,
                               _vp]),
    "askv_rmsnorm": (_i32, [_vp, _vp, _vp, _i32, _i32, _f32, _vp]),
    "askv_copy_sm": (_i32, [_vp, _vp, _sz, _vp]),
    "askv_silu_mul": (_i32, [_vp, _vp, _i32, _i32, _vp]),
}

_lock = threading.Lock()
_lib = None


class AskvError(RuntimeError):
    pass


def lib():
    """Load libaskv.so once; raise loudly if it is absent."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise AskvError(
                    f"{LIB_PATH} is not built; run `python -m paper_2403_19708_b200.build` "
                    "(there is no non-CUDA fallback)")
            handle = C.CDLL(str(LIB_PATH))
            for name, (res, args) in SIGNATURES.items():
                fn = getattr(handle, name)
                fn.restype = res
                fn.argtypes = args
            _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc == ASKV_OK:
        return
    msg = lib().askv_last_error().decode(errors="replace")
    if rc == ASKV_EINVAL:
        raise ValueError(f"{what}: {msg}")
    raise AskvError(f"{what} failed ({rc}): {msg}")
