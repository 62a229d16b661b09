"""ctypes binding of the C ABI in include/askv.h (libaskv.so, sm_100a).

There is deliberately no fallback: if the library is missing or fails to load
every operation raises (north star: "no CPU fallback").
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

LIB_PATH = Path(os.environ.get("ASKV_LIB") or Path(__file__).resolve().parent / "libaskv.so")

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
    "askv_attn_workspace_bytes_gqa": (_sz, [_i32, _i32, _i32, _i32, _i32, _i32]),
    "askv_gemm": (_i32, [_vp, _vp, _vp, _i32, _i32, _i32, _i32, _vp, _sz, _vp]),
    "askv_prefill_layers_batch": (_i32, [_vp, _i32, _vp]),
    "askv_issue_stats": (None, [_vp]),
    "askv_save_layers": (_i32, [_vp, _vp, _i32, _i64, _i64, _i32, _i32, _i64, _i64, _i32, _vp,
                                _vp, _vp, _vp, _vp, _vp, _vp]),
    "askv_nccl_unique_id": (_i32, [_vp]),
    "askv_nccl_comm_init": (_i32, [_i32, _i32, _vp, C.POINTER(_vp)]),
    "askv_nccl_comm_destroy": (_i32, [_vp]),
    "askv_nccl_allreduce_bf16": (_i32, [_vp, _vp, _i64, _vp, _vp]),
    "askv_attn_num_splits": (_i32, [_i32, _i32, _i32, _i32]),
    "askv_attn_num_splits_gqa": (_i32, [_i32, _i32, _i32, _i32, _i32]),
    "askv_preload_layer": (_i32, [_vp, _vp, _pi64, _i32, _i64, _i64, _i64, _i64, _vp, _vp]),
    "askv_save_layer": (_i32, [_vp, _pi64, _i32, _i64, _i64, _i32, _i64, _i64, _i32, _vp, _vp,
                               _vp]),
    "askv_rmsnorm": (_i32, [_vp, _vp, _vp, _i32, _i32, _f32, _vp]),
    "askv_copy_sm": (_i32, [_vp, _vp, _sz, _vp]),
    "askv_event_create": (_i32, [C.POINTER(C.c_void_p), _i32]),
    "askv_event_destroy": (_i32, [_vp]),
    "askv_event_record": (_i32, [_vp, _vp]),
    "askv_stream_wait_event": (_i32, [_vp, _vp]),
    "askv_event_elapsed_ms": (_i32, [_vp, _vp, C.POINTER(C.c_float)]),
    "askv_event_synchronize": (_i32, [_vp]),
    "askv_prefill_layers": (_i32, [_vp, _vp]),
    "askv_prefill_plan_size": (_sz, []),
    "askv_stamp": (_i32, [_vp, _vp]),
    "askv_gemm_autotune": (_i32, [_i32, _i32, _i32, _sz, _vp]),
    "askv_l2_persist": (_i32, [_sz, C.POINTER(C.c_size_t)]),
    "askv_silu_mul": (_i32, [_vp, _vp, _i32, _i32, _vp]),
}

_pp = C.POINTER(C.c_void_p)
ALLREDUCE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p)


class PrefillPlan(C.Structure):
    """ctypes mirror of askv_prefill_plan (include/askv.h)."""
    _fields_ = [
        ("layers", C.c_int32), ("d_model", C.c_int32), ("n_heads", C.c_int32),
        ("n_kv_heads", C.c_int32), ("head_dim", C.c_int32), ("ffn", C.c_int32),
        ("n_new", C.c_int32), ("kept", C.c_int32), ("head", C.c_int32),
        ("rms_eps", C.c_float), ("attn_scale", C.c_float), ("attn_splits", C.c_int32),
        ("w_in", _pp), ("w_qkv", _pp), ("w_o", _pp), ("w_post", _pp), ("w_gu", _pp),
        ("w_down", _pp),
        ("x", C.c_void_p), ("h", C.c_void_p), ("qkv", C.c_void_p), ("q_rot", C.c_void_p),
        ("kv", C.c_void_p), ("attn_out", C.c_void_p), ("gu", C.c_void_p), ("act", C.c_void_p),
        ("attn_ws", C.c_void_p), ("attn_ws_bytes", C.c_size_t),
        ("gemm_ws", C.c_void_p), ("gemm_ws_bytes", C.c_size_t),
        ("rope_table", C.c_void_p), ("rope_positions", C.c_int32),
        ("src_kind", C.c_int32), ("src_layer", _pp), ("src_block_off", C.c_void_p),
        ("block_tokens", C.c_int32), ("src_row_stride", C.c_int64),
        ("ev_src_ready", _pp), ("ev_src_free", _pp),
        ("save_rows", _pp), ("ev_save_free", _pp), ("ev_save_ready", _pp),
        ("promote_base", C.c_void_p), ("promote_block_ids", C.POINTER(C.c_int64)),
        ("promote_nblocks", C.c_int32),
        ("block_bytes", C.c_int64), ("chunk_bytes", C.c_int64), ("row_bytes", C.c_int64),
        ("stamps", C.c_void_p), ("stamp_flags", C.c_int32),
        ("allreduce", ALLREDUCE_FN), ("allreduce_ctx", C.c_void_p),
        ("kv_layers", _pp), ("graph", C.c_int32), ("kv_alt", C.c_void_p),
        ("mirror_base", C.c_void_p), ("mirror_block_ids", C.POINTER(C.c_int64)),
        ("mirror_nblocks", C.c_int32),
        ("nccl_comm", C.c_void_p), ("tp_rank", C.c_int32),
        ("src_rows", C.c_int64),
    ]


_lock = threading.Lock()
_lib = None


class AskvError(RuntimeError):
    pass


def _preload_torch_cublaslt() -> None:
    """libaskv.so needs libcublasLt.so.12.  torch ships its own copy (pip
    nvidia-cublas); if ours (the CUDA toolkit's) were loaded first, torch's
    libcublas would bind to a mismatched cuBLASLt and fail (CUBLAS_STATUS_
    INVALID_VALUE).  Load torch's copy first, globally, so one cuBLASLt serves
    both."""
    try:
        import nvidia.cublas as nc
    except ImportError:
        return
    import os
    for base in nc.__path__:
        path = os.path.join(base, "lib", "libcublasLt.so.12")
        if os.path.exists(path):
            C.CDLL(path, mode=C.RTLD_GLOBAL)
            return


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
            _preload_torch_cublaslt()
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
