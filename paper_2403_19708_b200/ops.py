"""torch-facing wrappers over the C ABI (device memory and streams come from
torch; the compute is libaskv.so).  Every wrapper launches on the current
CUDA stream unless ``stream`` is given."""

from __future__ import annotations

import ctypes as C
import math
from functools import lru_cache

import numpy as np
import torch

from ._lib import check, lib

BF16 = torch.bfloat16


def _stream(stream) -> int:
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _ptr(t):
    return None if t is None else t.data_ptr()


def _check_positions(positions, table: "RopeTable") -> None:
    """Explicit positions index the cos/sin table, which the kernels do not
    bound-check: every entry must lie in [0, table.max_pos) (a host sync; this
    is the numeric API, the layer loop uses pos0 + i and is checked natively)."""
    if positions is None or positions.numel() == 0:
        return
    lo, hi = int(positions.min()), int(positions.max())
    if lo < 0 or hi >= table.max_pos:
        raise ValueError(f"positions [{lo}, {hi}] outside the RoPE table's "
                         f"[0, {table.max_pos})")


def _require_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("expected a CUDA tensor")


class RopeTable:
    """fp64-derived fp32 (cos, sin) table, shape (max_pos, head_dim/2, 2)."""

    def __init__(self, max_pos: int, head_dim: int, theta_base: float = 10000.0,
                 device=None):
        self.max_pos = int(max_pos)
        self.head_dim = int(head_dim)
        self.theta_base = float(theta_base)
        self.table = torch.empty((self.max_pos, self.head_dim // 2, 2), dtype=torch.float32,
                                 device=device or "cuda")
        check(lib().askv_rope_table(self.table.data_ptr(), self.max_pos, self.head_dim,
                                    self.theta_base, _stream(None)), "rope_table")


@lru_cache(maxsize=16)
def _cached_table(max_pos: int, head_dim: int, theta_base: float, device: str) -> RopeTable:
    return RopeTable(max_pos, head_dim, theta_base, device)


def rope_table(max_pos: int, head_dim: int, theta_base: float = 10000.0, device="cuda"):
    # round up so repeated calls with growing positions share a table
    cap = 1 << max(12, int(math.ceil(math.log2(max(1, max_pos)))))
    return _cached_table(cap, int(head_dim), float(theta_base), str(torch.device(device)))


def reembed(src: torch.Tensor, kept: int, n_kv_heads: int, head_dim: int, table: RopeTable,
            dst: torch.Tensor, *, first_token: int = 0, pos0: int = 0, positions=None,
            block_off: torch.Tensor | None = None, block_tokens: int = 0,
            src_row_stride: int | None = None, dst_row_stride: int | None = None,
            stream=None) -> None:
    """K2: dst[i] = [rope(K, pos), V] of source row first_token+i (see askv.h)."""
    _require_cuda(src, dst, block_off, positions)
    _check_positions(positions, table)
    row = 2 * n_kv_heads * head_dim
    check(lib().askv_reembed(
        src.data_ptr(), _ptr(block_off), int(block_tokens),
        int(src_row_stride if src_row_stride is not None else row), int(first_token), int(kept),
        int(n_kv_heads), int(head_dim), table.table.data_ptr(), table.max_pos,
        _ptr(positions), int(pos0), dst.data_ptr(),
        int(dst_row_stride if dst_row_stride is not None else row), _stream(stream)), "reembed")


def rotate_rows(x: torch.Tensor, n_heads: int, head_dim: int, table: RopeTable,
                out: torch.Tensor, *, positions=None, pos0: int = 0, stream=None) -> None:
    _require_cuda(x, out, positions)
    _check_positions(positions, table)
    n = x.shape[0]
    check(lib().askv_rotate_rows(x.data_ptr(), int(x.stride(0)), int(n), int(n_heads),
                                 int(head_dim), table.table.data_ptr(), table.max_pos,
                                 _ptr(positions), int(pos0), out.data_ptr(), int(out.stride(0)),
                                 _stream(stream)), "rotate_rows")


def rope_new(qkv: torch.Tensor, n_new: int, n_heads: int, n_kv_heads: int, head_dim: int,
             table: RopeTable, pos0: int, q_out: torch.Tensor, kv_out: torch.Tensor,
             save_out: torch.Tensor | None = None, *, kv_row_stride: int | None = None,
             stream=None) -> None:
    _require_cuda(qkv, q_out, kv_out, save_out)
    row = 2 * n_kv_heads * head_dim
    check(lib().askv_rope_new(
        qkv.data_ptr(), int(qkv.stride(0)), int(n_new), int(n_heads), int(n_kv_heads),
        int(head_dim), table.table.data_ptr(), table.max_pos, int(pos0), q_out.data_ptr(),
        kv_out.data_ptr(), int(kv_row_stride if kv_row_stride is not None else row),
        _ptr(save_out), _stream(stream)), "rope_new")


def attn_workspace_bytes(n_cached: int, n_new: int, n_heads: int, head_dim: int,
                         num_splits: int = 0, n_kv_heads: int | None = None) -> int:
    if n_kv_heads is None:
        return int(lib().askv_attn_workspace_bytes(n_cached, n_new, n_heads, head_dim,
                                                   num_splits))
    return int(lib().askv_attn_workspace_bytes_gqa(n_cached, n_new, n_heads, n_kv_heads,
                                                   head_dim, num_splits))


def attn_num_splits(n_cached: int, n_new: int, n_heads: int, sm_count: int = 0,
                    n_kv_heads: int | None = None) -> int:
    if n_kv_heads is None or n_kv_heads == n_heads:
        return int(lib().askv_attn_num_splits(n_cached, n_new, n_heads, sm_count))
    return int(lib().askv_attn_num_splits_gqa(n_cached, n_new, n_heads, n_kv_heads, sm_count))


def prefill_attn(q: torch.Tensor, kv: torch.Tensor, n_cached: int, n_new: int, n_heads: int,
                 n_kv_heads: int, head_dim: int, out: torch.Tensor,
                 workspace: torch.Tensor | None = None, *, num_splits: int = 0,
                 kv_row_stride: int | None = None, scale: float | None = None,
                 stream=None) -> None:
    """K3: out[i,h] = softmax(q k^T/sqrt(d)) v over keys j <= n_cached + i."""
    _require_cuda(q, kv, out, workspace)
    row = 2 * n_kv_heads * head_dim
    ws_ptr = None if workspace is None else workspace.data_ptr()
    ws_bytes = 0 if workspace is None else workspace.numel() * workspace.element_size()
    check(lib().askv_prefill_attn(
        q.data_ptr(), kv.data_ptr(), int(kv_row_stride if kv_row_stride is not None else row),
        int(n_cached), int(n_new), int(n_heads), int(n_kv_heads), int(head_dim),
        float(scale if scale is not None else 1.0 / math.sqrt(head_dim)), out.data_ptr(),
        ws_ptr, int(ws_bytes), int(num_splits), _stream(stream)), "prefill_attn")


def _ids(block_ids):
    arr = np.ascontiguousarray(np.asarray(block_ids, dtype=np.int64))
    return arr, arr.ctypes.data_as(C.POINTER(C.c_int64))


def preload_layer(dst: torch.Tensor, host_base: torch.Tensor, block_ids, block_bytes: int,
                  layer_off: int, chunk_bytes: int, tail_bytes: int = 0, *,
                  stream=None) -> None:
    """K1: H2D of one layer's blocks into a contiguous HBM slot."""
    arr, p = _ids(block_ids)
    check(lib().askv_preload_layer(dst.data_ptr(), host_base.data_ptr(), p, len(arr),
                                   int(block_bytes), int(layer_off), int(chunk_bytes),
                                   int(tail_bytes), _stream(stream), None), "preload_layer")


def save_layer(host_base: torch.Tensor, block_ids, block_bytes: int, layer_off: int,
               block_tokens: int, row_bytes: int, first_token: int, n_tokens: int,
               src: torch.Tensor, *, stream=None) -> None:
    """K4: D2H of n_tokens rows into the session's host tail blocks."""
    arr, p = _ids(block_ids)
    check(lib().askv_save_layer(host_base.data_ptr(), p, len(arr), int(block_bytes),
                                int(layer_off), int(block_tokens), int(row_bytes),
                                int(first_token), int(n_tokens), src.data_ptr(),
                                _stream(stream), None), "save_layer")


def rmsnorm(x: torch.Tensor, w: torch.Tensor, eps: float = 1e-5, out=None, *, stream=None):
    """y = x * rsqrt(mean(x^2) + eps) * w over the last dim (bf16)."""
    _require_cuda(x, w)
    x = x.contiguous()
    out = torch.empty_like(x) if out is None else out
    rows = x.numel() // x.shape[-1]
    check(lib().askv_rmsnorm(x.data_ptr(), w.data_ptr(), out.data_ptr(), int(rows),
                             int(x.shape[-1]), float(eps), _stream(stream)), "rmsnorm")
    return out


def silu_mul(gu: torch.Tensor, out=None, *, stream=None):
    """silu(gu[:, :F]) * gu[:, F:] for gu = [rows, 2F] (bf16)."""
    _require_cuda(gu)
    rows, two_f = gu.shape
    ffn = two_f // 2
    out = torch.empty((rows, ffn), dtype=gu.dtype, device=gu.device) if out is None else out
    check(lib().askv_silu_mul(gu.data_ptr(), out.data_ptr(), int(rows), int(ffn),
                              _stream(stream)), "silu_mul")
    return out


def copy_sm(dst: torch.Tensor, src: torch.Tensor, *, stream=None) -> torch.Tensor:
    """dst <- src by SMs (pinned host <-> device via UVA), for few-KB transfers."""
    n = src.numel() * src.element_size()
    if dst.numel() * dst.element_size() < n:
        raise ValueError("copy_sm: destination too small")
    if not src.is_cuda and not src.is_pinned():
        raise ValueError("copy_sm: host source must be pinned")
    check(lib().askv_copy_sm(dst.data_ptr(), src.data_ptr(), int(n), _stream(stream)), "copy_sm")
    return dst


class NativeEvent:
    """A cudaEvent_t owned through the C ABI (recorded / waited by the native
    layer loop and the IO threads alike)."""

    __slots__ = ("handle", "_pool")

    def __init__(self, timing: bool = False, pool=None):
        h = C.c_void_p()
        check(lib().askv_event_create(C.byref(h), 1 if timing else 0), "event_create")
        self.handle = h.value
        self._pool = pool

    def record(self, stream) -> "NativeEvent":
        check(lib().askv_event_record(self.handle, stream.cuda_stream), "event_record")
        return self

    def wait(self, stream) -> None:
        """Make `stream` wait for this event."""
        check(lib().askv_stream_wait_event(stream.cuda_stream, self.handle), "stream_wait_event")

    def synchronize(self) -> None:
        """Block the host until the work recorded before this event is done."""
        check(lib().askv_event_synchronize(self.handle), "event_synchronize")

    def elapsed_ms(self, end: "NativeEvent") -> float:
        ms = C.c_float()
        check(lib().askv_event_elapsed_ms(self.handle, end.handle, C.byref(ms)), "elapsed_ms")
        return float(ms.value)

    elapsed_time = elapsed_ms   # torch.cuda.Event spelling

    def __del__(self):
        try:
            if self.handle:
                lib().askv_event_destroy(self.handle)
        except Exception:
            pass
