"""GPU-backed mirror of the reference numeric API (kvsim.rope).

Same names, argument meaning and error behaviour as
/root/reference/pkg/src/kvsim/rope.py, computed by the sm_100a kernels in
libaskv.so on bf16 CUDA tensors (the reference computes in float64 numpy;
parity tolerances are stated in DESIGN.md and tests/test_rope_gpu.py):

  KvRecord(keys, values)                  rope.py:25-52
  rotate_matrix(x, positions, theta)      rope.py:63-74
  rope_rotate(vec, position, theta)       rope.py:77-85
  attention_with_decoupled_cache(...)     rope.py:118-144

Extensions: keys/values/q may carry a head axis -- (S, H, d) / (N, Hq, d) --
with grouped-query sharing (Hq a multiple of Hkv); an empty record is plain
causal prefill (the reference crashes on it, rope.py:69; SPEC.md:451 says it is
valid).  head_dim must be 64 or 128 (the kernels' tile shapes).
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import ops

DEFAULT_THETA_BASE = 10000.0
SUPPORTED_HEAD_DIMS = (64, 128)


def _as_bf16(x, device="cuda") -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=device, dtype=torch.bfloat16)
    return torch.as_tensor(np.asarray(x, dtype=np.float32), device=device).to(torch.bfloat16)


def _check_dim(d: int) -> None:
    if d % 2 != 0:
        raise ValueError("head_dim must be even")
    if d not in SUPPORTED_HEAD_DIMS:
        raise ValueError(f"head_dim {d} unsupported on the B200 path (64 or 128)")


class KvRecord:
    """Cached keys/values of one sequence, stored pre-rotation (rope.py:25-52).

    Physically one bf16 tensor ``rows`` of shape (seq_len, 2, H, d) -- the
    K|V row layout of the host blocks -- with ``keys``/``values`` as views.
    """

    def __init__(self, keys, values):
        k = _as_bf16(keys)
        v = _as_bf16(values, k.device)
        if k.dim() == 2:
            k = k.unsqueeze(1)
            v = v.unsqueeze(1) if v.dim() == 2 else v
            self._squeeze = True
        else:
            self._squeeze = False
        if k.dim() != 3 or v.shape != k.shape:
            raise ValueError("keys and values must be matching 2-D arrays")
        if k.shape[-1] % 2 != 0:
            raise ValueError("head_dim must be even")
        self.rows = torch.stack([k, v], dim=1).contiguous()

    @classmethod
    def from_rows(cls, rows: torch.Tensor, squeeze: bool = False) -> "KvRecord":
        rec = cls.__new__(cls)
        rec.rows = rows
        rec._squeeze = squeeze
        return rec

    @property
    def keys(self) -> torch.Tensor:
        k = self.rows[:, 0]
        return k[:, 0] if self._squeeze else k

    @property
    def values(self) -> torch.Tensor:
        v = self.rows[:, 1]
        return v[:, 0] if self._squeeze else v

    @property
    def seq_len(self) -> int:
        return self.rows.shape[0]

    @property
    def head_dim(self) -> int:
        return self.rows.shape[-1]

    @property
    def n_heads(self) -> int:
        return self.rows.shape[2]

    def truncated(self, start: int, end: int) -> "KvRecord":
        """Keep rows [start:end) (rope.py:48-52); always a copy."""
        if not 0 <= start <= end <= self.seq_len:
            raise ValueError("bad keep range")
        return KvRecord.from_rows(self.rows[start:end].clone(), self._squeeze)


def _positions_tensor(positions, n: int, device) -> torch.Tensor:
    pos = np.asarray(positions, dtype=np.int64).reshape(-1)
    if pos.shape[0] != n:
        raise ValueError(f"positions length {pos.shape[0]} != {n}")
    if n and pos.min() < 0:
        raise ValueError("position must be >= 0")
    return torch.as_tensor(pos.astype(np.int32), device=device)


def rotate_matrix(x, positions, theta_base: float = DEFAULT_THETA_BASE) -> torch.Tensor:
    """Rotate each row of x ((S, d) or (S, H, d)) by its position (rope.py:63-74)."""
    x = _as_bf16(x)
    squeeze = x.dim() == 2
    x3 = x.unsqueeze(1) if squeeze else x
    s, h, d = x3.shape
    _check_dim(d)
    pos = _positions_tensor(positions, s, x.device)
    out = torch.empty_like(x3)
    if s:
        table = ops.rope_table(int(pos.max().item()) + 1, d, theta_base, x.device)
        ops.rotate_rows(x3.contiguous().view(s, h * d), h, d, table, out.view(s, h * d),
                        positions=pos)
    return out[:, 0] if squeeze else out


def rope_rotate(vec, position: int, theta_base: float = DEFAULT_THETA_BASE) -> torch.Tensor:
    """Rotate one head vector to `position` (rope.py:77-85)."""
    if position < 0:
        raise ValueError("position must be >= 0")
    v = _as_bf16(vec)
    if v.dim() != 1:
        raise ValueError("expected a 1-D head vector")
    return rotate_matrix(v[None, :], [position], theta_base)[0]


def attention_with_decoupled_cache(record: KvRecord, new_q, new_k, new_v, positions,
                                   theta_base: float = DEFAULT_THETA_BASE, *,
                                   num_splits: int = 0) -> torch.Tensor:
    """Attention of new tokens over a cache re-embedded at `positions`
    (rope.py:118-144).  New tokens take positions[-1]+1 .. (0.. when empty)."""
    q = _as_bf16(new_q)
    k = _as_bf16(new_k)
    v = _as_bf16(new_v)
    squeeze = q.dim() == 2
    if squeeze:
        q, k, v = q.unsqueeze(1), k.unsqueeze(1), v.unsqueeze(1)
    n, hq, d = q.shape
    hkv = k.shape[1]
    if k.shape != (n, hkv, d) or v.shape != k.shape:
        raise ValueError("new_q/new_k/new_v shapes disagree")
    if record.seq_len and (record.n_heads != hkv or record.head_dim != d):
        raise ValueError("record heads/head_dim disagree with new tokens")
    if hq % hkv:
        raise ValueError("query heads must be a multiple of kv heads")
    _check_dim(d)
    s = record.seq_len
    pos = np.asarray(positions, dtype=np.int64).reshape(-1)
    if pos.shape[0] != s:
        raise ValueError(f"positions length {pos.shape[0]} != cached length {s}")
    next_pos = int(pos[-1]) + 1 if s else 0
    dev = q.device
    table = ops.rope_table(max(next_pos + n, int(pos.max()) + 1 if s else 1), d, theta_base, dev)
    kv = torch.empty((s + n, 2, hkv, d), dtype=torch.bfloat16, device=dev)
    if s:
        ops.reembed(record.rows.to(dev), s, hkv, d, table, kv,
                    positions=_positions_tensor(pos, s, dev))
    qkv = torch.cat([q.reshape(n, hq * d), k.reshape(n, hkv * d), v.reshape(n, hkv * d)], dim=1)
    q_rot = torch.empty((n, hq, d), dtype=torch.bfloat16, device=dev)
    ops.rope_new(qkv, n, hq, hkv, d, table, next_pos, q_rot, kv[s:])
    out = torch.empty((n, hq, d), dtype=torch.bfloat16, device=dev)
    splits = num_splits or ops.attn_num_splits(s, n, hq, n_kv_heads=hkv)
    ws = None
    nbytes = ops.attn_workspace_bytes(s, n, hq, d, splits, n_kv_heads=hkv)
    if nbytes:
        ws = torch.empty(nbytes, dtype=torch.uint8, device=dev)
    ops.prefill_attn(q_rot, kv, s, n, hq, hkv, d, out, ws, num_splits=splits,
                     scale=1.0 / math.sqrt(d))
    return out[:, 0] if squeeze else out
