"""Multi-GPU plumbing for the KV-reuse path: one process per GPU.

Sessions are independent on this path: a session's KV,
truncation and prefill touch only that session, so ranks take disjoint session
shards by a stable hash and run with no collective on the data path.  The only
cross-rank traffic is the benchmark's max-over-ranks timing and token totals.
(The 70B TP=8 output-projection all-reduce of config C5 is the one real
collective in the north star; it is not on this module's path.)
"""

from __future__ import annotations

import os
import zlib

import torch
import torch.distributed as dist


def shard_of(session_id: str, world: int) -> int:
    """Stable owner rank of a session (crc32; identical on every rank/host)."""
    return zlib.crc32(session_id.encode()) % world


def shard(session_ids, rank: int, world: int) -> list:
    return [s for s in session_ids if shard_of(s, world) == rank]


def env_rank_world() -> tuple[int, int, int]:
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def init(backend: str, device: torch.device | None = None) -> None:
    """Initialise the default group from torchrun's env (127.0.0.1 rendezvous)."""
    if dist.is_initialized():
        return
    kw = {"device_id": device} if (backend == "nccl" and device is not None) else {}
    dist.init_process_group(backend, **kw)


def _reduce(x: float, op, device) -> float:
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=op)
    return float(t.item())


def max_over_ranks(x: float, device=None) -> float:
    return _reduce(x, dist.ReduceOp.MAX, device or "cpu")


def sum_over_ranks(x: float, device=None) -> float:
    return _reduce(x, dist.ReduceOp.SUM, device or "cpu")
