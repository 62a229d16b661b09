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


class NcclAllReduce:
    """tp_reduce hook for a real TP group: in-place sum over the default group
    (NCCL over NVLink / NVSwitch), ordered on the runner's compute stream."""

    def __init__(self, group=None):
        self.group = group

    def __call__(self, t: torch.Tensor, stream) -> None:
        with torch.cuda.stream(stream):
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)


class ThreadAllReduce:
    """tp_reduce hook for a 1-GPU emulation of a TP group: one Python thread per
    rank, each driving its own Runner/streams; partials are summed on the GPU
    in a fixed rank order (deterministic) and copied back in place."""

    def __init__(self, world: int):
        import threading

        self.world = world
        self._bar = threading.Barrier(world)
        self._slots: list = [None] * world
        self._done = None

    def bind(self, rank: int):
        return lambda t, stream: self._reduce(rank, t, stream)

    def _reduce(self, rank: int, t: torch.Tensor, stream) -> None:
        ev = torch.cuda.Event()
        ev.record(stream)
        self._slots[rank] = (t, ev, stream)
        self._bar.wait()
        if rank == 0:
            with torch.cuda.stream(stream):
                for _, e, _ in self._slots:
                    stream.wait_event(e)
                acc = self._slots[0][0].float()
                for r in range(1, self.world):
                    acc += self._slots[r][0].float()
                total = acc.to(t.dtype)
                done = torch.cuda.Event()
                done.record(stream)
            for _, _, s in self._slots[1:]:
                total.record_stream(s)   # other ranks read it on their streams
            self._done = (total, done)
        self._bar.wait()
        total, done = self._done
        stream.wait_event(done)
        with torch.cuda.stream(stream):
            t.copy_(total)
        self._bar.wait()
