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


class NcclComm:
    """This rank's NCCL communicator over the tensor-parallel group, handed to
    the native layer loop (askv_prefill_plan.nccl_comm): the W_o / W_down
    all-reduces are issued from C++ on the compute stream and captured into
    the layer graph -- no host callback per call (config C5).
    Rank 0 draws the ncclUniqueId; it reaches the others through the default
    torch.distributed group (any backend) unless `unique_id` is given."""

    def __init__(self, rank: int, world: int, *, unique_id: bytes | None = None, group=None):
        import ctypes as C

        from . import _lib

        lib = _lib.lib()
        self.rank, self.world = int(rank), int(world)
        if unique_id is None:
            buf = (C.c_char * 128)()
            if self.rank == 0:
                _lib.check(lib.askv_nccl_unique_id(buf), "nccl_unique_id")
            uid = [bytes(buf)]
            if self.world > 1:
                dist.broadcast_object_list(uid, src=0, group=group)
            unique_id = uid[0]
        if len(unique_id) != 128:
            raise ValueError("ncclUniqueId is 128 bytes")
        self._id = (C.c_char * 128).from_buffer_copy(unique_id)
        h = C.c_void_p()
        _lib.check(lib.askv_nccl_comm_init(self.world, self.rank, self._id, C.byref(h)),
                   "nccl_comm_init")
        self.handle = h.value
        self.native_comm = self

    def __call__(self, t: torch.Tensor, stream) -> None:
        """In-place bf16 sum of `t` over the group on `stream`."""
        from . import _lib

        if t.dtype != torch.bfloat16 or not t.is_contiguous():
            raise ValueError("NcclComm sums contiguous bf16 tensors")
        _lib.check(_lib.lib().askv_nccl_allreduce_bf16(t.data_ptr(), t.data_ptr(), t.numel(),
                                                       self.handle, stream.cuda_stream),
                   "nccl_allreduce")

    def close(self) -> None:
        from . import _lib

        if self.handle:
            _lib.check(_lib.lib().askv_nccl_comm_destroy(self.handle), "nccl_comm_destroy")
            self.handle = None


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
