"""Physical disk tier behind ``KvStore.move``.

The reference's third storage level (§3.1, 3.3; store.py Tier.DISK,
sim.py:300-366 evict-to-disk / scheduler-aware prefetch, policy.py:122-150) is
accounting-only there: an item on disk is charged the disk bandwidth when it is
loaded.  Here an item moved to disk really leaves the pinned host arena: its
blocks are written, in block-table order, to one file per session, and the
arena blocks are freed; moving it back allocates blocks and reads the file into
them.  The path is disk -> pinned DRAM -> (K1) HBM, as in the paper.

IO runs on a pool of IO threads (the paper's dedicated IO threads):
each block is split into ``chunk_bytes`` pieces issued as positional reads /
writes (``os.preadv`` / ``os.pwritev`` release the GIL), with ``O_DIRECT`` when
the file system and the buffer alignment allow it (page-aligned pinned blocks of
a multiple of 4 KiB), so the copy does not go through the page cache.
Truncation of an item on disk is a front-offset edit of its file (no IO).
"""

from __future__ import annotations

import hashlib
import os
import threading
import time
from concurrent.futures import Future, ThreadPoolExecutor
from dataclasses import dataclass

_ALIGN = 4096


@dataclass
class DiskMeta:
    nblocks: int      # blocks held in the file, starting at `first`
    first: int        # index of the first live block in the file (front drops)
    head: int         # first valid row inside the first live block
    valid: int        # valid rows
    dropped: int      # front blocks released so far (mirrors KvStore.dropped)


class DiskTier:
    """One file per session under `directory`; block-granular IO."""

    def __init__(self, directory: str, block_bytes: int, *, io_threads: int = 8,
                 chunk_bytes: int = 8 << 20, direct: bool = True):
        os.makedirs(directory, exist_ok=True)
        self.dir = directory
        self.block_bytes = int(block_bytes)
        self.chunk_bytes = int(chunk_bytes)
        self.pool = ThreadPoolExecutor(max_workers=io_threads, thread_name_prefix="askv-disk")
        self.meta: dict[str, DiskMeta] = {}
        self.direct = direct and hasattr(os, "O_DIRECT")
        self._lock = threading.Lock()
        self.bytes_written = 0
        self.bytes_read = 0
        self.write_seconds = 0.0
        self.read_seconds = 0.0

    # ---------------------------------------------------------------- helpers
    def path(self, sid: str) -> str:
        return os.path.join(self.dir, hashlib.sha1(sid.encode()).hexdigest()[:20] + ".kv")

    def _open(self, path: str, flags: int, buf_addr: int) -> int:
        aligned = (buf_addr % _ALIGN == 0 and self.block_bytes % _ALIGN == 0
                   and self.chunk_bytes % _ALIGN == 0)
        if self.direct and aligned:
            try:
                return os.open(path, flags | os.O_DIRECT, 0o600)
            except OSError:            # e.g. tmpfs: no O_DIRECT
                pass
        return os.open(path, flags, 0o600)

    def _pieces(self, table, base_off):
        """(arena offset, file offset, length) pieces of the given blocks."""
        out = []
        for i, b in enumerate(table):
            for c in range(0, self.block_bytes, self.chunk_bytes):
                n = min(self.chunk_bytes, self.block_bytes - c)
                out.append((b * self.block_bytes + c, (base_off + i) * self.block_bytes + c, n))
        return out

    # ---------------------------------------------------------------- API
    def write(self, sid: str, arena, table: list[int], head: int, valid: int,
              dropped: int) -> Future:
        """Write the session's blocks (arena block ids `table`) to its file."""
        buf = arena.buffer.numpy()
        path = self.path(sid)
        fd = self._open(path, os.O_WRONLY | os.O_CREAT | os.O_TRUNC, arena.buffer.data_ptr())
        pieces = self._pieces(table, 0)
        t0 = time.perf_counter()

        def one(p):
            a, f, n = p
            mv = memoryview(buf[a:a + n])
            done = 0
            while done < n:
                done += os.pwritev(fd, [mv[done:]], f + done)

        futs = [self.pool.submit(one, p) for p in pieces]
        out: Future = Future()

        def finish():
            try:
                for f in futs:
                    f.result()
                os.close(fd)
                with self._lock:
                    self.meta[sid] = DiskMeta(len(table), 0, head, valid, dropped)
                    self.bytes_written += len(table) * self.block_bytes
                    self.write_seconds += time.perf_counter() - t0
                out.set_result(len(table) * self.block_bytes)
            except BaseException as exc:   # surfaced to the caller
                out.set_exception(exc)

        threading.Thread(target=finish, daemon=True).start()
        return out

    def read(self, sid: str, arena, table: list[int]) -> Future:
        """Read the session's live blocks into arena blocks `table` (allocated
        by the caller, len(table) == meta.nblocks)."""
        m = self.meta[sid]
        if len(table) != m.nblocks:
            raise ValueError(f"read of {sid}: {len(table)} blocks for {m.nblocks} on disk")
        buf = arena.buffer.numpy()
        fd = self._open(self.path(sid), os.O_RDONLY, arena.buffer.data_ptr())
        pieces = self._pieces(table, m.first)
        t0 = time.perf_counter()

        def one(p):
            a, f, n = p
            mv = memoryview(buf[a:a + n])
            done = 0
            while done < n:
                r = os.preadv(fd, [mv[done:]], f + done)
                if r <= 0:
                    raise IOError(f"short read of {sid}")
                done += r

        futs = [self.pool.submit(one, p) for p in pieces]
        out: Future = Future()

        def finish():
            try:
                for f in futs:
                    f.result()
                os.close(fd)
                with self._lock:
                    self.bytes_read += len(table) * self.block_bytes
                    self.read_seconds += time.perf_counter() - t0
                out.set_result(len(table) * self.block_bytes)
            except BaseException as exc:
                out.set_exception(exc)

        threading.Thread(target=finish, daemon=True).start()
        return out

    def drop_front_rows(self, sid: str, drop: int, block_tokens: int) -> None:
        """Truncate an item on disk: keep its most recent rows (a front-offset
        edit of the file, no IO)."""
        m = self.meta[sid]
        total = m.head + drop
        nb = total // block_tokens
        m.first += nb
        m.nblocks -= nb
        m.dropped += nb
        m.head = total - nb * block_tokens
        m.valid = max(0, m.valid - drop)

    def trim_blocks(self, sid: str, keep: int) -> None:
        m = self.meta[sid]
        m.nblocks = min(m.nblocks, keep)

    def delete(self, sid: str) -> None:
        with self._lock:
            self.meta.pop(sid, None)
        try:
            os.unlink(self.path(sid))
        except FileNotFoundError:
            pass

    def close(self) -> None:
        self.pool.shutdown(wait=True)
