"""Multi-turn serving loop: the reference simulator's job start / finish
semantics driving the real B200 runner.

Reference call sites (sim.py):
  _start_job   :408-466  overflow truncation -> store lookup -> reuse or recompute
  _handle_overflow :468-483   drop `cut` tokens from the front until it fits
  _finish_job  :519-565  save-time truncation -> save (computed tokens)
  _truncate_tokens :576-581

Differences from the simulator, by design: time is real (CUDA events), the
KV bytes are real (pinned host arena blocks), and output tokens' KV — produced
by decode in a real server, which is outside the prefill hot path — is
produced here by a teacher-forced append prefill of the supplied output ids so
the next turn finds a complete history (SURVEY.md §7.2 "Output tokens' KV").
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import torch

from .model import LlamaShape, TierConfig, profile_for
from .policy import JobQueue, PolicyConfig, make_room, plan_prefetch
from .runner import Job, JobResult, LlamaWeights, ResidentKv, Runner
from .store import CapacityError, HitClass, HostArena, KvStore, Tier


def overflow_kept(hist: int, new: int, window: int, cut: int) -> int:
    """Kept history after load-time truncation, closed form of sim.py:471-474:
    the number of `cut` chunks dropped is ceil((hist + new - W) / cut)."""
    if hist + new <= window:
        return hist
    m = -(-(hist + new - window) // cut)
    return max(0, hist - m * cut)


def save_truncate(tokens: int, window: int, cut: int) -> int:
    """sim.py:576-581 in closed form."""
    if tokens <= window:
        return max(tokens, 0)
    return tokens - cut * (-(-(tokens - window) // cut))


def rolling_kept(kept: int, sizes, window: int, cut: int) -> int:
    """Context after appending chunks with a rolling window: before each chunk
    that would overflow, drop `cut`-sized front chunks (sim.py:468-483).  For
    chunk sizes <= min(cut, W - cut) this ends exactly at
    save_truncate(kept + sum(sizes)) (sim.py:576-581), which
    tests/test_store_cpu.py checks over ratios 0.1-0.9; a larger chunk can
    overflow by more than the save-time rule drops (ratio 0.75, chunk > W/4)."""
    for c in sizes:
        if kept + c > window:
            kept = overflow_kept(kept, c, window, cut)
        kept += c
    return kept


@dataclass
class TurnOutcome:
    session_id: str
    turn: int
    hit: str
    kept: int
    drop: int
    new: int
    prompt: int
    overflowed: bool
    result: JobResult                 # last chunk of the input prefill (first-token logits)
    append: JobResult | None          # last chunk of the teacher-forced output append
    results: list = field(default_factory=list)   # every input-prefill chunk (TTFT = sum)
    decode: list = field(default_factory=list)    # one JobResult per decoded token
    generated: torch.Tensor | None = None         # decoded token ids (host int64)

    def ttft_s(self) -> float:
        """Isolated time to first token: sum of the input chunks' makespans
        (call after Runner.finalize(outcome.results))."""
        return sum(r.timeline.makespan for r in self.results)


class HbmTier:
    """HBM-resident session tier (the reference's
    Mode.HBM_DRAM, sim.py:61, 102-108): an LRU cache of sessions' KV blocks in
    device memory that mirrors the host block tables one-to-one.  Host DRAM
    stays the backing store (saves are written through), so eviction from HBM
    is a table drop.  A turn whose session is HBM-resident re-embeds straight
    from HBM (no host link); otherwise its pre-loaded rows are promoted."""

    def __init__(self, n_blocks: int, block_bytes: int, device):
        from collections import OrderedDict, deque

        self.block_elems = block_bytes // 2
        self.arena = torch.empty(n_blocks * self.block_elems, dtype=torch.bfloat16,
                                 device=device)
        self.free = deque(range(n_blocks))
        # block -> session that held it last; a session that gets such a block
        # must order its writes after that session's in-flight saves (fence)
        self.prev_owner: dict[int, str] = {}
        self.fence: dict[str, set] = {}
        self.tab: dict[str, list[int]] = {}
        self.dropped: dict[str, int] = {}
        self.valid: set[str] = set()          # mirror holds every row the host holds
        self.lru: "OrderedDict[str, None]" = OrderedDict()
        self.device = device
        self.hits = 0
        self.promotions = 0

    def _release(self, sid: str, ids) -> None:
        for b in ids:
            self.prev_owner[b] = sid
        self.free.extend(ids)

    def _take(self, sid: str) -> int:
        b = self.free.popleft()
        prev = self.prev_owner.pop(b, None)
        if prev is not None and prev != sid:
            self.fence.setdefault(sid, set()).add(prev)
        return b

    def drop(self, sid: str) -> None:
        ids = self.tab.pop(sid, None)
        if ids:
            self._release(sid, ids)
        self.dropped.pop(sid, None)
        self.valid.discard(sid)
        self.lru.pop(sid, None)

    def sync(self, sid: str, host_tab: list[int] | None, host_dropped: int, pinned) -> bool:
        """Mirror the host table's front drops and growth; False if it cannot."""
        if host_tab is None:
            self.drop(sid)
            return False
        ids = self.tab.setdefault(sid, [])
        self.dropped.setdefault(sid, host_dropped)
        k = host_dropped - self.dropped[sid]
        if k > 0:
            self._release(sid, ids[:k])
            del ids[:k]
            self.dropped[sid] = host_dropped
        if len(ids) > len(host_tab):
            self._release(sid, ids[len(host_tab):])
            del ids[len(host_tab):]
        while len(ids) < len(host_tab):
            if not self.free and not self._evict(exclude=pinned | {sid}):
                self.drop(sid)
                return False
            ids.append(self._take(sid))
        self.lru[sid] = None
        self.lru.move_to_end(sid)
        return True

    def _evict(self, exclude) -> bool:
        for victim in self.lru:
            if victim not in exclude:
                self.drop(victim)
                return True
        return False

    def offsets(self, sid: str) -> torch.Tensor:
        return torch.as_tensor([b * self.block_elems for b in self.tab[sid]],
                               dtype=torch.int64, device=self.device)


class Engine:
    """One GPU's serving loop for the reuse path.  Prefills are processed in
    chunks of at most `chunk` = min(max_new, cut, W - cut) tokens (chunked prefill: a
    chunk after the first reuses the rows its predecessor just saved), with the
    reference's window truncation applied before any chunk that would overflow,
    so positions never exceed the window."""

    def __init__(self, shape: LlamaShape, *, host_blocks: int, block_tokens: int = 128,
                 device="cuda", seed: int = 0, weights: LlamaWeights | None = None,
                 read_buffer_bytes: int = 1 << 30, max_new: int = 1024,
                 truncation_ratio: float = 0.5, ttl: float = math.inf, pin: bool = True,
                 tp_reduce=None, hbm_blocks: int = 0, disk_dir: str | None = None,
                 disk_blocks: int = 0, autotune: bool | int = True,
                 policy: PolicyConfig | None = None, dram_bytes: int | None = None,
                 numa_node: int | None = None):
        self.shape = shape
        # placement policy (policy.py:92-204): the reference's scheduler-aware
        # ranking over `queue` (the serving loop's JobQueue when one drives this
        # engine, sim.Server; empty otherwise = coldest first)
        self.policy = policy if policy is not None else PolicyConfig()
        self.queue = JobQueue()
        self.profile = profile_for(shape, truncation_ratio=truncation_ratio)
        self.block_tokens = block_tokens
        block_bytes = block_tokens * shape.kv_bytes_per_token
        self.arena = HostArena(host_blocks, block_bytes, pin=pin, numa_node=numa_node)
        disk = None
        if disk_dir is not None and disk_blocks > 0:
            from .disk import DiskTier
            disk = DiskTier(disk_dir, block_bytes)
        # accounting capacity: the arena, or less (`dram_bytes`) so the
        # physical spare covers the rows of the jobs in flight
        dram = host_blocks * block_bytes if dram_bytes is None else min(
            int(dram_bytes), host_blocks * block_bytes)
        tiers = TierConfig(dram_capacity=dram,
                           disk_capacity=disk_blocks * block_bytes if disk else 0)
        self.store = KvStore(self.profile, tiers, block_bytes=block_bytes, ttl=ttl,
                             evictor=self._make_room, arena=self.arena,
                             block_tokens=block_tokens, disk=disk)
        self.disk_evictions = 0
        self.disk_promotions = 0
        self.last_disk_wait_s = 0.0
        self.prefetched: set[str] = set()
        self.window = shape.context_window
        self.cut = self.profile.cut_tokens
        # chunks <= min(cut, W - cut) keep the rolling window equal to the
        # reference's save-time truncation for every ratio (rolling_kept)
        self.chunk = max(1, min(max_new, self.cut, self.window - self.cut))
        self.hbm = HbmTier(hbm_blocks, block_bytes, device) if hbm_blocks > 0 else None
        self.runner = Runner(shape, weights=weights, device=device, seed=seed,
                             block_tokens=block_tokens, host_arena=self.arena,
                             hbm_arena=self.hbm.arena if self.hbm else None,
                             read_buffer_bytes=read_buffer_bytes, max_new=max_new,
                             max_ctx=self.window + self.chunk, tp_reduce=tp_reduce,
                             # tune the GEMMs over full prompts too (misses recompute them)
                             autotune=(self.window + self.chunk + max_new
                                       if autotune is True else autotune))
        self.store.io_fence = self.runner.fence
        if self.hbm is not None:
            # any physical release / demotion of a session's host rows ends
            # its HBM mirror (the mirror is only valid against those rows)
            self.store.on_release = self.hbm.drop
        self.context: dict[str, int] = {}
        self.tokens: dict[str, torch.Tensor] = {}   # conversation token ids (for misses)

    def _make_room(self, needed: float) -> None:
        """Free DRAM with the reference's placement policy (sim.py:298-327 via
        policy.make_room): victims ranked by the scheduler-aware key over
        `self.queue` (policy.py:159-172), demoted to the disk tier when there is
        one (dropping disk victims while it is full), else evicted out."""
        def count(action, sid, nbytes, counted):
            if action == "evict_to_disk":
                self.disk_evictions += 1

        make_room(self.store, self.queue, self.policy, needed, on_evict=count)

    def _ensure_arena(self, sid: str, rows: int) -> None:
        """Physical room for the session's rows before the saver writes them
        (the accounting follows at save()): demote / evict LRU sessions."""
        st = self.store
        need = -(-(st.head_row(sid) + rows) // self.block_tokens) - len(st.tables.get(sid, ()))
        while st.arena.free_blocks < need:
            before = st.arena.free_blocks
            # the store's evictor: this engine's policy, or the serving loop's
            # when one drives the engine (sim.Server installs its own)
            (st.evictor or self._make_room)((need - before) * st.block_bytes)
            if st.arena.free_blocks == before:
                raise CapacityError(f"host arena full: {need} blocks for {sid}")

    def _admit(self, sid: str, turn_index: int, kept: int, now: float) -> HitClass:
        """Store lookup at job start (sim.py:419-431).  A disk hit is promoted
        to DRAM first (read from its file into arena blocks, unless a prefetch
        already brought it in); the turn then takes the normal pre-load path."""
        hit = HitClass.MISS
        if turn_index > 0:
            hit = self.store.lookup(sid, now)
            if hit is not HitClass.MISS and self.store.peek(sid).tokens != kept:
                self.store.remove(sid)
                hit = HitClass.MISS
        self.store.pinned.add(sid)
        self.prefetched.discard(sid)
        t0 = time.perf_counter()
        if hit is HitClass.DISK_HIT and self.store.disk is not None:
            self._promote(sid, wait=True)
        elif sid in self.store.pending:
            self.store.wait(sid)      # prefetched: only the rest of the read is exposed
        self.last_disk_wait_s = time.perf_counter() - t0
        return hit

    def _promote(self, sid: str, wait: bool) -> None:
        it = self.store.peek(sid)
        blocks = self.store.charge(it.bytes)
        target = blocks + self.store.mem_buffer_reserve
        if self.store.mem_free < target:
            (self.store.evictor or self._make_room)(target - self.store.mem_free)
        self.store.move(sid, Tier.MEMORY, wait=wait)
        self.disk_promotions += 1

    def prefetch(self, sids=None) -> list[str]:
        """Scheduler-aware prefetch (policy.py:122-150, sim.py:329-366): start
        disk -> DRAM reads for the sessions of upcoming jobs; the reads run on
        the disk IO threads while the current prefill proceeds.  `sids` None =
        the reference's pick over `self.queue` (plan_prefetch)."""
        if sids is None:
            sids = plan_prefetch(self.queue, self.store, self.policy, exclude=self.prefetched)
        started = []
        for sid in sids:
            it = self.store.peek(sid)
            if it is None or it.tier is not Tier.DISK or self.store.disk is None:
                continue
            self.store.pinned.add(sid)       # not a victim of its own room-making
            try:
                self._promote(sid, wait=False)
                self.prefetched.add(sid)
                started.append(sid)
            except CapacityError:
                pass
            finally:
                self.store.pinned.discard(sid)
        return started

    def _hbm_sync(self, sid: str) -> bool:
        if self.hbm is None:
            return False
        ok = self.hbm.sync(sid, self.store.tables.get(sid), self.store.dropped.get(sid, 0),
                           self.store.pinned)
        return ok

    def install_history(self, sid: str, ids: torch.Tensor, now: float = 0.0) -> JobResult:
        """Prefill and store a session history as-is (one job, no truncation):
        a pre-stored long document / history larger than the window, the
        starting point of config C4 (32K history served at W = 4096)."""
        ids = ids.reshape(-1).to(torch.int64)
        n = int(ids.numel())
        if self.store.peek(sid) is not None:
            self.store.remove(sid)
        if self.hbm is not None:
            self.hbm.drop(sid)        # the rows are rewritten: a mirror would be stale
        tab = self.store.reserve_rows(sid, n)
        res = self.runner.run([Job(sid, ids, kept=0, source="none", block_ids=tab, save=True,
                                   head=self.store.head_row(sid))])[0]
        self.store.mark_written(sid, n)
        self.store.save(sid, n, now)
        self.context[sid] = n
        self.tokens[sid] = ids
        return res

    def _prefill(self, sid: str, ids: torch.Tensor, kept: int, want_logits: bool,
                 kv_cache: ResidentKv | None = None, prestage_layers: int = 0):
        """Chunked prefill of `ids` after `kept` stored rows, saving every chunk's
        K/V; rolling window truncation before a chunk that would overflow.
        With `kv_cache` the last chunk leaves every layer's rotated rows resident
        in it (and reuses them when the cache already holds the kept rows).
        Returns (results, kept_after, rows_dropped)."""
        results, dropped = [], 0
        pos, n = 0, int(ids.numel())
        while pos < n:
            c = min(self.chunk, n - pos)
            if kept + n - pos <= self.window and n - pos <= self.runner.max_new:
                c = n - pos   # no overflow possible: one job (same rows as chunking)
            if kept + c > self.window:
                k2 = overflow_kept(kept, c, self.window, self.cut)
                self.store.drop_front_rows(sid, kept - k2)
                dropped += kept - k2
                kept = k2
                if kv_cache is not None:
                    kv_cache.rows = 0          # positions shifted: re-embed from the store
            self._ensure_arena(sid, kept + c)
            tab = self.store.reserve_rows(sid, kept + c)
            job = Job(sid, ids[pos:pos + c], kept=kept, source="host" if kept else "none",
                      block_ids=tab, save=True, head=self.store.head_row(sid),
                      prestage_layers=prestage_layers if pos == 0 else 0)
            if kv_cache is not None and pos + c == n:
                job.kv_cache = kv_cache
                if kept and kv_cache.rows == kept:
                    job.source = "resident"    # rows already rotated in HBM (decode)
            if self.hbm is not None:
                resident = sid in self.hbm.valid
                if self._hbm_sync(sid):
                    hids = list(self.hbm.tab[sid])
                    job.mirror_block_ids = hids
                    job.fence_sessions = self.hbm.fence.pop(sid, set())
                    if job.source == "resident":
                        pass
                    elif kept and resident:
                        job.source = "hbm"        # no host link for this chunk
                        job.dev_block_off = self.hbm.offsets(sid)
                        self.hbm.hits += 1
                    elif kept:
                        job.promote_block_ids = hids
                        self.hbm.promotions += 1
                    self.hbm.valid.add(sid)
            results.append(self.runner.run([job], want_logits=want_logits)[0])
            kept += c
            self.store.mark_written(sid, kept)
            pos += c
        return results, kept, dropped

    def turn(self, sid: str, turn_index: int, new_ids: torch.Tensor,
             out_ids: torch.Tensor | None = None, now: float = 0.0,
             want_logits: bool = False) -> TurnOutcome:
        new_ids = new_ids.reshape(-1).to(torch.int64)
        out_ids = None if out_ids is None else out_ids.reshape(-1).to(torch.int64)
        hist = self.context.get(sid, 0)
        new = int(new_ids.numel())
        overflowed = hist + new > self.window
        kept = hist
        if overflowed:
            kept = overflow_kept(hist, new, self.window, self.cut)
            if self.store.peek(sid) is not None:
                if kept == 0:
                    self.store.remove(sid)
                else:
                    self.store.truncate_item(sid, kept, now)
            self.context[sid] = kept
            if sid in self.tokens:
                self.tokens[sid] = self.tokens[sid][hist - kept:]
        hit = self._admit(sid, turn_index, kept, now)
        hist_ids = self.tokens.get(sid, torch.empty(0, dtype=torch.int64))
        if hit is HitClass.MISS or kept == 0:
            hit = HitClass.MISS
            if self.store.peek(sid) is None:
                self.store.release_rows(sid)
            if self.hbm is not None:
                self.hbm.drop(sid)
            # recompute the whole (truncated) prompt, sim.py:432-435
            results, rows, _ = self._prefill(sid, torch.cat([hist_ids, new_ids]), 0,
                                             want_logits)
        else:
            results, rows, _ = self._prefill(sid, new_ids, kept, want_logits)
        append = None
        if out_ids is not None and out_ids.numel():
            ares, rows, _ = self._prefill(sid, out_ids, rows, False)
            append = ares[-1]
        n_out = 0 if out_ids is None else int(out_ids.numel())
        raw = kept + new + n_out
        ctx = save_truncate(raw, self.window, self.cut)
        if ctx != rows:
            raise AssertionError(f"rolling window {rows} != save truncation {ctx}")
        all_ids = torch.cat([hist_ids, new_ids] + ([out_ids] if n_out else []))
        self.tokens[sid] = all_ids[raw - ctx:]
        self.context[sid] = ctx
        if ctx > 0:
            self.store.save(sid, ctx, now)
        self._hbm_sync(sid)
        self.store.pinned.discard(sid)
        return TurnOutcome(sid, turn_index, hit.value, kept, hist - kept, new, kept + new,
                           overflowed, results[-1], append, results)

    def generate(self, sid: str, turn_index: int, new_ids: torch.Tensor, steps: int, *,
                 out_ids: torch.Tensor | None = None, now: float = 0.0,
                 want_logits: bool = False) -> TurnOutcome:
        """One turn with a real decode phase: the prompt
        goes through the reuse prefill, then `steps` tokens are decoded one at a
        time with every layer's rotated K|V resident in HBM (no re-embed per
        step); each step's new K|V row is saved to the session's blocks on the
        save stream while the next step runs — the decode branch of
        plan_async_save (overlap.py:126-200; sim.py:491-501, 528).  Greedy
        (argmax, chained on the device) unless `out_ids` teacher-forces the
        tokens fed at each step.  Store bookkeeping as in `turn` (the outputs
        are appended to the history, save-time truncation sim.py:576-581)."""
        if steps < 1:
            return self.turn(sid, turn_index, new_ids, None, now, want_logits)
        if out_ids is not None and int(out_ids.numel()) < steps:
            raise ValueError("out_ids must cover every decode step")
        cap = self.window + self.chunk
        if getattr(self, "_kv", None) is None or self._kv.capacity < cap:
            self._kv = ResidentKv(self.shape, cap, self.runner.device)
        kv = self._kv
        kv.rows = 0
        new_ids = new_ids.reshape(-1).to(torch.int64)
        hist = self.context.get(sid, 0)
        new = int(new_ids.numel())
        overflowed = hist + new > self.window
        kept = hist
        if overflowed:
            kept = overflow_kept(hist, new, self.window, self.cut)
            if self.store.peek(sid) is not None:
                if kept == 0:
                    self.store.remove(sid)
                else:
                    self.store.truncate_item(sid, kept, now)
            self.context[sid] = kept
            if sid in self.tokens:
                self.tokens[sid] = self.tokens[sid][hist - kept:]
        hit = self._admit(sid, turn_index, kept, now)
        hist_ids = self.tokens.get(sid, torch.empty(0, dtype=torch.int64))
        if hit is HitClass.MISS or kept == 0:
            hit = HitClass.MISS
            if self.store.peek(sid) is None:
                self.store.release_rows(sid)
            if self.hbm is not None:
                self.hbm.drop(sid)
            results, rows, _ = self._prefill(sid, torch.cat([hist_ids, new_ids]), 0,
                                             want_logits, kv_cache=kv)
        else:
            results, rows, _ = self._prefill(sid, new_ids, kept, want_logits, kv_cache=kv)
        dev = self.runner.device
        tok = (out_ids.reshape(-1)[:1].to(dev) if out_ids is not None
               else results[-1].next_token)
        fed, decode = [], []
        for s in range(steps):
            fed.append(tok)
            res, rows, _ = self._prefill(sid, tok.reshape(1), rows, want_logits, kv_cache=kv)
            decode.append(res[-1])
            if s + 1 < steps:
                tok = (out_ids.reshape(-1)[s + 1:s + 2].to(dev) if out_ids is not None
                       else res[-1].next_token)
        gen = torch.cat([t.reshape(1) for t in fed]).cpu()
        raw = kept + new + steps
        ctx = save_truncate(raw, self.window, self.cut)
        if ctx != rows:
            raise AssertionError(f"rolling window {rows} != save truncation {ctx}")
        all_ids = torch.cat([hist_ids, new_ids, gen])
        self.tokens[sid] = all_ids[raw - ctx:]
        self.context[sid] = ctx
        if ctx > 0:
            self.store.save(sid, ctx, now)
        self._hbm_sync(sid)
        self.store.pinned.discard(sid)
        return TurnOutcome(sid, turn_index, hit.value, kept, hist - kept, new, kept + new,
                           overflowed, results[-1], None, results, decode, gen)

