"""Measured timing: the reference's ``overlap.plan_preload`` /
``plan_async_save`` executed on the real B200 engine (SURVEY.md §8(b) item 2,
§8(f) row 3).

The reference plans a job's load / compute / save schedule analytically
(/root/reference/pkg/src/kvsim/overlap.py:69-123, :126-200) and its simulator
charges ``Timeline.makespan`` as the prefill time and ``stall_total`` as the
exposed transfer (sim.py:432-449, :533-542).  ``MeasuredExecutor`` has the
same two calls with the same arguments and return type, but each call *runs*
the job -- K1 pre-load of the session's kept rows over the host link, K2
re-embed, K3 attention, the projections, K4 save -- and returns the Timeline
measured on the device (device timestamps on the compute stream, timing
events on the copy streams, runner.Runner.finalize).

How the reference's arguments map onto the real engine:

* ``read_buffer`` (= min(hbm_read_buffer, bandwidth * queue wait), sim.py:439)
  with ``prev_job_running``: the head start.  Those bytes were moved by the
  pre-loader while the job waited in the queue, so the job's first
  ``floor(read_buffer / layer_bytes)`` layers are made resident before its
  measured region starts (Job.prestage_layers).  No wait -> no head start:
  the load starts with the job, exactly as overlap.py:91-93.
* ``bandwidth``: the real link decides; a disk hit (bandwidth = the disk's)
  first reads the session from the disk tier into the host arena, and that
  read's wall time is charged to the job (stall and makespan).
* ``plan_async_save``: the new tokens' K|V were already written back by K4
  during the prefill (layer by layer, overlapped); the output tokens' K|V --
  produced by decode in a server, outside this path -- are materialised by a
  teacher-forced append prefill over the resident rotated rows (no reload),
  saved the same way.  The returned Timeline holds those measured save
  intervals; ``stall_total`` is the save residue that outlives the compute
  and does not fit the write buffer (overlap.py:193-199), 0 when it fits.

Called with ``job=`` (sim.Server passes it) the plan runs on that session's
real rows.  Called with the reference's exact signature (no ``job``: a
maintainer rebinding ``kvsim.sim.plan_preload``) it runs a synthetic session
of that shape -- ``hist_tokens`` stored rows of random pre-RoPE K|V and
``new_tokens`` random tokens -- and returns the measured Timeline of it.
"""

from __future__ import annotations

import time
import zlib

import numpy as np
import torch

from .overlap import Timeline
from .runner import Job, ResidentKv, Runner
from .store import HitClass, Tier


def head_start_layers(read_buffer: float, prev_job_running: bool, kept: int,
                      row_bytes: int, layers: int) -> int:
    """Layers resident at job start: the read buffer's head start
    (overlap.py:91-93: min(read_buffer, kv bytes) moved before t = 0 when the
    previous job was running) in whole layers."""
    if not prev_job_running or read_buffer <= 0 or kept <= 0:
        return 0
    per_layer = kept * row_bytes
    return int(min(layers, read_buffer // per_layer))


def _merge(results) -> Timeline:
    """One Timeline for a chunked prefill: the chunks run back to back."""
    tl = Timeline()
    off = 0.0
    for r in results:
        t = r.timeline
        sh = lambda iv, o=off: [(a + o, b + o) for a, b in iv]  # noqa: E731
        tl.load_intervals += sh(t.load_intervals)
        tl.compute_intervals += sh(t.compute_intervals)
        tl.save_intervals += sh(t.save_intervals)
        tl.stall_total += t.stall_total
        tl.max_gap = max(tl.max_gap, t.max_gap)
        off += t.makespan
    tl.makespan = off
    return tl


def _rebase(tl: Timeline, first, prestaged: int) -> Timeline:
    """Start the job at its first activity: loads of layers >= `prestaged`
    that the pre-loader began before the compute stream reached the job
    (host issue latency) belong to the job, not to a head start -- with no
    head start loading begins at t = 0 (overlap.py:91-93), so the measured
    makespan and stall include that time.  `first`: the first chunk's load
    intervals (one per layer)."""
    late = [a for a, _ in first[prestaged:]]
    start = min([0.0] + late)
    if start >= 0.0:
        return tl
    sh = -start
    mv = lambda iv: [(a + sh, b + sh) for a, b in iv]  # noqa: E731
    tl.load_intervals = mv(tl.load_intervals)
    tl.compute_intervals = mv(tl.compute_intervals)
    tl.save_intervals = mv(tl.save_intervals)
    tl.makespan += sh
    tl.stall_total += sh
    tl.max_gap = max(tl.max_gap, sh)
    return tl


class MeasuredExecutor:
    """plan_preload / plan_async_save on the real engine (one GPU).

    engine:  engine.Engine whose store the serving loop shares
             (sim.run(..., store=engine.store)) -- the loop does the
             accounting (truncation, lookup, eviction, save), this does the
             physical work.
    save:    False for the recompute comparator (Mode.RECOMPUTE: nothing
             cached, every job one full-prompt prefill without saves).
    """

    measured = True

    def __init__(self, engine, *, save: bool = True, seed: int = 0,
                 want_logits: bool = False):
        self.eng = engine
        self.save = save
        self.seed = seed
        self.want_logits = want_logits
        s = engine.shape
        cap = engine.window + engine.chunk
        self.kv = ResidentKv(s, cap, engine.runner.device)
        self._rows: dict[str, int] = {}        # session -> rows after its prefill
        self._save_tl: dict[str, list] = {}    # session -> prefill chunks' results
        self.logits: dict[tuple, torch.Tensor] = {}
        self.disk_read_s = 0.0
        self.jobs = 0
        self.prestaged_layers = 0     # sum over jobs of layers resident at start

    # ------------------------------------------------------------ token ids
    def _ids(self, sid: str, turn: int, kind: int, n: int) -> torch.Tensor:
        g = np.random.default_rng([self.seed, zlib.crc32(sid.encode()), turn, kind])
        return torch.as_tensor(g.integers(0, self.eng.shape.vocab, n), dtype=torch.int64)

    def _history(self, sid: str, context: int) -> torch.Tensor:
        """The session's last `context` conversation ids (the loop truncated
        the stored item to them, sim.py:468-483)."""
        ids = self.eng.tokens.get(sid, torch.empty(0, dtype=torch.int64))
        if ids.numel() < context:
            raise RuntimeError(f"{sid}: {ids.numel()} known ids < context {context}")
        return ids[ids.numel() - context:]

    # ------------------------------------------------------------ the two plans
    def plan_preload(self, hist_tokens, new_tokens, profile, tiers, read_buffer,
                     prev_job_running=True, *, bandwidth=None, job=None) -> Timeline:
        if job is None:
            return self._synthetic(int(hist_tokens), int(new_tokens), float(read_buffer),
                                   bool(prev_job_running))
        eng, st = self.eng, self.eng.store
        sid = job.session_id
        context = int(job.context)
        hist = self._history(sid, context)
        turn_new = int(job.new_tokens) - (context if job.hit is HitClass.MISS else 0)
        new_ids = self._ids(sid, job.turn_index, 0, turn_new)
        st.pinned.add(sid)
        disk_s = 0.0
        k = 0
        try:
            if not self.save:
                return self._recompute(sid, torch.cat([hist, new_ids]), job)
            if job.hit is HitClass.MISS or hist_tokens == 0:
                if st.peek(sid) is None:
                    st.release_rows(sid)
                if eng.hbm is not None:
                    eng.hbm.drop(sid)
                self.kv.rows = 0
                res, rows, _ = eng._prefill(sid, torch.cat([hist, new_ids]), 0,
                                            self.want_logits, kv_cache=self.kv)
            else:
                it = st.peek(sid)
                if it is not None and it.tier is Tier.DISK:
                    t0 = time.perf_counter()       # the disk leg of a disk hit
                    eng._promote(sid, wait=True)
                    disk_s = time.perf_counter() - t0
                elif sid in st.pending:
                    t0 = time.perf_counter()       # a prefetch still landing
                    st.wait(sid)
                    disk_s = time.perf_counter() - t0
                k = head_start_layers(read_buffer, prev_job_running and disk_s == 0.0,
                                      context, eng.shape.row_bytes, eng.shape.layers)
                self.prestaged_layers += k
                self.kv.rows = 0
                res, rows, _ = eng._prefill(sid, new_ids, context, self.want_logits,
                                            kv_cache=self.kv, prestage_layers=k)
            torch.cuda.synchronize(eng.runner.device)
            Runner.finalize(res)
        finally:
            st.pinned.discard(sid)
        eng.tokens[sid] = torch.cat([hist, new_ids])[-rows:] if rows else hist[:0]
        self._rows[sid] = rows
        self._save_tl[sid] = res
        self.jobs += len(res)
        if self.want_logits:
            self.logits[(sid, job.turn_index)] = res[-1].logits
        tl = _merge(res)
        if res and res[0].timeline.load_intervals:
            tl = _rebase(tl, res[0].timeline.load_intervals, k)
        if disk_s:
            tl.load_intervals.insert(0, (0.0, disk_s))
            tl.load_intervals[1:] = [(a + disk_s, b + disk_s) for a, b in tl.load_intervals[1:]]
            tl.compute_intervals = [(a + disk_s, b + disk_s) for a, b in tl.compute_intervals]
            tl.save_intervals = [(a + disk_s, b + disk_s) for a, b in tl.save_intervals]
            tl.stall_total += disk_s
            tl.max_gap = max(tl.max_gap, disk_s)
            tl.makespan += disk_s
            self.disk_read_s += disk_s
        return tl

    def plan_async_save(self, prompt_tokens, decode_steps, profile, tiers, write_buffer, *,
                        bandwidth=None, job=None) -> Timeline:
        if job is None or not self.save:
            return Timeline()
        eng = self.eng
        sid = job.session_id
        pre = self._save_tl.pop(sid, [])
        rows = self._rows.pop(sid, None)
        if rows is None:
            raise RuntimeError(f"{sid}: save planned without a prefill")
        n_out = int(job.output_tokens)
        app = []
        if n_out > 0:
            out_ids = self._ids(sid, job.turn_index, 1, n_out)
            eng.store.pinned.add(sid)
            try:
                app, rows, _ = eng._prefill(sid, out_ids, rows, False, kv_cache=self.kv)
            finally:
                eng.store.pinned.discard(sid)
            torch.cuda.synchronize(eng.runner.device)
            Runner.finalize(app)
            eng.tokens[sid] = torch.cat([eng.tokens[sid], out_ids])[-rows:]
            self.jobs += len(app)
        self._rows_after = rows
        # save intervals of the prefill's K4 (on its own clock) then the append's
        tl = Timeline()
        p = _merge(pre) if pre else Timeline()
        a = _merge(app) if app else Timeline()
        tl.compute_intervals = p.compute_intervals + [(x + p.makespan, y + p.makespan)
                                                       for x, y in a.compute_intervals]
        tl.save_intervals = p.save_intervals + [(x + p.makespan, y + p.makespan)
                                                for x, y in a.save_intervals]
        compute_end = p.makespan + a.makespan
        last = max((y for _, y in tl.save_intervals), default=0.0)
        residue_s = max(0.0, last - compute_end)
        saved = (sum(r.bytes_saved for r in pre) + sum(r.bytes_saved for r in app))
        busy = sum(y - x for x, y in tl.save_intervals)
        rate = saved / busy if busy > 0 else 0.0
        over = max(0.0, residue_s * rate - float(write_buffer)) / rate if rate > 0 else 0.0
        tl.stall_total = over
        tl.max_gap = over
        tl.makespan = compute_end + over
        return tl

    # ------------------------------------------------------------ hooks
    def saved(self, sid: str, tokens: int) -> None:
        """The loop stored `tokens` (or nothing): physical rows follow."""
        st = self.eng.store
        if st.peek(sid) is None:      # nothing stored (StoreSizeError): rows go,
            st.release_rows(sid)      # the ids stay for the next turn's recompute
        else:
            ids = self.eng.tokens.get(sid)
            if ids is not None and ids.numel() > tokens:
                self.eng.tokens[sid] = ids[ids.numel() - tokens:]

    def released(self, sid: str) -> None:
        self.eng.tokens.pop(sid, None)

    # ------------------------------------------------------------ other shapes
    def _recompute(self, sid, ids, job) -> Timeline:
        """Recompute comparator: one full-prompt prefill, nothing saved.  A
        prompt longer than the window (one turn of more new tokens than W:
        the reference keeps 0 history and prefills them all, sim.py:473) runs
        as the engine's chunked prefill with the rolling window, through a
        scratch session whose rows are dropped afterwards."""
        eng = self.eng
        if ids.numel() > eng.window:
            tmp = "__recompute__"
            eng.store.release_rows(tmp)
            try:
                r, _, _ = eng._prefill(tmp, ids, 0, self.want_logits)
                torch.cuda.synchronize(eng.runner.device)
                Runner.finalize(r)
                eng.runner.fence(tmp)
            finally:
                eng.store.release_rows(tmp)
        else:
            r = eng.runner.run([Job(sid, ids, kept=0)], want_logits=self.want_logits)
            torch.cuda.synchronize(eng.runner.device)
            Runner.finalize(r)
        tl = _merge(r)
        out = self._ids(sid, job.turn_index, 1, int(job.output_tokens))
        eng.tokens[sid] = torch.cat([ids, out])
        self.jobs += len(r)
        if self.want_logits:
            self.logits[(sid, job.turn_index)] = r[-1].logits
        return tl

    def _synthetic(self, hist: int, new: int, read_buffer: float,
                   prev_job_running: bool) -> Timeline:
        """The reference signature without a session: a scratch session of
        `hist` stored rows (random pre-RoPE K|V in fresh arena blocks) and
        `new` random tokens, run and measured, then released."""
        eng = self.eng
        st = eng.store
        sid = "__plan_preload__"
        if new < 1:   # load only (overlap.py:112-115): time the pre-load of every layer
            return self._load_only(hist)
        if hist == 0:
            r = eng.runner.run([Job(sid, self._ids(sid, 0, 0, new), kept=0)])
            torch.cuda.synchronize(eng.runner.device)
            Runner.finalize(r)
            return r[0].timeline
        st.release_rows(sid)
        tab = st.reserve_rows(sid, hist + new)
        bb = st.block_bytes
        g = torch.Generator().manual_seed(hist)
        view = st.arena.buffer.view(torch.bfloat16)
        for b in tab:
            view[b * bb // 2:(b + 1) * bb // 2].copy_(
                torch.randn(bb // 2, generator=g).to(torch.bfloat16))
        k = head_start_layers(read_buffer, prev_job_running, hist, eng.shape.row_bytes,
                              eng.shape.layers)
        job = Job(sid, self._ids(sid, 0, 0, new), kept=hist, source="host", block_ids=tab,
                  save=True, prestage_layers=k)
        try:
            r = eng.runner.run([job])
            torch.cuda.synchronize(eng.runner.device)
            Runner.finalize(r)
            eng.runner.fence(sid)
        finally:
            st.release_rows(sid)
        return _rebase(r[0].timeline, r[0].timeline.load_intervals, k)

    def _load_only(self, hist: int) -> Timeline:
        from . import ops

        eng, st = self.eng, self.eng.store
        tl = Timeline()
        if hist == 0:
            return tl
        sid = "__plan_preload__"
        torch.cuda.synchronize(eng.runner.device)   # slot 0 is borrowed below
        eng.runner.fence(None)
        st.release_rows(sid)
        tab = st.reserve_rows(sid, hist)
        r = eng.runner
        nb = -(-hist // r.block_tokens)
        tail = (hist - (nb - 1) * r.block_tokens) * r.row_bytes
        slot = r.slots[0]
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(eng.shape.layers + 1)]
        try:
            with torch.cuda.stream(r.s_load):
                evs[0].record()
                for layer in range(eng.shape.layers):
                    ops.preload_layer(slot, st.arena.buffer, tab[:nb], r.block_bytes,
                                      layer * r.chunk_bytes, r.chunk_bytes, tail,
                                      stream=r.s_load)
                    evs[layer + 1].record()
            torch.cuda.synchronize(r.device)
        finally:
            st.release_rows(sid)
        t = [evs[0].elapsed_time(e) * 1e-3 for e in evs]
        tl.load_intervals = list(zip(t[:-1], t[1:]))
        tl.makespan = t[-1]
        tl.stall_total = t[-1]
        tl.max_gap = t[-1]
        return tl


def reset(engine) -> None:
    """Forget every stored session (accounting and rows) between runs."""
    engine.runner.fence(None)
    st = engine.store
    for sid in list(st.items):
        st.remove(sid)
    for sid in list(st.tables):
        st.release_rows(sid)
    engine.tokens.clear()
    engine.context.clear()


def serve(workload, engine, cfg, *, recompute: bool = False, seed: int = 0,
          want_logits: bool = False, executor_cls=None):
    """Replay `workload` through the reference serving loop (sim.Server: job
    queue, continuous batching, truncation, scheduler-aware eviction /
    prefetch) with every prefill and save measured on this GPU.  Returns
    (EventLog, executor).  `recompute` = the reference's Mode.RECOMPUTE
    comparator (nothing cached; every job a full-prompt prefill)."""
    from dataclasses import replace

    from . import sim

    reset(engine)
    cls = executor_cls or MeasuredExecutor
    ex = cls(engine, save=not recompute, seed=seed, want_logits=want_logits)
    cfg = replace(cfg, mode=sim.Mode.RECOMPUTE if recompute else sim.Mode.REUSE)
    engine.policy = cfg.policy
    log = sim.run(workload, cfg, ex, store=None if recompute else engine.store)
    torch.cuda.synchronize(engine.runner.device)
    return log, ex
