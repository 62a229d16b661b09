"""LLaMA-shaped prefill runner with AttentionStore KV reuse on one B200.

Per job (one conversation turn) and per layer l, on three CUDA streams:

  copy stream   K1  H2D of the session's kept pre-RoPE K/V blocks for layer l
                    into a read-buffer slot (runs ahead across layers and jobs:
                    the slot ring is the HBM read buffer, §3.2.1)
  compute       rms_norm -> QKV GEMM (cuBLAS) -> rope_new (q/k RoPE, pre-RoPE
                    copy to the write buffer) -> [wait load_l] -> K2 reembed
                    (truncate + re-embed kept rows) -> K3 attention (tcgen05)
                    -> O GEMM + residual -> rms_norm -> gate/up GEMM -> SiLU*mul
                    -> down GEMM + residual
  save stream   K4  D2H of the new tokens' pre-RoPE K/V for layer l from the
                    write buffer into the session's tail blocks (§3.2.2)

Sources of reused KV: ``"host"`` (pinned host arena via K1, the AttentionStore
path), ``"hbm"`` (HBM-resident arena gathered in place by K2 through a device
block table), or none (miss / recompute: the whole prompt
is prefilled).  Every timing is a CUDA event on the stream doing the work; the
per-job ``Timeline`` follows overlap.py:31-66 (see overlap.py here).

The projections are plain cuBLAS GEMMs through torch; everything on the
AttentionStore path itself is libaskv.so (rope_new, reembed, prefill_attn,
preload_layer, save_layer).
"""

from __future__ import annotations

import math
import queue
import threading
from dataclasses import dataclass, field

import torch
import torch.nn.functional as F

from . import ops
from .model import LlamaShape
from .overlap import Timeline

BF16 = torch.bfloat16


class LlamaWeights:
    """Random-init N(0, 0.02) bf16 weights of a LLaMA-shaped decoder
    (seeded torch.Generator; RMSNorm gains = 1)."""

    def __init__(self, shape: LlamaShape, *, seed: int = 0, device="cuda", std: float = 0.02):
        self.shape = s = shape
        g = torch.Generator(device=device).manual_seed(seed)

        def rnd(*dims):
            return (torch.randn(*dims, generator=g, device=device, dtype=torch.float32)
                    * std).to(BF16)

        self.embed = rnd(s.vocab, s.d_model)
        self.layers = []
        for _ in range(s.layers):
            self.layers.append({
                "w_in": torch.ones(s.d_model, dtype=BF16, device=device),
                "wqkv": rnd(s.qkv_cols, s.d_model),                 # [out, in]
                "wo": rnd(s.d_model, s.n_heads * s.head_dim),
                "w_post": torch.ones(s.d_model, dtype=BF16, device=device),
                "wgu": rnd(2 * s.ffn, s.d_model),                   # gate | up
                "wd": rnd(s.d_model, s.ffn),
            })
        self.w_final = torch.ones(s.d_model, dtype=BF16, device=device)
        self.lm_head = rnd(s.vocab, s.d_model)

    def shard(self, rank: int, tp: int) -> "LlamaWeights":
        """Head-parallel tensor-parallel shard (Megatron layout):
        q-heads [r*Hq/tp, (r+1)*Hq/tp), kv-heads [r*Hkv/tp, ...), the matching
        rows of W_qkv / columns of W_o, rows r of the gate/up split and columns of
        W_down.  Norms, embedding and lm_head are replicated."""
        s = self.shape
        sh = s.tp_shard(tp)
        hd = s.head_dim
        out = LlamaWeights.__new__(LlamaWeights)
        out.shape = sh
        out.embed = self.embed
        out.w_final = self.w_final
        out.lm_head = self.lm_head
        qa, qb = rank * sh.n_heads * hd, (rank + 1) * sh.n_heads * hd
        ka, kb = rank * sh.n_kv_heads * hd, (rank + 1) * sh.n_kv_heads * hd
        fa, fb = rank * sh.ffn, (rank + 1) * sh.ffn
        qoff, koff, voff = 0, s.n_heads * hd, (s.n_heads + s.n_kv_heads) * hd
        out.layers = []
        for l in self.layers:
            wqkv = torch.cat([l["wqkv"][qoff + qa: qoff + qb], l["wqkv"][koff + ka: koff + kb],
                              l["wqkv"][voff + ka: voff + kb]]).contiguous()
            wgu = torch.cat([l["wgu"][fa:fb], l["wgu"][s.ffn + fa: s.ffn + fb]]).contiguous()
            out.layers.append({"w_in": l["w_in"], "wqkv": wqkv,
                               "wo": l["wo"][:, qa:qb].contiguous(), "w_post": l["w_post"],
                               "wgu": wgu, "wd": l["wd"][:, fa:fb].contiguous()})
        return out

    def to_numpy(self) -> dict:
        """float64 copies in the oracle's [in, out] convention (tests only)."""
        f = lambda t: t.float().cpu().numpy().astype("float64")  # noqa: E731
        return {
            "embed": f(self.embed),
            "layers": [{"w_in": f(l["w_in"]), "wqkv": f(l["wqkv"]).T, "wo": f(l["wo"]).T,
                        "w_post": f(l["w_post"]),
                        "wg": f(l["wgu"][: self.shape.ffn]).T,
                        "wu": f(l["wgu"][self.shape.ffn:]).T, "wd": f(l["wd"]).T}
                       for l in self.layers],
            "w_final": f(self.w_final),
            "lm_head": f(self.lm_head).T,
        }


@dataclass
class Job:
    """One prefill job (a conversation turn) for the runner.

    token_ids: (N,) int64 new tokens (device or host).
    kept:      reused history rows (positions 0..kept-1); 0 = miss/recompute.
    source:    "host" | "hbm" | "none" — where the kept rows live.
    block_ids: the session's block table (covers kept rows, plus the tail
               rows [kept, kept+N) when save=True).
    save:      write the new tokens' pre-RoPE K/V back (K4).
    """

    session_id: str
    token_ids: torch.Tensor
    kept: int = 0
    source: str = "none"
    block_ids: list[int] = field(default_factory=list)
    save: bool = False
    dev_block_off: torch.Tensor | None = None  # "hbm": element offsets per block
    head: int = 0   # row of session token 0 inside block_ids[0] (store.head_row)
    prestage: bool = False  # start the job only once all its layers are pre-loaded

    @property
    def n_new(self) -> int:
        return int(self.token_ids.numel())

    @property
    def prompt_tokens(self) -> int:
        return self.kept + self.n_new


@dataclass
class JobResult:
    session_id: str
    kept: int
    n_new: int
    timeline: Timeline | None
    first_token: torch.Tensor          # (1,) int64 argmax of the last position (pinned host)
    logits: torch.Tensor | None = None  # (vocab,) fp32 if requested
    bytes_loaded: int = 0
    bytes_saved: int = 0


def attention_flops(kept: int, n: int, hq: int, hd: int) -> int:
    """Algorithmic FLOPs of causal prefill attention over [kept | new]
    (QK^T and PV, unmasked entries only): 4 * Hq * hd * (N*kept + N(N+1)/2)."""
    return 4 * hq * hd * (n * kept + n * (n + 1) // 2)


class _Unit:
    """One (job, layer) pre-load: a read-buffer slot, its DMA events and a host
    flag set once the IO thread has submitted the DMA."""
    __slots__ = ("seq", "slot", "start", "end", "issued")


class _IOThread(threading.Thread):
    """Submits copy-engine work (pre-load / save DMA batches) from its own host
    thread, FIFO.  A multi-GB pre-load queue can block cudaMemcpyBatchAsync on
    stream back-pressure; on the compute thread that would starve kernel
    issue (the paper's system likewise uses dedicated IO threads)."""

    def __init__(self, device, name):
        super().__init__(name=name, daemon=True)
        dev = torch.device(device)
        self.device_index = dev.index if dev.index is not None else torch.cuda.current_device()
        self.q: queue.Queue = queue.Queue()
        self.error = None
        self.start()

    def run(self):
        try:
            torch.cuda.set_device(self.device_index)
        except BaseException as exc:
            self.error = exc
        while True:
            fn = self.q.get()
            if fn is None:
                return
            try:
                fn()
            except BaseException as exc:  # surfaced on the compute thread
                self.error = exc

    def submit(self, fn):
        if self.error is not None:
            raise RuntimeError("IO thread failed") from self.error
        self.q.put(fn)


class Runner:
    """Executes Jobs back to back; owns streams, HBM buffers and the read /
    write buffer rings.  One Runner per GPU (one process per GPU)."""

    def __init__(self, shape: LlamaShape, *, weights: LlamaWeights | None = None,
                 device="cuda", seed: int = 0, theta_base: float = 10000.0,
                 block_tokens: int = 128, host_arena=None, hbm_arena: torch.Tensor | None = None,
                 read_buffer_bytes: int = 4 << 30, write_buffer_bytes: int = 2 << 30,
                 max_new: int = 1024, max_ctx: int | None = None, timeline: bool = True,
                 tp_reduce=None):
        self.shape = s = shape
        self.device = torch.device(device)
        self.w = weights or LlamaWeights(shape, seed=seed, device=device)
        self.block_tokens = block_tokens
        self.row_elems = s.row_elems
        self.row_bytes = s.row_bytes
        self.chunk_bytes = block_tokens * s.row_bytes
        self.block_bytes = s.layers * self.chunk_bytes
        self.host_arena = host_arena
        self.hbm_arena = hbm_arena
        self.max_ctx = max_ctx or s.context_window
        self.max_new = max_new
        self.timeline = timeline
        self.table = ops.RopeTable(self.max_ctx + max_new + 1, s.head_dim, theta_base,
                                   self.device)
        self.s_compute = torch.cuda.Stream(device=self.device)
        self.s_load = torch.cuda.Stream(device=self.device)
        self.s_save = torch.cuda.Stream(device=self.device)
        # read buffer: ring of per-layer slots of max_ctx rows
        self.slot_rows = self.max_ctx + block_tokens   # + a partial head block
        slot_bytes = self.slot_rows * s.row_bytes
        self.n_slots = max(2, int(read_buffer_bytes // slot_bytes))
        self.slots = torch.empty((self.n_slots, self.slot_rows, s.row_elems), dtype=BF16,
                                 device=self.device)
        self._units: dict = {}          # (jid, layer) -> _Unit
        self._seq = 0                    # pre-load units enqueued so far
        self._freed: dict = {}           # unit seq -> (event on s_compute, host flag)
        self._io_load = _IOThread(self.device, "askv-preload")
        self._io_save = _IOThread(self.device, "askv-save")
        # write buffer: ring of per-layer slots of max_new rows
        self.n_wslots = max(2, int(write_buffer_bytes // (max_new * s.row_bytes)))
        self.wbuf = torch.empty((self.n_wslots, max_new, s.row_elems), dtype=BF16,
                                device=self.device)
        self._wseq = 0
        self._wdone = [None] * self.n_wslots   # (event on s_save, host flag) per slot
        self._last_save: dict = {}             # session -> (event, flag) of its last save
        self._bufs = {}
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        # tensor parallelism (config C5): tp_reduce(t, stream) sums the row-parallel
        # partials of W_o and W_down over the TP group in place (NCCL all-reduce
        # over NVLink in a multi-GPU run; dist.ThreadAllReduce in the 1-GPU emulation)
        self.tp_reduce = tp_reduce
        self.launches = 0          # libaskv kernel launches issued (all streams)
        self.probe = None          # list -> (kind, ev0, ev1, work) per probed launch

    # ------------------------------------------------------------------ buffers
    def _buf(self, name, rows, cols, dtype=BF16):
        t = self._bufs.get(name)
        if t is None or t.shape[0] < rows or t.shape[1] != cols:
            t = torch.empty((max(rows, 1), cols), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[:rows]

    def _workspace(self, nbytes):
        if self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._ws

    # ------------------------------------------------------------------ K1 pre-loader
    def _enqueue_loads(self, jid, job: Job):
        """Queue the job's L pre-load units for the IO thread.  Unit seq k uses
        slot k % n_slots and first waits (host flag, then device event) for the
        release of unit k - n_slots, so the copy stream runs as far ahead as
        the read buffer allows -- across jobs, i.e. the read-buffer head start."""
        if job.source != "host" or job.kept == 0:
            return
        if self.host_arena is None:
            raise RuntimeError("host-sourced job but the runner has no host arena")
        rows = job.head + job.kept
        if rows > self.slot_rows:
            raise ValueError(f"kept {job.kept} exceeds read-buffer slot rows {self.slot_rows}")
        nb = -(-rows // self.block_tokens)
        tail = (rows - (nb - 1) * self.block_tokens) * self.row_bytes
        ids = list(job.block_ids[:nb])
        dep = self._last_save.get(job.session_id)
        for layer in range(self.shape.layers):
            u = _Unit()
            u.seq = self._seq
            u.slot = u.seq % self.n_slots
            u.start = torch.cuda.Event(enable_timing=self.timeline)
            u.end = torch.cuda.Event(enable_timing=self.timeline)
            u.issued = threading.Event()
            self._seq += 1
            self._units[(jid, layer)] = u
            prev = u.seq - self.n_slots
            if prev >= 0 and prev not in self._freed:
                self._freed[prev] = (torch.cuda.Event(), threading.Event())
            freed = self._freed.get(prev) if prev >= 0 else None

            def submit(u=u, layer=layer, freed=freed, dep=dep):
                try:
                    with torch.cuda.stream(self.s_load):
                        if freed is not None:   # slot reuse: its previous reader is done
                            freed[1].wait()
                            self.s_load.wait_event(freed[0])
                        if dep is not None:     # rows saved by this session's previous turn
                            dep[1].wait()
                            self.s_load.wait_event(dep[0])
                        u.start.record(self.s_load)
                        ops.preload_layer(self.slots[u.slot], self.host_arena.buffer, ids,
                                          self.block_bytes, layer * self.chunk_bytes,
                                          self.chunk_bytes, tail, stream=self.s_load)
                        u.end.record(self.s_load)
                finally:
                    u.issued.set()

            self._io_load.submit(submit)

    def _acquire(self, jid, layer) -> _Unit:
        u = self._units.pop((jid, layer), None)
        if u is None:
            raise RuntimeError("pre-load unit was never enqueued")
        if not u.issued.wait(timeout=600):
            raise RuntimeError("pre-load IO thread stalled")
        if self._io_load.error is not None:
            raise RuntimeError("pre-load IO thread failed") from self._io_load.error
        return u

    def _release(self, u: _Unit):
        """The slot's reader (K2) is enqueued: record it and wake the IO thread."""
        ent = self._freed.get(u.seq)
        if ent is None:
            ent = self._freed[u.seq] = (torch.cuda.Event(), threading.Event())
        ent[0].record(self.s_compute)
        ent[1].set()
        self._freed.pop(u.seq - 2 * self.n_slots, None)

    def _submit_save(self, produced, arena, job, layer, kept, n, wslot, sv0, sv1, flag):
        def submit():
            try:
                with torch.cuda.stream(self.s_save):
                    self.s_save.wait_event(produced)
                    if sv0 is not None:
                        sv0.record(self.s_save)
                    ops.save_layer(arena, job.block_ids, self.block_bytes,
                                   layer * self.chunk_bytes, self.block_tokens, self.row_bytes,
                                   job.head + kept, n, self.wbuf[wslot], stream=self.s_save)
                    sv1.record(self.s_save)
            finally:
                flag.set()

        self._io_save.submit(submit)

    def close(self) -> None:
        for t in (self._io_load, self._io_save):
            t.q.put(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ main entry
    def run(self, jobs: list[Job], *, want_logits: bool = False) -> list[JobResult]:
        """Issue all jobs back to back; returns results whose timelines are
        resolved by ``finalize`` (call after synchronising)."""
        base = id(jobs)
        sids = [j.session_id for j in jobs]
        if len(set(sids)) != len(sids):
            raise ValueError("a session may appear once per run() call (its next turn "
                             "depends on this turn's save)")
        for i, job in enumerate(jobs):
            self._enqueue_loads((base, i), job)
        results = []
        for i, job in enumerate(jobs):
            results.append(self._run_job((base, i), job, want_logits))
        self.drain_io()
        return results

    def drain_io(self) -> None:
        """Wait until the IO threads have submitted everything queued so far, so
        a later device synchronise covers this run's loads and saves."""
        for t in (self._io_load, self._io_save):
            done = threading.Event()
            t.submit(done.set)
            done.wait()
            if t.error is not None:
                raise RuntimeError(f"{t.name} failed") from t.error

    def _run_job(self, jid, job: Job, want_logits: bool) -> JobResult:
        s = self.shape
        n, kept = job.n_new, job.kept
        if n < 1:
            raise ValueError("a job needs at least one new token")
        if job.save and n > self.max_new:
            raise ValueError(f"{n} saved rows exceed the write-buffer slot ({self.max_new})")
        if kept + n > self.table.max_pos:
            raise ValueError("context exceeds the runner's RoPE table")
        if job.save and len(job.block_ids) * self.block_tokens < job.head + kept + n:
            raise ValueError("save needs block_ids covering kept + new rows")
        arena = None
        if job.save:
            arena = self.hbm_arena if job.source == "hbm" else (
                self.host_arena.buffer if self.host_arena is not None else None)
            if arena is None:
                raise RuntimeError("save requested but no arena for it")
        hd, hq, hkv = s.head_dim, s.n_heads, s.n_kv_heads
        cs = self.s_compute
        ev = (lambda: torch.cuda.Event(enable_timing=True)) if self.timeline else None
        rec = {"layers": [], "waits": [], "saves": [], "loads": []}
        first = torch.empty(1, dtype=torch.int64, pin_memory=True)
        logits_out = None
        with torch.cuda.stream(cs):
            if job.prestage and job.source == "host" and kept:
                if s.layers > self.n_slots:
                    raise RuntimeError("read buffer too small to prestage a whole job")
                last = self._units[(jid, s.layers - 1)]
                if not last.issued.wait(timeout=600):
                    raise RuntimeError("pre-load IO thread stalled")
                cs.wait_event(last.end)
            t0 = ev() if ev else None
            if t0:
                t0.record(cs)
            if job.token_ids.is_cuda:
                ids = job.token_ids
            else:  # pinned host ids: SM copy, not behind the pre-load DMAs
                src = job.token_ids if job.token_ids.is_pinned() else job.token_ids.pin_memory()
                ids = ops.copy_sm(torch.empty(n, dtype=torch.int64, device=self.device),
                                  src.to(torch.int64), stream=cs)
                self.launches += 1
            x = F.embedding(ids, self.w.embed)
            q_rot = self._buf("q", n, hq * hd)
            kvbuf = self._buf("kv", kept + n, self.row_elems)
            ao = self._buf("ao", n, hq * hd)
            splits = ops.attn_num_splits(kept, n, hq)
            wsb = ops.attn_workspace_bytes(kept, n, hq, hd, splits)
            ws = self._workspace(wsb) if wsb else None
            for layer, lw in enumerate(self.w.layers):
                l0 = ev() if ev else None
                if l0:
                    l0.record(cs)
                h = ops.rmsnorm(x, lw["w_in"], 1e-5, stream=cs)
                qkv = F.linear(h, lw["wqkv"])
                wslot = None
                if job.save:
                    wslot = self._wseq % self.n_wslots
                    self._wseq += 1
                    if self._wdone[wslot] is not None:   # slot's previous D2H finished
                        self._wdone[wslot][1].wait()
                        cs.wait_event(self._wdone[wslot][0])
                ops.rope_new(qkv, n, hq, hkv, hd, self.table, kept, q_rot, kvbuf[kept:],
                             self.wbuf[wslot] if wslot is not None else None, stream=cs)
                self.launches += 1
                if job.save:
                    produced = torch.cuda.Event()
                    produced.record(cs)
                    sv0 = ev() if ev else None
                    sv1 = torch.cuda.Event(enable_timing=self.timeline)
                    flag = threading.Event()
                    self._submit_save(produced, arena, job, layer, kept, n, wslot, sv0, sv1,
                                      flag)
                    self._wdone[wslot] = (sv1, flag)
                    rec["saves"].append((sv0, sv1, flag))
                if kept:
                    if job.source == "host":
                        u = self._acquire(jid, layer)
                        w0 = ev() if ev else None
                        if w0:
                            w0.record(cs)
                        cs.wait_event(u.end)
                        w1 = ev() if ev else None
                        if w1:
                            w1.record(cs)
                        rec["waits"].append((w0, w1))
                        rec["loads"].append((u.start, u.end))
                        p0 = self._probe_begin()
                        ops.reembed(self.slots[u.slot], kept, hkv, hd, self.table, kvbuf,
                                    first_token=job.head, pos0=0, stream=cs)
                        self._probe_end(p0, "reembed", 2 * kept * s.row_bytes)
                        self.launches += 1
                        self._release(u)
                    elif job.source == "hbm":
                        if job.dev_block_off is None:
                            raise ValueError("hbm job needs dev_block_off")
                        src = self.hbm_arena[layer * self.block_tokens * self.row_elems:]
                        p0 = self._probe_begin()
                        ops.reembed(src, kept, hkv, hd, self.table, kvbuf,
                                    first_token=job.head, pos0=0, block_off=job.dev_block_off,
                                    block_tokens=self.block_tokens, stream=cs)
                        self._probe_end(p0, "reembed", 2 * kept * s.row_bytes)
                        self.launches += 1
                    else:
                        raise ValueError(f"job with kept={kept} needs a source")
                p0 = self._probe_begin()
                ops.prefill_attn(q_rot, kvbuf, kept, n, hq, hkv, hd, ao, ws,
                                 num_splits=splits, stream=cs)
                self._probe_end(p0, "attention", attention_flops(kept, n, hq, hd))
                self.launches += 2 if splits > 1 else 1
                if self.tp_reduce is None:
                    x = torch.addmm(x, ao, lw["wo"].t())
                else:
                    y = torch.mm(ao, lw["wo"].t())
                    self.tp_reduce(y, cs)
                    x = x + y
                h = ops.rmsnorm(x, lw["w_post"], 1e-5, stream=cs)
                gu = F.linear(h, lw["wgu"])
                a = ops.silu_mul(gu, stream=cs)
                if self.tp_reduce is None:
                    x = torch.addmm(x, a, lw["wd"].t())
                else:
                    y = torch.mm(a, lw["wd"].t())
                    self.tp_reduce(y, cs)
                    x = x + y
                self.launches += 3
                l1 = ev() if ev else None
                if l1:
                    l1.record(cs)
                rec["layers"].append((l0, l1))
            hl = ops.rmsnorm(x[-1:], self.w.w_final, 1e-5, stream=cs)
            logits = F.linear(hl, self.w.lm_head).float()
            ops.copy_sm(first, logits.argmax(dim=-1), stream=cs)
            self.launches += 1
            if want_logits:
                logits_out = logits[0].clone()
            t1 = ev() if ev else None
            if t1:
                t1.record(cs)
        if job.save:
            _, sv1, flag = rec["saves"][-1]
            self._last_save[job.session_id] = (sv1, flag)
        res = JobResult(job.session_id, kept, n, None, first, logits_out,
                        bytes_loaded=kept * s.kv_bytes_per_token if job.source == "host" else 0,
                        bytes_saved=n * s.kv_bytes_per_token if job.save else 0)
        res._events = (t0, t1, rec) if ev else None
        return res

    def _probe_begin(self):
        if self.probe is None:
            return None
        e = torch.cuda.Event(enable_timing=True)
        e.record(self.s_compute)
        return e

    def _probe_end(self, e0, kind, work):
        if e0 is None:
            return
        e1 = torch.cuda.Event(enable_timing=True)
        e1.record(self.s_compute)
        self.probe.append((kind, e0, e1, work))

    def join(self) -> None:
        """Make the compute stream wait for all loads and saves queued so far
        (waits for the IO threads to submit them first)."""
        self.drain_io()
        self.s_compute.wait_stream(self.s_load)
        self.s_compute.wait_stream(self.s_save)

    # ------------------------------------------------------------------ timelines
    @staticmethod
    def finalize(results: list[JobResult]) -> None:
        """Resolve CUDA events into seconds (call after synchronising)."""
        for r in results:
            evs = getattr(r, "_events", None)
            if not evs:
                continue
            t0, t1, rec = evs
            f = lambda e: t0.elapsed_time(e) * 1e-3  # noqa: E731
            tl = Timeline()
            tl.makespan = f(t1)
            waits = [(f(a), f(b)) for a, b in rec["waits"]]
            stall = sum(b - a for a, b in waits)
            tl.load_intervals = [(f(a), f(b)) for a, b in rec["loads"]]
            for *_, flag in rec["saves"]:
                flag.wait()
            tl.save_intervals = [(f(a), f(b)) for a, b, _ in rec["saves"]]
            comp = []
            wi = iter(waits)
            for li, (a, b) in enumerate(rec["layers"]):
                la, lb = f(a), f(b)
                if waits:
                    wa, wb = next(wi)
                    comp.extend([(la, wa), (wb, lb)])
                else:
                    comp.append((la, lb))
            tl.compute_intervals = comp
            tl.stall_total = stall if stall > 1e-9 else 0.0
            tl.max_gap = max((b - a for a, b in waits), default=0.0)
            r.timeline = tl
            r._events = None
