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

The per-layer loop of a job is issued natively by ``askv_prefill_layers``
(csrc/runtime.cu): projections are plain cuBLASLt GEMMs, everything else is
libaskv.so's own kernels (rmsnorm, rope_new, reembed, prefill_attn, silu_mul);
pre-load / save DMAs (preload_layer, save_layer) are submitted by two IO
threads here.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import queue
import threading
from dataclasses import dataclass, field

import numpy as np
import torch
import torch.nn.functional as F

from . import _lib, ops
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
    # HBM session tier: write-through copy of the saved
    # rows into these HBM-arena blocks, and/or promotion of the pre-loaded rows
    # (host source) into them; both mirror block_ids one-to-one.
    mirror_block_ids: list | None = None
    promote_block_ids: list | None = None
    head: int = 0   # row of session token 0 inside block_ids[0] (store.head_row)
    # sessions whose HBM-tier blocks this job's mirror / promotion reuses: their
    # last saves (write-through on the save stream) must land first
    fence_sessions: set = field(default_factory=set)
    prestage: bool = False  # start the job only once all its layers are pre-loaded
    # read-buffer head start (overlap.py:91-93, sim.py:439): start the job once
    # its first `prestage_layers` layers are pre-loaded (the bytes the loader
    # moved while the job waited in the queue); 0 = none, >= layers = all
    prestage_layers: int = 0
    # resident rotated KV (decode): the job writes all its
    # layers' rows into kv_cache; source "resident" = kept rows already there
    kv_cache: "ResidentKv | None" = None

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
    next_token: torch.Tensor | None = None  # (1,) int64 argmax on the device (greedy decode)


class ResidentKv:
    """One session's rotated K|V rows for every layer, kept in HBM across the
    jobs of a turn (prefill, then one decode step per generated token):
    [layers][capacity][2][Hkv][hd] bf16.  `rows` = valid rows (positions
    0..rows-1)."""

    def __init__(self, shape: LlamaShape, capacity: int, device="cuda"):
        self.capacity = int(capacity)
        self.buf = torch.empty((shape.layers, self.capacity, shape.row_elems), dtype=BF16,
                               device=device)
        self.rows = 0

    def layer_ptrs(self) -> list[int]:
        return [self.buf[l].data_ptr() for l in range(self.buf.shape[0])]


def attention_flops(kept: int, n: int, hq: int, hd: int) -> int:
    """Algorithmic FLOPs of causal prefill attention over [kept | new]
    (QK^T and PV, unmasked entries only): 4 * Hq * hd * (N*kept + N(N+1)/2)."""
    return 4 * hq * hd * (n * kept + n * (n + 1) // 2)


class _Unit:
    """One (job, layer) pre-load: a read-buffer slot and a host flag set once
    the IO thread has submitted its DMA (the slot's ``ready`` event is then
    recorded behind it)."""
    __slots__ = ("seq", "slot", "times", "issued")


class _EventPool:
    """Recycled timing events for per-job timelines (creating ~10 events per
    layer per job would cost more host time than issuing the layer)."""

    def __init__(self):
        self.free: list = []

    def get(self) -> ops.NativeEvent:
        return self.free.pop() if self.free else ops.NativeEvent(timing=True)


class _Lease:
    """The timing events of one job; they go back to the pool when the job's
    result is dropped (by then run() has drained the IO threads, so no record
    of them is still to be submitted)."""
    __slots__ = ("pool", "events")

    def __init__(self, pool: _EventPool):
        self.pool, self.events = pool, []

    def get(self) -> ops.NativeEvent:
        e = self.pool.get()
        self.events.append(e)
        return e

    def __del__(self):
        try:
            self.pool.free.extend(self.events)
        except Exception:
            pass


def _await(ev: threading.Event, what: str, timeout: float = 600.0) -> None:
    """Host wait on an IO-thread flag that fails loudly instead of hanging
    (a failed job can leave a flag that nobody will set)."""
    if not ev.wait(timeout):
        raise RuntimeError(f"{what} stalled ({timeout:.0f} s)")


def _ptr_array(items) -> "C.Array":
    """ctypes void*[] of device pointers / event handles (None -> NULL)."""
    return (C.c_void_p * len(items))(*items)


class _IOThread(threading.Thread):
    """Submits copy-engine work (pre-load / save DMA batches) from its own host
    thread, FIFO.  A multi-GB pre-load queue can block the copy calls on
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
    write buffer rings.  One Runner per GPU (one process per GPU).

    Each job's layer loop is issued by the native runtime
    (``askv_prefill_layers``, csrc/runtime.cu); this class only fills the plan
    (pointers, per-layer slots and events) and drives the pre-load / save IO
    threads around it."""

    def __init__(self, shape: LlamaShape, *, weights: LlamaWeights | None = None,
                 device="cuda", seed: int = 0, theta_base: float = 10000.0,
                 block_tokens: int = 128, host_arena=None, hbm_arena: torch.Tensor | None = None,
                 read_buffer_bytes: int = 4 << 30, write_buffer_bytes: int = 2 << 30,
                 max_new: int = 1024, max_ctx: int | None = None, timeline: bool = True,
                 tp_reduce=None, gemm_workspace_bytes: int = 32 << 20, graph: bool = True,
                 autotune: bool | int = True, overlap: bool = False):
        self.shape = s = shape
        self.graph = graph   # issue each job's layer loop as one CUDA graph launch
        # K2 of layer l+1 alongside K3 of layer l (second stream, two KV buffers)
        self.overlap = overlap
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
        L = s.layers
        # read buffer: ring of per-layer slots of max_ctx rows.  A job's L units
        # are all submitted before its layer loop is issued, so the ring holds
        # at least L + 1 slots.
        self.slot_rows = self.max_ctx + block_tokens   # + a partial head block
        slot_bytes = self.slot_rows * s.row_bytes
        self.n_slots = max(L + 1, int(read_buffer_bytes // slot_bytes))
        self.slots = torch.empty((self.n_slots, self.slot_rows, s.row_elems), dtype=BF16,
                                 device=self.device)
        self._slot_ready = [ops.NativeEvent() for _ in range(self.n_slots)]
        self._slot_free = [ops.NativeEvent() for _ in range(self.n_slots)]
        self._units: dict = {}          # (jid, layer) -> _Unit
        self._seq = 0                    # pre-load units enqueued so far
        self._freed: dict = {}           # unit seq -> host flag: its slot's reader is issued
        self._io_load = _IOThread(self.device, "askv-preload")
        self._io_save = _IOThread(self.device, "askv-save")
        # write buffer: ring of per-layer slots of max_new rows (>= L: one job's
        # layers never share a slot)
        self.n_wslots = max(L, int(write_buffer_bytes // (max_new * s.row_bytes)))
        self.wbuf = torch.empty((self.n_wslots, max_new, s.row_elems), dtype=BF16,
                                device=self.device)
        self._wseq = 0
        self._wready = [ops.NativeEvent() for _ in range(self.n_wslots)]
        self._wdone = [ops.NativeEvent() for _ in range(self.n_wslots)]
        self._wflag: list = [None] * self.n_wslots   # host flag: slot's last save submitted
        self._sess_ev: dict = {}                     # session -> event of its last save
        self._last_save: dict = {}                   # session -> (event, host flag)
        self._sess_load_ev: dict = {}                # session -> event of its last pre-load
        self._last_load: dict = {}                   # session -> (event, host flag)
        self._pool = _EventPool()
        self._leases: dict = {}
        self._pinned_inflight: list = []   # (pinned ids buffer, event of the copy reading it)
        # device timestamp ring (globaltimer ns) for the compute-stream timeline:
        # a CUDA timing event on the compute stream costs ~24 us while the
        # pre-loader saturates the host link (tools/event_probe.cu), a stamp
        # kernel inside the layer graph ~1 us.
        self._stamps = torch.zeros(1 << 18, dtype=torch.int64, device=self.device)
        self._stamp_pos = 0
        self._bufs = {}
        self._ws = torch.empty(0, dtype=torch.uint8, device=self.device)
        self._gemm_ws = torch.empty(gemm_workspace_bytes, dtype=torch.uint8, device=self.device)
        # L2 set-aside for the evict_last K/V rows (ASKV_L2_PERSIST_MB, default 0 = off)
        persist_mb = int(os.environ.get("ASKV_L2_PERSIST_MB", "0"))
        if persist_mb > 0:
            got = C.c_size_t()
            _lib.check(_lib.lib().askv_l2_persist(persist_mb << 20, C.byref(got)), "l2_persist")
            self.l2_persist_bytes = got.value
        if autotune:   # once per projection shape (cached in-process by the library)
            # n range: the new tokens of a reuse job (an int widens it, e.g. to
            # the full prompts of recompute jobs)
            tune_n = max_new if autotune is True else int(autotune)
            tp_n = s.n_heads * s.head_dim
            for m_, k_ in ((s.qkv_cols, s.d_model), (s.d_model, tp_n),
                           (2 * s.ffn, s.d_model), (s.d_model, s.ffn)):
                _lib.check(_lib.lib().askv_gemm_autotune(
                    m_, k_, tune_n, gemm_workspace_bytes,
                    self.s_compute.cuda_stream), "gemm_autotune")
        self._w_arrays = {
            key: _ptr_array([lw[key].data_ptr() for lw in self.w.layers])
            for key in ("w_in", "wqkv", "wo", "w_post", "wgu", "wd")}
        # tensor parallelism (config C5): tp_reduce(t, stream) sums the row-parallel
        # partials of W_o and W_down over the TP group in place (NCCL all-reduce
        # over NVLink in a multi-GPU run; dist.ThreadAllReduce in the 1-GPU emulation).
        # The native loop calls back into it between the partial GEMM and the
        # residual add.
        # A dist.NcclComm goes to the native loop as a communicator (ncclAllReduce
        # on the compute stream, captured into the layer graph, residual folded
        # into rank 0's GEMM epilogue); any other callable is a host callback.
        self.tp_reduce = tp_reduce
        self._cb_error = None
        self._nccl = getattr(tp_reduce, "native_comm", None)
        self._ar_cb = (_lib.ALLREDUCE_FN(self._allreduce)
                       if tp_reduce is not None and self._nccl is None else None)
        self.launches = 0          # libaskv kernel launches issued (all streams)
        self.probe = None          # list -> (kind, ev0, ev1, work) per probed launch

    # ------------------------------------------------------------------ buffers
    def _buf(self, name, rows, cols, dtype=BF16, zero=False):
        t = self._bufs.get(name)
        if t is None or t.shape[0] < rows or t.shape[1] != cols:
            alloc = torch.zeros if zero else torch.empty
            t = alloc((max(rows, 1), cols), dtype=dtype, device=self.device)
            self._bufs[name] = t
        return t[:rows]

    def _workspace(self, nbytes):
        if self._ws.numel() < nbytes:
            self._ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        return self._ws

    def _allreduce(self, ptr, elems, stream, ctx):
        try:
            h = self._bufs["h"].view(-1)
            if h.data_ptr() != ptr:
                raise RuntimeError("all-reduce callback on an unexpected buffer")
            self.tp_reduce(h[:elems], self.s_compute)
        except BaseException as exc:  # re-raised after the native call returns
            self._cb_error = exc

    def _stamp_slice(self, n: int) -> tuple[int, int]:
        """Reserve n ring entries; returns (offset, allocation count after)."""
        cap = self._stamps.numel()
        off = self._stamp_pos % cap
        if off + n > cap:
            self._stamp_pos += cap - off
            off = 0
        self._stamp_pos += n
        return off, self._stamp_pos

    def _stamp_values(self, off: int, end: int, n: int) -> list[int]:
        if self._stamp_pos - end + n > self._stamps.numel():
            raise RuntimeError("timeline stamps overwritten: finalize() results sooner")
        return self._stamps[off:off + n].tolist()

    def _stamp_ptr(self, off: int, i: int) -> int:
        return self._stamps.data_ptr() + 8 * (off + i)

    def probe_durations(self, probe) -> list[tuple[str, float, float, float]]:
        """(kind, seconds, algorithmic work, bytes actually moved -- K2 only)
        of each probed launch (after synchronising)."""
        out, cache = [], {}
        for kind, off, end, n, i0, i1, work, moved in probe:
            if (off, end) not in cache:
                cache[(off, end)] = self._stamp_values(off, end, n)
            v = cache[(off, end)]
            out.append((kind, (v[i1] - v[i0]) * 1e-9, work, moved))
        return out

    def _lease(self, jid):
        if not self.timeline:
            return None
        lease = self._leases.get(jid)
        if lease is None:
            lease = self._leases[jid] = _Lease(self._pool)
        return lease

    # ------------------------------------------------------------------ K1 pre-loader
    def _enqueue_loads(self, jid, job: Job):
        """Queue the job's L pre-load units for the IO thread.  Unit seq k uses
        slot k % n_slots and first waits (host flag, then the slot's ``free``
        event) for the release of unit k - n_slots, so the copy stream runs as
        far ahead as the read buffer allows -- across jobs, i.e. the
        read-buffer head start."""
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
        lease = self._lease(jid)
        load_ev = self._sess_load_ev.get(job.session_id)
        if load_ev is None:
            load_ev = self._sess_load_ev[job.session_id] = ops.NativeEvent()
        L = self.shape.layers
        for layer in range(L):
            u = _Unit()
            u.seq = self._seq
            u.slot = u.seq % self.n_slots
            u.times = (lease.get(), lease.get()) if lease else None
            u.issued = threading.Event()
            self._seq += 1
            self._units[(jid, layer)] = u
            prev = u.seq - self.n_slots
            freed = self._freed.setdefault(prev, threading.Event()) if prev >= 0 else None

            def submit(u=u, layer=layer, freed=freed, dep=dep):
                try:
                    sl = self.s_load
                    if freed is not None:   # slot reuse: its previous reader is done
                        freed.wait()
                        self._slot_free[u.slot].wait(sl)
                    if dep is not None:     # rows saved by this session's previous turn
                        dep[1].wait()
                        dep[0].wait(sl)
                    if u.times:
                        u.times[0].record(sl)
                    ops.preload_layer(self.slots[u.slot], self.host_arena.buffer, ids,
                                      self.block_bytes, layer * self.chunk_bytes,
                                      self.chunk_bytes, tail, stream=sl)
                    self._slot_ready[u.slot].record(sl)
                    if layer == L - 1:
                        load_ev.record(sl)
                    if u.times:
                        u.times[1].record(sl)
                finally:
                    u.issued.set()

            self._io_load.submit(submit)
            if layer == L - 1:
                self._last_load[job.session_id] = (load_ev, u.issued)

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
        """The slot's reader (K2) is issued and its ``free`` event recorded:
        wake the IO thread."""
        self._freed.setdefault(u.seq, threading.Event()).set()
        self._freed.pop(u.seq - 2 * self.n_slots, None)

    def _submit_saves(self, arena, job, kept, n, wslots, times, flag, sess_ev):
        """K4 for all of a job's layers from the save IO thread in one native
        call: layer l waits its write-buffer slot's ``ready`` event, copies
        the rows into the session's blocks, records the slot's ``done``."""
        L = len(wslots)
        ids = np.ascontiguousarray(np.asarray(job.block_ids, dtype=np.int64))
        src = _ptr_array([self.wbuf[w].data_ptr() for w in wslots])
        ready = _ptr_array([self._wready[w].handle for w in wslots])
        done = _ptr_array([self._wdone[w].handle for w in wslots])
        t0 = _ptr_array([a.handle for a, _ in times]) if times else None
        t1 = _ptr_array([b.handle for _, b in times]) if times else None
        base = arena.data_ptr()

        def submit():
            try:
                _lib.check(_lib.lib().askv_save_layers(
                    base, ids.ctypes.data_as(C.POINTER(C.c_int64)), len(ids), self.block_bytes,
                    self.chunk_bytes, L, self.block_tokens, self.row_bytes, job.head + kept, n,
                    src, ready, done, t0, t1, sess_ev.handle, self.s_save.cuda_stream),
                    "save_layers")
            finally:
                flag.set()

        self._io_save.submit(submit)

    def fence(self, session_id: str | None = None) -> None:
        """Block the host until the GPU copies touching the host arena are done:
        the session's last pre-load (K1) and save (K4), or with None every
        pre-load and save queued so far.  Host-side accesses to arena blocks
        (the disk tier's pwrite / pread) call this first: the copy streams run
        asynchronously to the host, and a freed block may still be the source of
        an H2D or the target of a D2H in flight."""
        if session_id is None:
            self.drain_io()
            self.s_load.synchronize()
            self.s_save.synchronize()
            return
        for dep in (self._last_save.get(session_id), self._last_load.get(session_id)):
            if dep is not None:
                dep[1].wait()
                dep[0].synchronize()

    def close(self) -> None:
        for t in (self._io_load, self._io_save):
            t.q.put(None)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------------ main entry
    def run(self, jobs: list[Job], *, want_logits: bool = False,
            batch: bool = False) -> list[JobResult]:
        """Issue all jobs back to back; returns results whose timelines are
        resolved by ``finalize`` (call after synchronising).

        batch=True: one pass over the layers for all jobs
        (askv_prefill_layers_batch): projections / norms / MLP over the jobs'
        concatenated new tokens, pre-load wait / K2 / K3 / saves per job.  A
        scheduler knob -- throughput for time to first token: every job's
        result carries the batch's timeline."""
        base = id(jobs)
        sids = [j.session_id for j in jobs]
        if len(set(sids)) != len(sids):
            raise ValueError("a session may appear once per run() call (its next turn "
                             "depends on this turn's save)")
        for i, job in enumerate(jobs):
            self._enqueue_loads((base, i), job)
        results = []
        if batch and len(jobs) > 1:
            results = self._run_batch(base, jobs, want_logits)
        else:
            for i, job in enumerate(jobs):
                results.append(self._run_job((base, i), job, want_logits))
        self.drain_io()
        return results

    def _run_batch(self, base, jobs: list[Job], want_logits: bool) -> list[JobResult]:
        s = self.shape
        L = s.layers
        if any(j.kv_cache is not None or j.source == "resident" for j in jobs):
            raise ValueError("batched jobs cannot use a resident KV cache")
        if self.tp_reduce is not None:
            raise ValueError("batched jobs cannot be tensor parallel")
        n_save = sum(1 for j in jobs if j.save)
        if n_save * L > self.n_wslots:
            raise ValueError(f"a batch of {n_save} saving jobs needs {n_save * L} write-buffer "
                             f"slots ({self.n_wslots} allocated)")
        ns = [j.n_new for j in jobs]
        tot = sum(ns)
        kv_rows = sum(j.kept + j.n_new for j in jobs)
        hq, hd = s.n_heads, s.head_dim
        big = {"x": self._buf("bx", tot, s.d_model), "h": self._buf("h", tot, s.d_model),
               "qkv": self._buf("qkv", tot, s.qkv_cols), "q": self._buf("q", tot, hq * hd),
               "ao": self._buf("ao", tot, hq * hd), "gu": self._buf("gu", tot, 2 * s.ffn),
               "act": self._buf("act", tot, s.ffn),
               # zero-initialised once: a varlen K3 reads past each job's last row
               # into the next job's (masked, P = 0) -- rows that must hold finite
               # values (0 x NaN would poison the output); they are zeros or
               # rows written by earlier passes, never uninitialised memory
               "kv": self._buf("kv", kv_rows, self.row_elems, zero=True)}
        # one attention workspace for the whole batch (its K3s run one after
        # another on the compute stream): size it for the largest job first, so
        # no job's plan keeps a pointer to a buffer a later job reallocated
        need = 0
        for j in jobs:
            sp = ops.attn_num_splits(j.kept, j.n_new, hq, n_kv_heads=s.n_kv_heads)
            need = max(need, ops.attn_workspace_bytes(j.kept, j.n_new, hq, hd, sp,
                                                      n_kv_heads=s.n_kv_heads))
        if need:
            self._workspace(need)
        plans, finishers, keep = [], [], []
        row0, kv0 = 0, 0
        probe0 = len(self.probe) if self.probe is not None else 0
        # one K3 launch for the batch (csrc/runtime.cu, ASKV_VARLEN): unless a
        # job reads its V from its own read-buffer slot (host source)
        varlen = (os.environ.get("ASKV_VARLEN", "1") != "0"
                  and not any(j.source == "host" and j.kept for j in jobs))
        for i, job in enumerate(jobs):
            sl = {k: v[row0:row0 + ns[i]] for k, v in big.items() if k != "kv"}
            sl["kv"] = big["kv"][kv0:kv0 + job.kept + job.n_new]
            p, fin, kp = self._run_job((base, i), job, want_logits, batch=sl)
            plans.append(p)
            finishers.append(fin)
            keep.append(kp)
            row0 += ns[i]
            kv0 += job.kept + job.n_new
        if varlen and self.probe is not None:
            # the batch's K3 launch stamps job 0's slots: one probe entry per
            # layer carrying every job's FLOPs
            mine = self.probe[probe0:]
            att = [e for e in mine if e[0] == "attention"]
            per_layer = {}
            for e in att:
                per_layer[e[4]] = per_layer.get(e[4], 0) + e[6]
            first = att[0][1] if att else None
            kept_att = [e[:6] + (per_layer[e[4]], 0) for e in att if e[1] == first]
            self.probe[probe0:] = [e for e in mine if e[0] != "attention"] + kept_att
        # one K2 launch per layer when every re-embedded job reads the HBM arena
        # (csrc/runtime.cu k2_batch): it stamps the first such job's slots
        k2_batch = (os.environ.get("ASKV_K2_BATCH", "1") != "0" and len(jobs) > 1
                    and any(j.kept for j in jobs)
                    and all(j.source == "hbm" for j in jobs if j.kept))
        if k2_batch and self.probe is not None:
            mine = self.probe[probe0:]
            re = [e for e in mine if e[0] == "reembed"]
            work, moved = {}, {}
            for e in re:
                work[e[4]] = work.get(e[4], 0) + e[6]
                moved[e[4]] = moved.get(e[4], 0) + e[7]
            first = re[0][1] if re else None
            kept_re = [e[:6] + (work[e[4]], moved[e[4]]) for e in re if e[1] == first]
            self.probe[probe0:] = [e for e in mine if e[0] != "reembed"] + kept_re
        arr = (_lib.PrefillPlan * len(plans))(*plans)
        _lib.check(_lib.lib().askv_prefill_layers_batch(C.addressof(arr), len(plans),
                                                        self.s_compute.cuda_stream),
                   "prefill_layers_batch")
        results = [fin() for fin in finishers]
        lead = results[0]
        for r in results[1:]:    # the layer timeline is the batch's (job 0's stamps)
            r._batch_leader = lead
        del keep
        return results

    def drain_io(self) -> None:
        """Wait until the IO threads have submitted everything queued so far, so
        a later device synchronise covers this run's loads and saves."""
        for t in (self._io_load, self._io_save):
            done = threading.Event()
            t.submit(done.set)
            _await(done, t.name)
            if t.error is not None:
                raise RuntimeError(f"{t.name} failed") from t.error

    def _run_job(self, jid, job: Job, want_logits: bool, batch: dict | None = None):
        s = self.shape
        L = s.layers
        n, kept = job.n_new, job.kept
        if n < 1:
            raise ValueError("a job needs at least one new token")
        if job.save and n > self.max_new:
            raise ValueError(f"{n} saved rows exceed the write-buffer slot ({self.max_new})")
        if kept + n > self.table.max_pos:
            raise ValueError("context exceeds the runner's RoPE table")
        if job.save and len(job.block_ids) * self.block_tokens < job.head + kept + n:
            raise ValueError("save needs block_ids covering kept + new rows")
        if job.source == "resident":
            if job.kv_cache is None or job.kv_cache.rows != kept:
                raise ValueError("resident job needs kv_cache holding exactly its kept rows")
        elif kept and job.source not in ("host", "hbm"):
            raise ValueError(f"job with kept={kept} needs a source")
        if kept and job.source == "hbm" and job.dev_block_off is None:
            raise ValueError("hbm job needs dev_block_off")
        arena = None
        in_hbm = False
        if job.save:
            # an "hbm" job whose session lives in the HBM arena (bench value
            # mode) saves there; an HBM-tier hit (mirror_block_ids set) keeps
            # host DRAM as the backing store -- its block ids are host blocks --
            # and the tier copy is the in-loop write-through
            in_hbm = job.source == "hbm" and job.mirror_block_ids is None
            arena = self.hbm_arena if in_hbm else (
                self.host_arena.buffer if self.host_arena is not None else None)
            if arena is None:
                raise RuntimeError("save requested but no arena for it")
        hd, hq, hkv = s.head_dim, s.n_heads, s.n_kv_heads
        cs = self.s_compute
        lease = self._lease(jid)
        self._leases.pop(jid, None)
        # stamp slice: [0] job begin, [1] job end, [2:] the native loop's stamps
        n_st = 3 + 7 * L
        st_off, st_end = self._stamp_slice(n_st) if (lease or self.probe is not None) \
            else (0, 0)
        keep = []                       # ctypes arrays alive through the native call

        def arr(items):
            a = _ptr_array(items)
            keep.append(a)
            return a

        first = torch.empty(1, dtype=torch.int64, pin_memory=True)
        logits_out = None
        rec = {"saves": [], "loads": []}
        # device inputs the caller made on its own stream (token ids, the HBM
        # tier's block offsets) must land before the job reads them: torch
        # streams are non-blocking, nothing else orders them
        caller = torch.cuda.current_stream(self.device)
        with torch.cuda.stream(cs):
            if caller.cuda_stream != cs.cuda_stream:
                cs.wait_stream(caller)
            # ... and stay allocated until the job's kernels have read them: the
            # caching allocator only knows the stream they were made on, so a
            # freed offsets tensor could otherwise be handed out (and
            # overwritten) while K2 is still queued on the compute stream
            for t in (job.dev_block_off, job.token_ids):
                if t is not None and t.is_cuda:
                    t.record_stream(cs)
            if job.source == "hbm" or job.mirror_block_ids is not None:
                # HBM-tier rows written by this session's previous saves (save
                # stream), and blocks reassigned from other sessions whose
                # write-through saves may still be in flight
                for sid in {job.session_id, *job.fence_sessions}:
                    dep = self._last_save.get(sid)
                    if dep is not None:
                        _await(dep[1], "save IO thread")
                        dep[0].wait(cs)

            units = None
            if kept and job.source == "host":
                units = [self._acquire(jid, l) for l in range(L)]
                k = L if job.prestage else min(L, max(0, int(job.prestage_layers)))
                if k:   # head start: layers 0..k-1 resident before the job begins
                    self._slot_ready[units[k - 1].slot].wait(cs)
            t0 = lease.get() if lease else None
            if t0:   # one timing event: the base of the copy streams' intervals
                _lib.check(_lib.lib().askv_stamp(self._stamp_ptr(st_off, 0), cs.cuda_stream),
                           "stamp")
                t0.record(cs)
            if job.token_ids.is_cuda:
                ids = job.token_ids
            else:  # pinned host ids: SM copy, not behind the pre-load DMAs
                src = job.token_ids if job.token_ids.is_pinned() else job.token_ids.pin_memory()
                src = src.to(torch.int64)
                ids = ops.copy_sm(torch.empty(n, dtype=torch.int64, device=self.device),
                                  src, stream=cs)
                self.launches += 1
                # torch's pinned-memory cache cannot see our kernel read the
                # staging buffer: hold it until the copy has run (a freed block
                # could be handed to the next job's ids before it does)
                done = torch.cuda.Event()
                done.record(cs)
                self._pinned_inflight = [(t, e) for t, e in self._pinned_inflight
                                         if not e.query()]
                self._pinned_inflight.append((src, done))
            if batch is None:
                x = F.embedding(ids, self.w.embed)
                buf = lambda name, rows, cols: self._buf(  # noqa: E731
                    name, rows, cols, zero=name == "kv")   # shared with batched passes
            else:   # this job's rows of the batch's shared buffers
                x = batch["x"]
                torch.index_select(self.w.embed, 0, ids, out=x)
                buf = lambda name, rows, cols: batch[name]  # noqa: E731
            buf("h", n, s.d_model)
            splits = ops.attn_num_splits(kept, n, hq, n_kv_heads=hkv)
            wsb = ops.attn_workspace_bytes(kept, n, hq, hd, splits, n_kv_heads=hkv)
            ws = self._workspace(wsb) if wsb else None

            p = _lib.PrefillPlan()
            p.layers, p.d_model, p.n_heads, p.n_kv_heads = L, s.d_model, hq, hkv
            p.head_dim, p.ffn, p.n_new, p.kept, p.head = hd, s.ffn, n, kept, job.head
            p.rms_eps, p.attn_scale, p.attn_splits = 1e-5, 1.0 / math.sqrt(hd), splits
            wa = self._w_arrays
            p.w_in, p.w_qkv, p.w_o = wa["w_in"], wa["wqkv"], wa["wo"]
            p.w_post, p.w_gu, p.w_down = wa["w_post"], wa["wgu"], wa["wd"]
            p.x = x.data_ptr()
            p.h = buf("h", n, s.d_model).data_ptr()
            p.qkv = buf("qkv", n, s.qkv_cols).data_ptr()
            p.q_rot = buf("q", n, hq * hd).data_ptr()
            if job.kv_cache is not None:
                if kept + n > job.kv_cache.capacity:
                    raise ValueError("context exceeds the resident KV capacity")
                p.kv_layers = arr(job.kv_cache.layer_ptrs())
            else:
                p.kv = buf("kv", kept + n, self.row_elems).data_ptr()
                if (batch is None and self.overlap and kept and job.source in ("host", "hbm")
                        and job.promote_block_ids is None and self.tp_reduce is None):
                    p.kv_alt = self._buf("kv2", kept + n, self.row_elems).data_ptr()
                    rec["overlap"] = True
            p.attn_out = buf("ao", n, hq * hd).data_ptr()
            p.gu = buf("gu", n, 2 * s.ffn).data_ptr()
            p.act = buf("act", n, s.ffn).data_ptr()
            if ws is not None:
                p.attn_ws, p.attn_ws_bytes = ws.data_ptr(), ws.numel()
            p.gemm_ws, p.gemm_ws_bytes = self._gemm_ws.data_ptr(), self._gemm_ws.numel()
            p.rope_table = self.table.table.data_ptr()
            p.rope_positions = self.table.max_pos
            p.block_tokens = self.block_tokens
            p.src_row_stride = self.row_elems
            p.block_bytes, p.chunk_bytes, p.row_bytes = (self.block_bytes, self.chunk_bytes,
                                                         self.row_bytes)
            if units is not None:
                p.src_kind = 1
                p.src_rows = self.slot_rows    # K3 reads the kept rows' V in the slot
                p.src_layer = arr([self.slots[u.slot].data_ptr() for u in units])
                p.ev_src_ready = arr([self._slot_ready[u.slot].handle for u in units])
                p.ev_src_free = arr([self._slot_free[u.slot].handle for u in units])
                if job.promote_block_ids is not None:   # into the HBM tier
                    ids64 = (C.c_int64 * len(job.promote_block_ids))(*job.promote_block_ids)
                    keep.append(ids64)
                    p.promote_base = self.hbm_arena.data_ptr()
                    p.promote_block_ids = ids64
                    p.promote_nblocks = len(job.promote_block_ids)
                for u in units:
                    if u.times:
                        rec["loads"].append(u.times)
            elif kept and job.source == "hbm":
                p.src_kind = 2
                base = self.hbm_arena.data_ptr()
                p.src_rows = self.hbm_arena.numel() * 2 // self.row_bytes
                p.src_layer = arr([base + l * self.chunk_bytes for l in range(L)])
                p.src_block_off = job.dev_block_off.data_ptr()
            # a session living in the HBM arena saves there inside the layer
            # loop (device-to-device, in stream order, captured in the graph):
            # no saver IO-thread work per layer
            save_in_loop = job.save and in_hbm
            if (job.save and job.mirror_block_ids is not None) or save_in_loop:
                # HBM tier write-through (or the arena save itself) inside the
                # layer loop (compute-stream order with promotions and K2 reads)
                tgt = job.block_ids if save_in_loop else job.mirror_block_ids
                mids = (C.c_int64 * len(tgt))(*tgt)
                keep.append(mids)
                p.mirror_base = self.hbm_arena.data_ptr()
                p.mirror_block_ids = mids
                p.mirror_nblocks = len(tgt)
            wslots = []
            if job.save:
                for _ in range(L):
                    w = self._wseq % self.n_wslots
                    self._wseq += 1
                    if self._wflag[w] is not None:   # its previous save is submitted
                        _await(self._wflag[w], "save IO thread")
                    wslots.append(w)
                p.save_rows = arr([self.wbuf[w].data_ptr() for w in wslots])
                if not save_in_loop:
                    p.ev_save_free = arr([self._wdone[w].handle for w in wslots])
                    p.ev_save_ready = arr([self._wready[w].handle for w in wslots])
            reemb = bool(kept) and job.source != "resident"
            if lease or self.probe is not None:
                p.stamps = self._stamp_ptr(st_off, 2)
                p.stamp_flags = (1 if lease else 0) | (2 if self.probe is not None else 0)
                rec["waited"] = reemb and units is not None
            if self.probe is not None:
                # K2's work: SURVEY §8(d) counts read K + write K (kept rows, the
                # K half of each row); V rows of whole 128-row tiles stay where
                # the pre-loader left them (K3 reads them there), the rest are copied
                v_src = (p.src_rows > 0 and job.kv_cache is None and
                         (p.src_kind == 1 or (p.src_kind == 2 and job.head == 0
                                              and self.block_tokens == 128)))
                v_copy = kept - (kept // 128) * 128 if v_src else kept
                k2_moved = kept * s.row_bytes + v_copy * s.row_bytes
                for l in range(L):
                    b = 2 + 1 + 7 * l
                    if reemb:
                        self.probe.append(("reembed", st_off, st_end, n_st, b + 3, b + 4,
                                           kept * s.row_bytes, k2_moved))
                    self.probe.append(("attention", st_off, st_end, n_st, b + 5, b + 6,
                                       attention_flops(kept, n, hq, hd), 0))
            if self._ar_cb is not None:
                p.allreduce = self._ar_cb
            elif self._nccl is not None:
                p.nccl_comm, p.tp_rank = self._nccl.handle, self._nccl.rank
            p.graph = 1 if self.graph else 0
            self._cb_error = None
            if batch is None:
                _lib.check(_lib.lib().askv_prefill_layers(C.addressof(p), cs.cuda_stream),
                           "prefill_layers")
            if self._cb_error is not None:
                raise RuntimeError("tensor-parallel all-reduce failed") from self._cb_error

        def finish() -> JobResult:
          nonlocal logits_out
          with torch.cuda.stream(cs):
            n_stamps = 0
            if lease:   # job begin / end + the last layer's end (the rest ride on kernels)
                n_stamps += 3
            self.launches += L * (4 + (1 if kept and job.source != "resident" else 0)
                                  + (2 if splits > 1 else 1)
                                  + (2 if self._ar_cb is not None else 0)) + n_stamps
            if units is not None:
                for u in units:
                    self._release(u)
            if save_in_loop:   # saved by the loop itself: later readers follow in stream order
                for w in wslots:
                    self._wflag[w] = None
                self._last_save.pop(job.session_id, None)
            elif job.save:
                sess_ev = self._sess_ev.get(job.session_id)
                if sess_ev is None:
                    sess_ev = self._sess_ev[job.session_id] = ops.NativeEvent()
                # every layer's save in one submission (askv_save_layers)
                flag = threading.Event()
                times = [(lease.get(), lease.get()) for _ in wslots] if lease else None
                for w in wslots:
                    self._wflag[w] = flag
                self._submit_saves(arena, job, kept, n, wslots, times, flag, sess_ev)
                if times:
                    rec["saves"].extend((t0_, t1_, flag) for t0_, t1_ in times)
                self._last_save[job.session_id] = (sess_ev, flag)
            hl = ops.rmsnorm(x[-1:], self.w.w_final, 1e-5, stream=cs)
            logits = F.linear(hl, self.w.lm_head).float()
            nxt = logits.argmax(dim=-1)
            ops.copy_sm(first, nxt, stream=cs)
            self.launches += 2
            if want_logits:
                logits_out = logits[0].clone()
            if lease:
                _lib.check(_lib.lib().askv_stamp(self._stamp_ptr(st_off, 1), cs.cuda_stream),
                           "stamp")
          res = JobResult(job.session_id, kept, n, None, first, logits_out,
                          bytes_loaded=(kept * s.kv_bytes_per_token if job.source == "host"
                                        else 0),
                          bytes_saved=n * s.kv_bytes_per_token if job.save else 0,
                          next_token=nxt)
          if job.kv_cache is not None:
              job.kv_cache.rows = kept + n
          res._events = (self, t0, (st_off, st_end, n_st), rec, lease) if lease else None
          return res

        if batch is not None:
            return p, finish, keep
        return finish()

    def join(self) -> None:
        """Make the compute stream wait for all loads and saves queued so far
        (waits for the IO threads to submit them first)."""
        self.drain_io()
        self.s_compute.wait_stream(self.s_load)
        self.s_compute.wait_stream(self.s_save)

    # ------------------------------------------------------------------ timelines
    @staticmethod
    def finalize(results: list[JobResult]) -> None:
        """Resolve CUDA events into seconds (call after synchronising).  The
        members of a batch (run(..., batch=True)) get the batch's timeline."""
        members = [r for r in results if getattr(r, "_batch_leader", None) is not None]
        for r in results:
            evs = getattr(r, "_events", None)
            if not evs or getattr(r, "_batch_leader", None) is not None:
                continue
            runner, t0, (off, end, n_st), rec, lease = evs
            ms = C.c_float()
            lib = _lib.lib()

            def f(e):   # copy-stream timing event -> seconds after job begin
                h = e if isinstance(e, int) else e.handle
                _lib.check(lib.askv_event_elapsed_ms(t0.handle, h, C.byref(ms)), "elapsed")
                return float(ms.value) * 1e-3

            v = runner._stamp_values(off, end, n_st)
            g = lambda i: (v[i] - v[0]) * 1e-9  # noqa: E731  compute-stream stamp -> seconds

            tl = Timeline()
            tl.makespan = g(1)
            L = (n_st - 3) // 7
            tl.load_intervals = [(f(a), f(b)) for a, b in rec["loads"]]
            for *_, flag in rec["saves"]:
                _await(flag, "save IO thread")
            tl.save_intervals = [(f(a), f(b)) for a, b, _ in rec["saves"]]
            comp, waits = [], []
            begin = g(2)
            for l in range(L):
                b = 3 + 7 * l
                end_l = g(b)
                if rec.get("waited"):   # rope_new end -> K2 begin (K3 begin when overlapped)
                    wa, wb = g(b + 1), g(b + (5 if rec.get("overlap") else 3))
                    waits.append((wa, wb))
                    comp.extend([(begin, wa), (wb, end_l)])
                else:
                    comp.append((begin, end_l))
                begin = end_l
            stall = sum(b - a for a, b in waits)
            tl.compute_intervals = comp
            tl.stall_total = stall if stall > 1e-9 else 0.0
            tl.max_gap = max((b - a for a, b in waits), default=0.0)
            r.timeline = tl
            r._events = None
        for r in members:
            lead = r._batch_leader
            if lead.timeline is None and getattr(lead, "_events", None):
                Runner.finalize([lead])
            r.timeline = lead.timeline
            r._events = None
