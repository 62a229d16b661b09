"""Per-job load / compute / save timelines — measured, not modeled.

The reference plans these analytically (/root/reference/pkg/src/kvsim/overlap.py:
Timeline :31-66, plan_preload :69-123, plan_async_save :126-200) and the
simulator charges ``Timeline.makespan`` as the prefill time and
``stall_total`` as the exposed transfer (sim.py:448-449).  The B200 engine
produces the same ``Timeline`` from CUDA events recorded on the copy, compute
and save streams:

* t = 0 is the moment the job owns the execution stream (the previous job's
  last layer finished), as in overlap.py:3-5;
* load_intervals: per-layer H2D DMA windows of the pre-loader (may start
  before 0 — that is the read-buffer head start);
* compute_intervals: per-layer execution windows;
* stall_total: time the compute stream spent blocked on pre-load events
  (= makespan - compute time, overlap.py:118);
* save_intervals: per-layer D2H windows of the asynchronous saver.
"""

from __future__ import annotations

import json
from dataclasses import dataclass, field


@dataclass
class Timeline:
    load_intervals: list[tuple[float, float]] = field(default_factory=list)
    compute_intervals: list[tuple[float, float]] = field(default_factory=list)
    save_intervals: list[tuple[float, float]] = field(default_factory=list)
    stall_total: float = 0.0
    max_gap: float = 0.0
    makespan: float = 0.0

    @property
    def compute_total(self) -> float:
        return sum(e - s for s, e in self.compute_intervals)

    @property
    def load_total(self) -> float:
        return sum(e - s for s, e in self.load_intervals)

    @property
    def save_total(self) -> float:
        return sum(e - s for s, e in self.save_intervals)

    @property
    def save_overrun(self) -> float:
        """Save time extending past the makespan (overlap.py:193-199)."""
        if not self.save_intervals:
            return 0.0
        return max(0.0, max(e for _, e in self.save_intervals) - self.makespan)

    def to_dict(self) -> dict:
        return {"load_intervals": self.load_intervals,
                "compute_intervals": self.compute_intervals,
                "save_intervals": self.save_intervals, "stall_total": self.stall_total,
                "max_gap": self.max_gap, "makespan": self.makespan}

    def to_json(self) -> str:
        return json.dumps(self.to_dict())


def ms_to_s(x: float) -> float:
    return x * 1e-3


# ---------------------------------------------------------------------------
# The reference's planner entry points, measured.
# overlap.py:69-72 / :126-128 signatures; bind() a measured.MeasuredExecutor
# (an engine on this process's GPU) first -- there is no analytical fallback.

_executor = None


def bind(executor) -> None:
    """Route plan_preload / plan_async_save to `executor`
    (measured.MeasuredExecutor); None unbinds."""
    global _executor
    _executor = executor


def _bound():
    if _executor is None:
        raise RuntimeError("overlap: no engine bound; call overlap.bind("
                           "measured.MeasuredExecutor(engine)) first")
    return _executor


def plan_preload(hist_tokens: int, new_tokens: int, profile, tiers, read_buffer: float,
                 prev_job_running: bool = True, *, bandwidth: float | None = None,
                 job=None) -> Timeline:
    """Run one job's layer-wise pre-load + prefill on the GPU and return its
    measured Timeline (overlap.py:69-123 plans it analytically).  Same
    argument checks as the reference (overlap.py:79-82)."""
    if hist_tokens < 0 or new_tokens < 0:
        raise ValueError("token counts must be >= 0")
    if read_buffer < 0:
        raise ValueError("read_buffer must be >= 0")
    return _bound().plan_preload(hist_tokens, new_tokens, profile, tiers, read_buffer,
                                 prev_job_running, bandwidth=bandwidth, job=job)


def plan_async_save(prompt_tokens: int, decode_steps: int, profile, tiers,
                    write_buffer: float, *, bandwidth: float | None = None,
                    job=None) -> Timeline:
    """Measured write-back Timeline of a job (overlap.py:126-200)."""
    if prompt_tokens < 0 or decode_steps < 0:
        raise ValueError("token counts must be >= 0")
    if write_buffer < 0:
        raise ValueError("write_buffer must be >= 0")
    return _bound().plan_async_save(prompt_tokens, decode_steps, profile, tiers, write_buffer,
                                    bandwidth=bandwidth, job=job)
