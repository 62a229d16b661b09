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
