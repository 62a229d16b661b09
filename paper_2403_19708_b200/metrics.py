"""Metric definitions reused from the reference (for reporting measured runs).

  percentile         metrics.py:87-97  (linear interpolation on sorted values)
  prefill_throughput metrics.py:118-119, 142  (sum prompt tokens / sum prefill s)
"""

from __future__ import annotations

import math


def percentile(values, q: float) -> float:
    v = sorted(values)
    if not v:
        return 0.0
    if len(v) == 1:
        return v[0]
    pos = q * (len(v) - 1)
    lo = int(math.floor(pos))
    hi = min(lo + 1, len(v) - 1)
    frac = pos - lo
    return v[lo] * (1 - frac) + v[hi] * frac


def prefill_throughput(prompt_tokens, prefill_seconds) -> float:
    tot = sum(prefill_seconds)
    return sum(prompt_tokens) / tot if tot else 0.0


def summarize(log) -> dict:
    """The reference's per-run report (metrics.py:100-156: hit rates over
    non-first evaluated turns, mean / p50 / p99 TTFT, prefill throughput)
    plus the exposed-transfer fraction of the measured prefills
    (sum stall / sum prefill, overlap.py:118) and p50 TTFT per hit class."""
    unfinished = [t for t in log.turns if math.isnan(t.done)]
    if unfinished:
        raise ValueError(f"{len(unfinished)} turn(s) unfinished")
    ev = [t for t in log.turns if not t.warmup]
    el = [t for t in ev if not t.is_first_turn]
    mem = sum(1 for t in el if t.hit_class == "memory_hit")
    disk = sum(1 for t in el if t.hit_class == "disk_hit")
    d = len(el)
    ttft = [t.ttft_s for t in ev]
    pre = sum(t.prefill_s for t in ev)
    by = {}
    for cls in ("memory_hit", "disk_hit", "miss"):
        v = [t.ttft_s for t in ev if t.hit_class == cls]
        if v:
            by[cls] = {"turns": len(v), "p50_ttft_s": percentile(v, 0.5),
                       "p50_prefill_s": percentile([t.prefill_s for t in ev
                                                    if t.hit_class == cls], 0.5)}
    return {
        "turns": len(ev), "hit_denominator": d,
        "overall_hit_rate": (mem + disk) / d if d else 0.0,
        "mem_hit_rate": mem / d if d else 0.0, "disk_hit_rate": disk / d if d else 0.0,
        "mean_ttft_s": sum(ttft) / len(ttft) if ttft else 0.0,
        "p50_ttft_s": percentile(ttft, 0.5), "p99_ttft_s": percentile(ttft, 0.99),
        "p50_prefill_s": percentile([t.prefill_s for t in ev], 0.5),
        "prefill_tokens_per_s": prefill_throughput([t.prompt_tokens for t in ev],
                                                   [t.prefill_s for t in ev]),
        "exposed_transfer_frac": (sum(t.stall_s for t in ev) / pre) if pre else 0.0,
        "by_hit_class": by,
        "evict_out": log.meta.get("evict_out_count", 0),
        "evict_to_disk": log.meta.get("evict_to_disk_count", 0),
        "sim_wall_time_s": log.meta.get("wall_time_s", 0.0),
    }
