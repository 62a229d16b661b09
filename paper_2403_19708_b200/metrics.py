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
