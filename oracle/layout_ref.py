"""Integer arithmetic of truncation and block accounting.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference anchors:
* load-time overflow truncation  sim.py:468-483 (_handle_overflow)
* save-time truncation           sim.py:576-581 (_truncate_tokens)
* save context arithmetic        sim.py:528-529
* hit / miss at job start        sim.py:414-443
* KV bytes                       model.py:243-247 (kv_size)
* block-granular charge          store.py:100-102 (KvStore.charge)
"""

from __future__ import annotations

import math
from dataclasses import dataclass


def cut_tokens(window: int, ratio: float) -> int:
    """Truncation chunk: max(1, int(ratio * W))  (sim.py:471, 578)."""
    return max(1, int(ratio * window))


def overflow_kept(hist: int, new: int, window: int, ratio: float) -> int:
    """Kept history after load-time truncation (sim.py:468-474).

    Drops ``cut`` tokens from the front until kept + new fits, or kept == 0.
    """
    if hist + new <= window:
        return hist
    cut = cut_tokens(window, ratio)
    kept = hist
    while kept > 0 and kept + new > window:
        kept = max(0, kept - cut)
    return kept


def save_truncate(tokens: int, window: int, ratio: float) -> int:
    """Context kept at save time: subtract cut while > W (sim.py:576-581)."""
    cut = cut_tokens(window, ratio)
    while tokens > window:
        tokens -= cut
    return max(tokens, 0)


def kv_size(tokens: int, kv_bytes_per_token: float) -> float:
    """model.py:243-247."""
    if tokens < 0:
        raise ValueError("tokens must be >= 0")
    return tokens * kv_bytes_per_token


def charge(nbytes: float, block_bytes: int) -> int:
    """store.py:100-102: ceil(bytes / block) * block."""
    return int(math.ceil(nbytes / block_bytes)) * block_bytes


def blocks_for(tokens: int, block_tokens: int) -> int:
    return -(-tokens // block_tokens)


@dataclass(frozen=True)
class TurnShape:
    session_id: str
    turn: int
    hist_raw: int      # context before this turn's load-time truncation
    kept: int          # history reused (0 on a miss)
    drop: int          # front tokens dropped by load-time truncation
    new: int
    output: int
    hit: bool
    overflowed: bool

    @property
    def prompt(self) -> int:
        return self.kept + self.new


def replay_session(session_id: str, turns, window: int, ratio: float,
                   initial_context: int = 0):
    """Per-turn shapes for one session assuming the store never evicts.

    Mirrors _start_job / _finish_job (sim.py:408-443, 519-555) for a store
    with unlimited capacity and TTL: turn 0 is a miss, later turns hit unless
    overflow truncation left kept == 0 (the item is removed, sim.py:476-477).
    ``initial_context`` models a pre-stored history (config C4).
    """
    out = []
    ctx = initial_context
    for k, (new, outp) in enumerate(turns):
        hist = ctx
        overflowed = hist + new > window
        kept = overflow_kept(hist, new, window, ratio) if overflowed else hist
        hit = (k > 0 or initial_context > 0) and kept > 0
        # ``kept`` is the truncated context either way; a miss recomputes all
        # prompt = kept + new tokens (sim.py:420, 432-434).
        out.append(TurnShape(session_id, k, hist, kept, hist - kept, new, outp,
                             hit, overflowed))
        ctx = save_truncate(kept + new + outp, window, ratio)
    return out
