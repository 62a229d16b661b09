"""Per-turn shapes replayed from the committed session fixtures.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The session lists come from the reference generator (trace.py:326-356) via
tests/golden/make_golden.py; the per-turn (kept, new, hit) follow
oracle.layout_ref.replay_session (sim.py:408-483, 519-581) and are pinned
against the reference simulator's own TurnRecords stored in the same fixture.
"""

from __future__ import annotations

import json
from pathlib import Path

from oracle.layout_ref import TurnShape, replay_session

GOLDEN = Path(__file__).resolve().parent.parent / "tests" / "golden"


def load(name: str) -> dict:
    return json.loads((GOLDEN / f"workload_{name}.json").read_text())


def shapes(name: str) -> list[TurnShape]:
    wl = load(name)
    out = []
    for s in wl["sessions"]:
        out.extend(replay_session(s["id"], s["turns"], wl["window"],
                                  wl["truncation_ratio"]))
    return out


def long_context_shapes(history: int = 32768, turns: int = 6, new: int = 256,
                        output: int = 64, window: int = 4096, ratio: float = 0.5):
    """Config C4: a stored 32K history then `turns` of 256 in / 64 out
     at W = 4096."""
    return replay_session("long", [(new, output)] * turns, window, ratio,
                          initial_context=history)
