"""The serving loop (paper_2403_19708_b200.sim) and placement policy
(paper_2403_19708_b200.policy) replay the reference simulator bit-exact.

Golden logs: tests/golden/sim_c2.json, produced by running the reference's own
sim.run on capacity-constrained C2 configurations (make_golden.py
sim_golden): scheduler-aware with a disk tier, without one, with explicit
windows, and the LRU baseline.  Here the same loop runs with the analytical
planners of the oracle (oracle/overlap_ref.py, itself pinned to the
reference's overlap.py) as its executor, so every evict_to_disk / evict_out /
prefetch decision, its order and its time, and every turn's hit class and
TTFT, must come out identical.  On the GPU the executor is the measured engine
(tests/test_measured_gpu.py); the policy and loop are this code either way.
"""

import json
import math
from pathlib import Path

import pytest

from oracle import overlap_ref
from paper_2403_19708_b200 import model, policy, sim

G = Path(__file__).resolve().parent / "golden"
GOLD = json.loads((G / "sim_c2.json").read_text())


class _Plan:
    def __init__(self, d):
        self.makespan = d["makespan"]
        self.stall_total = d["stall_total"]


class ModeledExecutor:
    """overlap.plan_preload / plan_async_save (analytical, oracle restatement)."""

    def plan_preload(self, hist, new, profile, tiers, read_buffer, prev_job_running=True, *,
                     bandwidth=None, job=None):
        return _Plan(overlap_ref.plan_preload(
            hist, new, kv_bytes_per_token=profile.kv_bytes_per_token,
            prefill_s_per_token=profile.prefill_seconds_per_token, layers=profile.layers,
            bandwidth=bandwidth if bandwidth is not None else tiers.pcie_bandwidth,
            read_buffer=read_buffer, prev_job_running=prev_job_running))

    def plan_async_save(self, prompt, steps, profile, tiers, write_buffer, *, bandwidth=None,
                        job=None):
        return _Plan(overlap_ref.plan_async_save(
            prompt, steps, kv_bytes_per_token=profile.kv_bytes_per_token,
            prefill_s_per_token=profile.prefill_seconds_per_token,
            decode_s_per_step=profile.decode_seconds_per_step,
            bandwidth=bandwidth if bandwidth is not None else tiers.pcie_bandwidth,
            write_buffer=write_buffer))


def _run(name):
    case = GOLD[name]
    c = case["case"]
    prof = model.ModelProfile(name="7b", kv_bytes_per_token=float(case["kv_bytes_per_token"]),
                              prefill_seconds_per_token=6e-5, decode_seconds_per_step=6e-3,
                              context_window=4096, layers=32)
    tiers = model.TierConfig(hbm_read_buffer=int(4e9), hbm_write_buffer=int(2e9),
                             dram_capacity=int(c["dram"]), disk_capacity=int(c["disk"]),
                             pcie_bandwidth=55e9, disk_bandwidth=3.2e9)
    pol = policy.PolicyConfig(kind=policy.PolicyKind(c["policy"]),
                              prefetch_window=c.get("prefetch_window"),
                              eviction_window=c.get("eviction_window"))
    cfg = sim.SimConfig(profile=prof, tiers=tiers, policy=pol, mode=sim.Mode.REUSE,
                        block_bytes=case["block_bytes"])
    wl = sim.load_workload(G / "workload_c2.json")
    return case, sim.run(wl, cfg, ModeledExecutor())


def _close(a, b):
    return a == b or (math.isfinite(a) and abs(a - b) <= 1e-9 * max(1.0, abs(b)))


@pytest.mark.parametrize("name", sorted(GOLD))
def test_event_log_matches_reference(name):
    case, log = _run(name)
    want = case["events"]
    got = [e.to_dict() for e in log.events]
    assert len(got) == len(want)
    for i, (g, w) in enumerate(zip(got, want)):
        # identical decision, order and subject; times / byte counts equal
        assert (g["kind"], g["session"], g["turn"], g.get("action"), g.get("hit")) == \
            (w["kind"], w["session"], w["turn"], w.get("action"), w.get("hit")), i
        assert _close(g["time"], w["time"]), (i, g, w)
        for k in ("bytes", "ttft"):
            if k in w:
                assert _close(g[k], w[k]), (i, k, g, w)


@pytest.mark.parametrize("name", sorted(GOLD))
def test_turn_records_and_meta_match_reference(name):
    case, log = _run(name)
    assert len(log.turns) == len(case["turns"])
    for t, w in zip(log.turns, case["turns"]):
        assert (t.session_id, t.turn_index, t.hit_class, t.prompt_tokens) == \
            (w["session"], w["turn"], w["hit"], w["prompt"])
        for a, b in ((t.ttft_s, w["ttft"]), (t.prefill_s, w["prefill"]),
                     (t.stall_s, w["stall"]), (t.done, w["done"]),
                     (t.bytes_evicted, w["evicted"])):
            assert _close(a, b), (t.session_id, t.turn_index, a, b)
    for k in ("evict_out_count", "evict_to_disk_count", "turns"):
        assert log.meta[k] == case["meta"][k], k
    for k in ("bytes_evicted", "wall_time_s", "engine_prefill_busy_s", "engine_decode_busy_s"):
        assert _close(log.meta[k], case["meta"][k]), k


def test_golden_cases_exercise_every_policy_decision():
    """The fixture must actually contain demotions, disk drops and prefetches
    (otherwise the order checks above prove little)."""
    kinds = {(e["kind"], e.get("action")) for c in GOLD.values() for e in c["events"]}
    assert {("evict_done", "evict_to_disk"), ("evict_done", "evict_out"),
            ("prefetch_done", None)} <= kinds
    hits = {t["hit"] for c in GOLD.values() for t in c["turns"]}
    assert hits == {"miss", "memory_hit", "disk_hit"}


def test_job_queue_positions_and_windows():
    q = policy.JobQueue()
    for i, s in enumerate("abcde"):
        q.push(s, 0, float(i))
    assert [q.position_of(s) for s in "abcde"] == [0, 1, 2, 3, 4]
    assert q.pop().session_id == "a"
    assert q.position_of("a") is None and q.position_of("c") == 1
    assert [e.session_id for e in q.window(2)] == ["b", "c"]
    with pytest.raises(ValueError):
        q.push("b", 1, 9.0)          # one waiting job per session
    with pytest.raises(ValueError):
        q.push("z", 0, 1.0)          # time order


def test_victim_ranking_matches_reference_key():
    """policy.py:159-172: never-queued (coldest first) < queued beyond the
    window (latest position first) < windowed (tail first, larger first)."""
    from paper_2403_19708_b200.store import KvStore

    prof = model.ModelProfile(name="p", kv_bytes_per_token=1.0, prefill_seconds_per_token=1e-4,
                              decode_seconds_per_step=1e-3, context_window=4096, layers=2)
    st = KvStore(prof, model.TierConfig(dram_capacity=10**6, disk_capacity=0), block_bytes=1)
    for i, (sid, tok) in enumerate([("cold", 10), ("warm", 10), ("q0", 30), ("q1", 20),
                                    ("q2", 40), ("q3", 10)]):
        st.save(sid, tok, float(i))
    q = policy.JobQueue()
    for i, s in enumerate(["q0", "q1", "q2", "q3"]):
        q.push(s, 1, float(i))
    cfg = policy.PolicyConfig(eviction_window=2)
    order = []
    while st.items:
        v = policy.select_evict_to_disk(q, st, cfg)
        order.append(v)
        st.remove(v)
    assert order == ["cold", "warm", "q3", "q2", "q1", "q0"]


@pytest.mark.skipif(not Path("/root/reference/pkg/src/kvsim").exists(),
                    reason="reference package not present (GPU box)")
def test_planner_dropin_rebinds_into_the_reference_simulator():
    """overlap.plan_preload / plan_async_save have the reference signatures:
    rebinding kvsim.sim's planners to them (bound here to the analytical
    executor; on a GPU to measured.MeasuredExecutor) leaves the reference
    simulator's C1 event log unchanged."""
    import sys

    sys.path.insert(0, "/root/reference/pkg/src")
    try:
        import kvsim.model as kmodel
        import kvsim.sim as ksim
        import kvsim.trace as ktrace
    finally:
        sys.path.remove("/root/reference/pkg/src")
    from paper_2403_19708_b200 import overlap

    wl_raw = json.loads((G / "workload_c1.json").read_text())
    sessions = [ktrace.Session(s["id"], [ktrace.Turn(a, b) for a, b in s["turns"]],
                               list(s["arrivals"])) for s in wl_raw["sessions"]]
    wl = ktrace.Workload(sessions)
    prof = kmodel.builtin_profile("llama-13b")
    cfg = ksim.SimConfig(profile=prof)

    def events():
        return [(e.time, e.kind.name, e.session_id, e.turn_index)
                for e in ksim.run(wl, cfg).events]

    want = events()
    orig = ksim.plan_preload, ksim.plan_async_save
    overlap.bind(ModeledExecutor())
    try:
        ksim.plan_preload, ksim.plan_async_save = overlap.plan_preload, overlap.plan_async_save
        got = events()
    finally:
        ksim.plan_preload, ksim.plan_async_save = orig
        overlap.bind(None)
    assert len(got) == len(want) > 0
    for g, w in zip(got, want):
        assert g[1:] == w[1:] and _close(g[0], w[0])
