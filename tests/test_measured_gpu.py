"""Measured mode: the reference serving loop (sim.Server) with every
plan_preload / plan_async_save executed by the real engine
(measured.MeasuredExecutor) -- SURVEY.md §8(b) item 2, §8(f) row 3.

Parity: each turn's first-token logits equal the float64 oracle run on the
rows the store held when the turn started (decoupled re-embedding at
0..kept-1, rope.py:118-144; truncation sim.py:468-483), and the loop's
decisions (hit class, prompt size) equal the modeled run's when timing
cannot change them.  The drop-in planners (overlap.plan_preload /
plan_async_save with the reference's signature) return measured Timelines.
"""

import json
from dataclasses import replace
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import llama_ref, rope_ref
from test_engine_gpu import LOGIT_TOL, session_cache
from test_sim_cpu import ModeledExecutor

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _setup(window=64, host_blocks=64, dram_blocks=None, seed=0):
    from paper_2403_19708_b200 import engine, model, sim
    shape = replace(model.shape("tiny"), context_window=window)
    bt = 16
    eng = engine.Engine(shape, host_blocks=host_blocks, block_tokens=bt, seed=seed,
                        max_new=64, read_buffer_bytes=32 << 20, autotune=False,
                        dram_bytes=None if dram_blocks is None
                        else dram_blocks * bt * shape.kv_bytes_per_token)
    wl = sim.load_workload(G / "workload_c1.json")
    tiers = model.TierConfig(hbm_read_buffer=8 << 20, hbm_write_buffer=8 << 20,
                             dram_capacity=eng.store.mem_capacity, disk_capacity=0,
                             pcie_bandwidth=50e9)
    prof = replace(eng.profile, prefill_seconds_per_token=1e-4,
                   decode_seconds_per_step=1e-3)
    cfg = sim.SimConfig(profile=prof, tiers=tiers, block_bytes=eng.store.block_bytes)
    return eng, wl, cfg, shape


def _checking_executor(shape, wnp, errs):
    from paper_2403_19708_b200 import measured
    from paper_2403_19708_b200.store import HitClass

    class Checking(measured.MeasuredExecutor):
        """Captures the stored rows before each job and checks the job's
        logits against the oracle over exactly those rows."""

        def plan_preload(self, hist, new, profile, tiers, rb, prev=True, *, bandwidth=None,
                         job=None):
            sid = job.session_id
            ctx = job.context
            miss = job.hit is HitClass.MISS or hist == 0
            cache = None if miss else session_cache(self.eng, sid, ctx)
            hist_ids = self._history(sid, ctx).clone()
            tl = super().plan_preload(hist, new, profile, tiers, rb, prev, bandwidth=bandwidth,
                                      job=job)
            turn_new = job.new_tokens - (ctx if job.hit is HitClass.MISS else 0)
            new_ids = self._ids(sid, job.turn_index, 0, turn_new).numpy()
            if miss:
                ids = np.concatenate([hist_ids.numpy(), new_ids])
                empty = [(np.zeros((0, shape.n_kv_heads, shape.head_dim)),) * 2] * shape.layers
                want, _ = llama_ref.forward(wnp, ids, empty, np.arange(0),
                                            n_heads=shape.n_heads, n_kv_heads=shape.n_kv_heads,
                                            head_dim=shape.head_dim)
            else:
                want, _ = llama_ref.forward(wnp, new_ids, cache, np.arange(ctx),
                                            n_heads=shape.n_heads, n_kv_heads=shape.n_kv_heads,
                                            head_dim=shape.head_dim)
            got = self.logits[(sid, job.turn_index)].cpu().numpy().astype(np.float64)
            errs.append((sid, job.turn_index, job.hit.value, rope_ref.rel_err(got, want[-1])))
            return tl

    return Checking


def test_measured_c1_matches_oracle_and_modeled_decisions():
    from paper_2403_19708_b200 import measured, sim
    eng, wl, cfg, shape = _setup()
    wnp = eng.runner.w.to_numpy()
    errs = []
    log, ex = measured.serve(wl, eng, cfg, want_logits=True,
                             executor_cls=_checking_executor(shape, wnp, errs))
    assert len(log.turns) == 12 and log.complete
    assert all(e[3] <= LOGIT_TOL for e in errs), errs
    assert {e[2] for e in errs} == {"miss", "memory_hit"}
    modeled = sim.run(wl, cfg, ModeledExecutor())
    for a, b in zip(log.turns, modeled.turns):
        assert (a.session_id, a.turn_index, a.hit_class, a.prompt_tokens, a.overflowed) == \
            (b.session_id, b.turn_index, b.hit_class, b.prompt_tokens, b.overflowed)
    assert any(t.overflowed for t in log.turns)
    for t in log.turns:
        tl = t.timeline
        assert tl is not None and tl.makespan > 0 and t.prefill_s == tl.makespan
        assert t.ttft_s >= t.prefill_s - 1e-12
        if t.hit_class == "memory_hit":
            assert len(tl.load_intervals) == shape.layers
    eng.store.check_invariants()


def test_measured_capacity_constrained_evictions_keep_parity():
    """DRAM for ~3 sessions: the loop's scheduler-aware make_room evicts
    through the real store (rows freed), evicted sessions recompute, and
    every turn still matches the oracle on the rows it found."""
    from paper_2403_19708_b200 import measured
    eng, wl, cfg, shape = _setup(window=4096, host_blocks=64, dram_blocks=18)
    # all sessions arrive together so the store fills before anyone's 2nd turn
    wl.sessions = [replace(s, arrival_times=tuple(t - s.arrival_times[0] for t in
                                                  s.arrival_times)) for s in wl.sessions]
    wnp = eng.runner.w.to_numpy()
    errs = []
    log, _ = measured.serve(wl, eng, cfg, want_logits=True,
                            executor_cls=_checking_executor(shape, wnp, errs))
    assert log.complete and all(e[3] <= LOGIT_TOL for e in errs), errs
    assert log.meta["evict_out_count"] > 0
    eng.store.check_invariants()
    for sid, it in eng.store.items.items():
        assert len(eng.store.tables[sid]) * 16 >= it.tokens


def test_recompute_comparator_matches_full_forward():
    from paper_2403_19708_b200 import measured
    eng, wl, cfg, shape = _setup(window=4096)
    wnp = eng.runner.w.to_numpy()
    log, ex = measured.serve(wl, eng, cfg, recompute=True, want_logits=True)
    assert all(t.hit_class == "miss" for t in log.turns)
    # the last turn of s0 recomputes its whole conversation
    t = [t for t in log.turns if t.session_id == "s0"][-1]
    ids = eng.tokens["s0"][:t.prompt_tokens].numpy()
    empty = [(np.zeros((0, shape.n_kv_heads, shape.head_dim)),) * 2] * shape.layers
    want, _ = llama_ref.forward(wnp, ids, empty, np.arange(0), n_heads=shape.n_heads,
                                n_kv_heads=shape.n_kv_heads, head_dim=shape.head_dim)
    got = ex.logits[("s0", t.turn_index)].cpu().numpy().astype(np.float64)
    assert rope_ref.rel_err(got, want[-1]) <= LOGIT_TOL


def test_dropin_planners_reference_signature():
    """overlap.plan_preload / plan_async_save called exactly as sim.py:434-441
    calls them (no job): a synthetic session of that shape, measured."""
    from paper_2403_19708_b200 import measured, overlap
    eng, wl, cfg, shape = _setup(window=4096)
    with pytest.raises(RuntimeError):
        overlap.bind(None)
        overlap.plan_preload(10, 5, cfg.profile, cfg.tiers, 0.0)
    overlap.bind(measured.MeasuredExecutor(eng))
    try:
        with pytest.raises(ValueError):
            overlap.plan_preload(-1, 5, cfg.profile, cfg.tiers, 0.0)
        cold = overlap.plan_preload(200, 30, cfg.profile, cfg.tiers, 0.0, False)
        assert len(cold.load_intervals) == shape.layers and cold.makespan > 0
        assert min(a for a, _ in cold.load_intervals) >= -1e-6   # no head start
        kvb = 200 * shape.kv_bytes_per_token
        warm = overlap.plan_preload(200, 30, cfg.profile, cfg.tiers, float(kvb), True)
        assert warm.stall_total <= 1e-4
        assert max(b for _, b in warm.load_intervals) <= 1e-6    # all loaded before t=0
        only = overlap.plan_preload(100, 0, cfg.profile, cfg.tiers, 0.0, False)
        assert len(only.load_intervals) == shape.layers and only.makespan > 0
        recomp = overlap.plan_preload(0, 64, cfg.profile, cfg.tiers, 0.0, False)
        assert recomp.load_intervals == [] and recomp.stall_total == 0.0
        assert overlap.plan_async_save(30, 4, cfg.profile, cfg.tiers, 1e9).stall_total == 0.0
        assert "__plan_preload__" not in eng.store.tables
    finally:
        overlap.bind(None)
