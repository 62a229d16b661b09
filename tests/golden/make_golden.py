"""Generate the golden fixtures by running the REFERENCE itself.

Run in the build container only (the reference does not exist on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes into tests/golden/:
  rope_golden.npz        rotate_matrix / attention_with_decoupled_cache /
                         reference_attention / naive_truncate_coupled outputs
                         on seeded inputs (rope.py)
  equivalence.json       rope.equivalence_report(100, 2024)  (rope.py:246-286)
  truncation.json        _handle_overflow / _truncate_tokens arithmetic
                         (sim.py:468-483, 576-581) over a grid
  store.json             KvStore charge + dump_state after a scripted op
                         sequence (store.py:100-102, 165-342)
  overlap.json           plan_preload / plan_async_save on random inputs
                         (overlap.py:69-200) and preload_buffer_size
  workload_c{1,2,3}.json generate_poisson sessions (trace.py:326-356) plus the
                         reference simulator's per-turn records in reuse mode
                         with unbounded tiers (sim.py:408-466)
  sim_c2.json            full event logs + turn records of capacity-constrained
                         C2 runs (evict_to_disk / evict_out / prefetch order,
                         sim.py:298-366; policy.py)
"""

from __future__ import annotations

import json
import math
import sys
import types
from dataclasses import replace
from pathlib import Path

import numpy as np

from kvsim import model, overlap, rope, sim, store, trace

OUT = Path(__file__).resolve().parent

# LLaMA-2 public shapes; kv bytes/token = 2 * L * Hkv * hd * 2
SHAPES = {
    "tiny": dict(layers=2, d_model=256, n_heads=4, n_kv_heads=4, head_dim=64),
    "7b": dict(layers=32, d_model=4096, n_heads=32, n_kv_heads=32, head_dim=128),
    "13b": dict(layers=40, d_model=5120, n_heads=40, n_kv_heads=40, head_dim=128),
    "70b": dict(layers=80, d_model=8192, n_heads=64, n_kv_heads=8, head_dim=128),
}


def kvb(shape):
    s = SHAPES[shape]
    return 2 * s["layers"] * s["n_kv_heads"] * s["head_dim"] * 2


def rope_golden():
    rng = np.random.default_rng(20240419)
    cases = []
    arrays = {}
    # (seq, d, n_new, keep_start) — includes hd 64/128 hot-path shapes
    specs = [(8, 4, 1, 4), (17, 8, 3, 0), (33, 16, 2, 16), (64, 32, 4, 32),
             (40, 64, 5, 20), (96, 128, 7, 64), (130, 128, 3, 2), (1, 64, 1, 0),
             (257, 128, 9, 128)]
    for ci, (seq, d, n, ks) in enumerate(specs):
        keys = rng.standard_normal((seq, d))
        values = rng.standard_normal((seq, d))
        q = rng.standard_normal((n, d))
        k = rng.standard_normal((n, d))
        v = rng.standard_normal((n, d))
        pos = np.arange(seq)
        rec = rope.KvRecord(keys, values)
        arrays[f"c{ci}_keys"] = keys
        arrays[f"c{ci}_values"] = values
        arrays[f"c{ci}_q"] = q
        arrays[f"c{ci}_k"] = k
        arrays[f"c{ci}_v"] = v
        # arbitrary (non-contiguous) positions exercise next_pos = positions[-1]+1
        gpos = np.sort(rng.choice(4 * seq + 8, size=seq, replace=False))
        arrays[f"c{ci}_gpos"] = gpos
        arrays[f"c{ci}_rot"] = rope.rotate_matrix(keys, gpos)
        arrays[f"c{ci}_full"] = rope.attention_with_decoupled_cache(rec, q, k, v, pos)
        arrays[f"c{ci}_gapped"] = rope.attention_with_decoupled_cache(rec, q, k, v, gpos)
        kept = rec.truncated(ks, seq)
        arrays[f"c{ci}_trunc"] = rope.attention_with_decoupled_cache(
            kept, q, k, v, np.arange(seq - ks))
        if seq * d <= 4096:
            arrays[f"c{ci}_loop"] = rope.reference_attention(
                q, np.concatenate([keys, k]), np.concatenate([values, v]),
                seq + np.arange(n), np.arange(seq + n), seq)
        baked = rope.bake_positions(rec, pos)
        arrays[f"c{ci}_naive"] = rope.naive_truncate_coupled(baked, ks, seq, q, k, v)
        arrays[f"c{ci}_weights"] = rope.attention_weights(
            rope.rotate_matrix(q, seq + np.arange(n)),
            rope.rotate_matrix(np.concatenate([keys, k]), np.arange(seq + n)), seq)
        cases.append(dict(seq=seq, d=d, n=n, keep_start=ks))
    # rope_rotate single-vector cases (rope.py:77-85)
    vecs = rng.standard_normal((6, 16))
    rpos = [0, 1, 7, 100, 4095, 32767]
    arrays["rr_vecs"] = vecs
    arrays["rr_pos"] = np.array(rpos)
    arrays["rr_out"] = np.stack([rope.rope_rotate(vv, p) for vv, p in zip(vecs, rpos)])
    np.savez_compressed(OUT / "rope_golden.npz", **arrays)
    (OUT / "rope_cases.json").write_text(json.dumps(cases, indent=1))


def equivalence():
    rep = rope.equivalence_report(100, 2024)
    (OUT / "equivalence.json").write_text(json.dumps(rep, indent=1, sort_keys=True))


def truncation():
    rows = []
    for w in (64, 100, 2048, 4096):
        for ratio in (0.25, 0.5, 0.75):
            prof = types.SimpleNamespace(context_window=w, truncation_ratio=ratio)
            fake = types.SimpleNamespace(profile=prof, store=None,
                                         state={"s": sim._SessionState()})
            for hist in sorted({0, 1, w // 2, w - 1, w, w + 1, 2 * w, 3 * w + 7,
                                8 * w, 32768}):
                for new in sorted({1, 7, w // 4, w - 1, w, w + 1, 2 * w + 3}):
                    if hist + new > w:
                        kept = sim._Engine._handle_overflow(fake, "s", hist, new)
                    else:
                        kept = hist
                    rows.append(dict(W=w, ratio=ratio, hist=hist, new=new, kept=kept))
            for tok in sorted({0, 1, w - 1, w, w + 1, 2 * w, 5 * w + 3, 40000}):
                rows.append(dict(W=w, ratio=ratio, save_tokens=tok,
                                 saved=sim._Engine._truncate_tokens(fake, tok)))
    (OUT / "truncation.json").write_text(json.dumps(rows))


def store_golden():
    out = []
    for shape, tb in (("13b", 128), ("7b", 256), ("tiny", 16)):
        prof = model.ModelProfile(name=shape, kv_bytes_per_token=float(kvb(shape)),
                                  prefill_seconds_per_token=1e-4,
                                  decode_seconds_per_step=1e-3,
                                  context_window=4096, layers=SHAPES[shape]["layers"])
        tiers = model.TierConfig(dram_capacity=10**15, disk_capacity=10**15)
        bb = tb * kvb(shape)
        st = store.KvStore(prof, tiers, block_bytes=bb)
        charges = {str(t): st.charge(model.kv_size(t, prof))
                   for t in (1, tb - 1, tb, tb + 1, 2142, 4096, 777)}
        ops = [("save", "a", 1000, 0.0), ("save", "b", 4096, 1.0), ("save", "a", 1500, 2.0),
               ("truncate", "b", 2048, 3.0), ("save", "c", tb, 4.0),
               ("truncate", "a", 1500, 5.0), ("save", "d", 3 * tb + 1, 6.0),
               ("remove", "c", 0, 7.0), ("truncate", "d", tb, 8.0)]
        dumps = []
        for op, sid, tok, now in ops:
            if op == "save":
                st.save(sid, tok, now)
            elif op == "truncate":
                st.truncate_item(sid, tok, now)
            else:
                st.remove(sid)
            st.check_invariants()
            dumps.append(json.loads(st.dump_state()))
        out.append(dict(shape=shape, block_tokens=tb, block_bytes=bb,
                        kv_bytes_per_token=kvb(shape), charges=charges,
                        ops=ops, dumps=dumps))
    (OUT / "store.json").write_text(json.dumps(out))


def overlap_golden():
    rng = np.random.default_rng(7)
    rows = []
    for _ in range(120):
        layers = int(rng.integers(1, 81))
        prof = model.ModelProfile(
            name="p", kv_bytes_per_token=float(rng.uniform(1e4, 3e6)),
            prefill_seconds_per_token=float(rng.uniform(1e-6, 5e-4)),
            decode_seconds_per_step=float(rng.uniform(1e-4, 5e-3)),
            context_window=4096, layers=layers)
        tiers = model.TierConfig(pcie_bandwidth=float(rng.uniform(5e9, 6e10)))
        hist = int(rng.integers(0, 4097))
        new = int(rng.integers(0, 1025))
        rb = float(rng.choice([0.0, rng.uniform(0, 5e9)]))
        prev = bool(rng.integers(0, 2))
        bw = None if rng.random() < 0.5 else float(rng.uniform(1e9, 6e10))
        pl = overlap.plan_preload(hist, new, prof, tiers, rb, prev, bandwidth=bw)
        steps = int(rng.integers(0, 64))
        wb = float(rng.choice([0.0, rng.uniform(0, 2e9)]))
        sv = overlap.plan_async_save(new, steps, prof, tiers, wb, bandwidth=bw)
        sbuf = model.preload_buffer_size(hist, new, prof, tiers)
        rows.append(dict(
            kvb=prof.kv_bytes_per_token, pspt=prof.prefill_seconds_per_token,
            dsps=prof.decode_seconds_per_step, layers=layers,
            pcie=tiers.pcie_bandwidth, bw=bw, hist=hist, new=new, read_buffer=rb,
            prev=prev, steps=steps, write_buffer=wb,
            preload=pl.to_dict(), save=sv.to_dict(), sbuf=sbuf))
    (OUT / "overlap.json").write_text(json.dumps(rows))


def workloads():
    specs = {
        "c1": dict(shape="tiny", gen=dict(n_sessions=4, rate=1.0,
                                          turn_dist={"kind": "fixed", "turns": 3},
                                          token_dist={"kind": "fixed", "input": 24,
                                                      "output": 8}, seed=0)),
        "c2": dict(shape="7b", gen=dict(n_sessions=64, rate=1.0, seed=7)),
        "c3": dict(shape="13b", gen=dict(n_sessions=512, rate=1.0, seed=7)),
    }
    for name, sp in specs.items():
        g = sp["gen"]
        wl = trace.generate_poisson(g["n_sessions"], g["rate"],
                                    turn_dist=g.get("turn_dist", "sharegpt"),
                                    token_dist=g.get("token_dist", "sharegpt"),
                                    seed=g["seed"])
        shape = sp["shape"]
        prof = model.ModelProfile(name=shape, kv_bytes_per_token=float(kvb(shape)),
                                  prefill_seconds_per_token=1.92e-4,
                                  decode_seconds_per_step=1e-3, context_window=4096,
                                  layers=SHAPES[shape]["layers"])
        tiers = model.TierConfig(dram_capacity=10**16, disk_capacity=10**16)
        cfg = sim.SimConfig(profile=prof, tiers=tiers, mode=sim.Mode.REUSE, ttl=1e12)
        log = sim.run(wl, cfg)
        sessions = [dict(id=s.session_id,
                         turns=[[t.new_input_tokens, t.output_tokens] for t in s.turns],
                         arrivals=list(s.arrival_times)) for s in wl.sessions]
        records = [dict(session=t.session_id, turn=t.turn_index, hit=t.hit_class,
                        prompt=t.prompt_tokens, new=t.new_tokens,
                        overflowed=t.overflowed, ttft_model=t.ttft_s,
                        prefill_model=t.prefill_s)
                   for t in log.turns]
        (OUT / f"workload_{name}.json").write_text(json.dumps(dict(
            name=name, shape=shape, generator=g, window=4096, truncation_ratio=0.5,
            sessions=sessions, records=records)))


# capacity-constrained C2 runs of the reference simulator: the event log pins
# the scheduler-aware eviction / prefetch order (policy.py, sim.py:298-366)
SIM_CASES = {
    "sa_disk": dict(dram=12e9, disk=40e9, policy="scheduler-aware"),
    "sa_nodisk": dict(dram=16e9, disk=0, policy="scheduler-aware"),
    "lru_disk": dict(dram=12e9, disk=40e9, policy="lru"),
    "sa_disk_window": dict(dram=10e9, disk=30e9, policy="scheduler-aware",
                           prefetch_window=4, eviction_window=6),
}


def sim_golden():
    from kvsim import policy
    wl = trace.generate_poisson(64, 1.0, seed=7)
    out = {}
    for name, c in SIM_CASES.items():
        prof = model.ModelProfile(name="7b", kv_bytes_per_token=float(kvb("7b")),
                                  prefill_seconds_per_token=6e-5, decode_seconds_per_step=6e-3,
                                  context_window=4096, layers=32)
        tiers = model.TierConfig(hbm_read_buffer=int(4e9), hbm_write_buffer=int(2e9),
                                 dram_capacity=int(c["dram"]), disk_capacity=int(c["disk"]),
                                 pcie_bandwidth=55e9, disk_bandwidth=3.2e9)
        pol = policy.PolicyConfig(kind=policy.PolicyKind(c["policy"]),
                                  prefetch_window=c.get("prefetch_window"),
                                  eviction_window=c.get("eviction_window"))
        cfg = sim.SimConfig(profile=prof, tiers=tiers, policy=pol, mode=sim.Mode.REUSE,
                            block_bytes=128 * kvb("7b"))
        log = sim.run(wl, cfg)
        out[name] = dict(
            case=c, block_bytes=128 * kvb("7b"), kv_bytes_per_token=kvb("7b"),
            events=[e.to_dict() for e in log.events],
            turns=[dict(session=t.session_id, turn=t.turn_index, hit=t.hit_class,
                        ttft=t.ttft_s, prefill=t.prefill_s, stall=t.stall_s,
                        prompt=t.prompt_tokens, done=t.done, evicted=t.bytes_evicted)
                   for t in log.turns],
            meta=log.meta)
    (OUT / "sim_c2.json").write_text(json.dumps(out))


if __name__ == "__main__":
    np.seterr(all="ignore")
    if sys.argv[1:] == ["sim"]:
        sim_golden()
        sys.exit(0)
    rope_golden()
    equivalence()
    truncation()
    store_golden()
    overlap_golden()
    workloads()
    sim_golden()
    print("golden fixtures written to", OUT, file=sys.stderr)
