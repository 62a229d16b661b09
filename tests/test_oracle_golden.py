"""Pin the CPU oracle against golden vectors produced by the reference itself
(tests/golden/make_golden.py ran kvsim from /root/reference)."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import layout_ref, overlap_ref, rope_ref, workload_ref

G = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def rg():
    return np.load(G / "rope_golden.npz")


@pytest.fixture(scope="module")
def cases():
    return json.loads((G / "rope_cases.json").read_text())


def test_rotate_matches_reference(rg, cases):
    for ci, _ in enumerate(cases):
        got = rope_ref.rotate(rg[f"c{ci}_keys"], rg[f"c{ci}_gpos"])
        np.testing.assert_allclose(got, rg[f"c{ci}_rot"], rtol=0, atol=1e-12)


def test_rope_rotate_single(rg):
    for vec, p, want in zip(rg["rr_vecs"], rg["rr_pos"], rg["rr_out"]):
        np.testing.assert_allclose(rope_ref.rotate(vec[None], [p])[0], want, atol=1e-12)


def test_decoupled_attention_matches_reference(rg, cases):
    for ci, c in enumerate(cases):
        seq, ks = c["seq"], c["keep_start"]
        args = [rg[f"c{ci}_{n}"] for n in ("keys", "values", "q", "k", "v")]
        full = rope_ref.decoupled_attention(*args, np.arange(seq))
        np.testing.assert_allclose(full, rg[f"c{ci}_full"], rtol=1e-12, atol=1e-12)
        gap = rope_ref.decoupled_attention(*args, rg[f"c{ci}_gpos"])
        np.testing.assert_allclose(gap, rg[f"c{ci}_gapped"], rtol=1e-12, atol=1e-12)
        kk, vv = rope_ref.truncate(args[0], args[1], ks, seq)
        tr = rope_ref.decoupled_attention(kk, vv, *args[2:], np.arange(seq - ks))
        np.testing.assert_allclose(tr, rg[f"c{ci}_trunc"], rtol=1e-12, atol=1e-12)
        if f"c{ci}_loop" in rg:
            assert rope_ref.rel_err(full, rg[f"c{ci}_loop"]) < 1e-12
        nv = rope_ref.naive_truncate_coupled(rope_ref.bake(args[0], np.arange(seq)),
                                             args[1], ks, seq, *args[2:])
        np.testing.assert_allclose(nv, rg[f"c{ci}_naive"], rtol=1e-12, atol=1e-12)


def test_attention_weights(rg, cases):
    for ci, c in enumerate(cases):
        seq, n = c["seq"], c["n"]
        q = rope_ref.rotate(rg[f"c{ci}_q"], seq + np.arange(n))
        k = rope_ref.rotate(np.concatenate([rg[f"c{ci}_keys"], rg[f"c{ci}_k"]]),
                            np.arange(seq + n))
        w = rope_ref.attention_weights(q, k, seq)
        np.testing.assert_allclose(w, rg[f"c{ci}_weights"], atol=1e-12)
        np.testing.assert_allclose(w.sum(-1), 1.0, atol=1e-9)


def test_equivalence_report_matches_reference():
    want = json.loads((G / "equivalence.json").read_text())
    got = rope_ref.equivalence_report(100, 2024)
    assert got["naive_diverging"] == want["naive_diverging"] == 100
    assert got["full_max_rel_err"] < 1e-12 and got["truncated_max_rel_err"] < 1e-12
    assert abs(got["naive_min_deviation"] - want["naive_min_deviation"]) < 1e-9
    assert abs(got["naive_median_deviation"] - want["naive_median_deviation"]) < 1e-9


def test_empty_cache_is_plain_prefill():
    rng = np.random.default_rng(0)
    q, k, v = (rng.standard_normal((5, 8)) for _ in range(3))
    got = rope_ref.decoupled_attention(np.zeros((0, 8)), np.zeros((0, 8)), q, k, v, [])
    want = rope_ref.loop_attention(q, k, v, np.arange(5), np.arange(5), 0)
    assert rope_ref.rel_err(got, want) < 1e-12


def test_positions_length_error():
    with pytest.raises(ValueError):
        rope_ref.decoupled_attention(np.zeros((3, 4)), np.zeros((3, 4)), np.zeros((1, 4)),
                                     np.zeros((1, 4)), np.zeros((1, 4)), [0, 1])


def test_multihead_gqa_is_per_head_composition():
    rng = np.random.default_rng(3)
    s, n, hq, hkv, d = 11, 4, 8, 2, 16
    K, V = rng.standard_normal((s, hkv, d)), rng.standard_normal((s, hkv, d))
    q, k, v = (rng.standard_normal((n, h, d)) for h in (hq, hkv, hkv))
    out = rope_ref.decoupled_attention_mh(K, V, q, k, v, np.arange(s))
    for h in range(hq):
        want = rope_ref.loop_attention(q[:, h], np.concatenate([K[:, h // 4], k[:, h // 4]]),
                                       np.concatenate([V[:, h // 4], v[:, h // 4]]),
                                       s + np.arange(n), np.arange(s + n), s)
        assert rope_ref.rel_err(out[:, h], want) < 1e-12


def test_truncation_matches_reference():
    rows = json.loads((G / "truncation.json").read_text())
    n = 0
    for r in rows:
        if "kept" in r:
            got = layout_ref.overflow_kept(r["hist"], r["new"], r["W"], r["ratio"])
            assert got == r["kept"], r
        else:
            assert layout_ref.save_truncate(r["save_tokens"], r["W"], r["ratio"]) == r["saved"], r
        n += 1
    assert n > 500


def test_store_charge_matches_reference():
    for case in json.loads((G / "store.json").read_text()):
        for tok, ch in case["charges"].items():
            nbytes = layout_ref.kv_size(int(tok), case["kv_bytes_per_token"])
            assert layout_ref.charge(nbytes, case["block_bytes"]) == ch
            assert ch // case["block_bytes"] == layout_ref.blocks_for(
                int(tok), case["block_tokens"])


def test_overlap_planners_match_reference():
    for r in json.loads((G / "overlap.json").read_text()):
        bw = r["bw"] if r["bw"] is not None else r["pcie"]
        pl = overlap_ref.plan_preload(
            r["hist"], r["new"], kv_bytes_per_token=r["kvb"], prefill_s_per_token=r["pspt"],
            layers=r["layers"], bandwidth=bw, read_buffer=r["read_buffer"],
            prev_job_running=r["prev"])
        for key in ("stall_total", "max_gap", "makespan"):
            assert pl[key] == pytest.approx(r["preload"][key], rel=1e-12, abs=1e-15)
        np.testing.assert_allclose(np.array(pl["load_intervals"]).reshape(-1),
                                   np.array(r["preload"]["load_intervals"]).reshape(-1),
                                   rtol=1e-12, atol=1e-15)
        np.testing.assert_allclose(np.array(pl["compute_intervals"]).reshape(-1),
                                   np.array(r["preload"]["compute_intervals"]).reshape(-1),
                                   rtol=1e-12, atol=1e-15)
        sv = overlap_ref.plan_async_save(
            r["new"], r["steps"], kv_bytes_per_token=r["kvb"], prefill_s_per_token=r["pspt"],
            decode_s_per_step=r["dsps"], bandwidth=bw, write_buffer=r["write_buffer"])
        for key in ("stall_total", "makespan"):
            assert sv[key] == pytest.approx(r["save"][key], rel=1e-12, abs=1e-15)
        np.testing.assert_allclose(np.array(sv["save_intervals"]).reshape(-1),
                                   np.array(r["save"]["save_intervals"]).reshape(-1),
                                   rtol=1e-12, atol=1e-15)
        sb = overlap_ref.preload_buffer_size(r["hist"], r["new"], kv_bytes_per_token=r["kvb"],
                                             prefill_s_per_token=r["pspt"],
                                             bandwidth=r["pcie"])
        assert sb == pytest.approx(r["sbuf"], rel=1e-12, abs=1e-6)


@pytest.mark.parametrize("name", ["c1", "c2", "c3"])
def test_workload_replay_matches_reference_sim(name):
    wl = workload_ref.load(name)
    recs = {(r["session"], r["turn"]): r for r in wl["records"]}
    shapes = workload_ref.shapes(name)
    assert len(shapes) == len(recs)
    for s in shapes:
        r = recs[(s.session_id, s.turn)]
        assert s.new == r["new"]
        assert s.prompt == r["prompt"], (s, r)
        assert s.hit == (r["hit"] != "miss"), (s, r)
        assert s.overflowed == r["overflowed"]


def test_long_context_c4_shapes():
    sh = workload_ref.long_context_shapes()
    # turn 0 keeps 2048 of 32768; turns 1-5 reuse 2368..3648
    assert [s.kept for s in sh] == [2048, 2368, 2688, 3008, 3328, 3648]
    assert sh[0].drop == 30720 and all(s.hit for s in sh)
