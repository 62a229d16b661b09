"""The GPU mirror of kvsim.rope (paper_2403_19708_b200.rope) against the oracle
and the reference's own golden vectors: same names, same errors, same
semantics (gapped positions, truncation, empty cache), bf16 tolerances."""

import json
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import rope_ref

pytestmark = pytest.mark.gpu
G = Path(__file__).resolve().parent / "golden"


def _rope():
    from paper_2403_19708_b200 import rope
    return rope


def bf(x):
    return torch.as_tensor(np.asarray(x, dtype=np.float32)).to(torch.bfloat16)


def f64(t):
    return t.float().cpu().numpy().astype(np.float64)


def test_golden_cases_through_gpu_api():
    rope = _rope()
    rg = np.load(G / "rope_golden.npz")
    cases = json.loads((G / "rope_cases.json").read_text())
    checked = 0
    for ci, c in enumerate(cases):
        if c["d"] not in (64, 128):
            continue
        # bf16-round the reference inputs and recompute the f64 oracle on them
        keys, values, q, k, v = (f64(bf(rg[f"c{ci}_{n}"]))
                                 for n in ("keys", "values", "q", "k", "v"))
        seq, ks = c["seq"], c["keep_start"]
        rec = rope.KvRecord(keys, values)
        for pos in (np.arange(seq), rg[f"c{ci}_gpos"]):
            got = f64(rope.attention_with_decoupled_cache(rec, q, k, v, pos))
            want = rope_ref.decoupled_attention(keys, values, q, k, v, pos)
            assert rope_ref.rel_err(got, want) < 1e-2
        tr = rec.truncated(ks, seq)
        got = f64(rope.attention_with_decoupled_cache(tr, q, k, v, np.arange(seq - ks)))
        kk, vv = rope_ref.truncate(keys, values, ks, seq)
        want = rope_ref.decoupled_attention(kk, vv, q, k, v, np.arange(seq - ks))
        assert rope_ref.rel_err(got, want) < 1e-2
        # and against the reference's own f64 output on the unrounded inputs
        assert rope_ref.rel_err(got, rg[f"c{ci}_trunc"]) < 3e-2
        checked += 1
    assert checked >= 3


def test_rotate_matrix_and_rope_rotate():
    rope = _rope()
    rng = np.random.default_rng(1)
    x = f64(bf(rng.standard_normal((50, 128))))
    pos = rng.integers(0, 4000, size=50)
    got = rope.rotate_matrix(x, pos)
    want = rope_ref.rotate(x, pos)
    assert np.abs(f64(got) - want).max() < 2e-2
    v0 = rope.rope_rotate(x[0], 0)
    assert torch.equal(v0.cpu(), bf(x[0]))           # position 0 is the identity
    with pytest.raises(ValueError):
        rope.rope_rotate(x[0], -1)
    n = np.linalg.norm(f64(rope.rope_rotate(x[3], 1234)))
    assert abs(n - np.linalg.norm(x[3])) / n < 1e-2  # isometry up to bf16 rounding


def test_errors_match_reference():
    rope = _rope()
    with pytest.raises(ValueError):
        rope.KvRecord(np.zeros((3, 4)), np.zeros((2, 4)))
    rec = rope.KvRecord(np.zeros((3, 64)), np.zeros((3, 64)))
    with pytest.raises(ValueError):
        rec.truncated(2, 1)
    with pytest.raises(ValueError):
        rope.attention_with_decoupled_cache(rec, np.zeros((1, 64)), np.zeros((1, 64)),
                                            np.zeros((1, 64)), [0, 1])


def test_empty_cache_single_token():
    """empty cache + one query = single-token attention (= v)."""
    rope = _rope()
    rec = rope.KvRecord(np.zeros((0, 128)), np.zeros((0, 128)))
    rng = np.random.default_rng(2)
    q, k, v = (f64(bf(rng.standard_normal((1, 128)))) for _ in range(3))
    got = rope.attention_with_decoupled_cache(rec, q, k, v, [])
    assert torch.equal(got.cpu(), bf(v))


def test_gqa_multihead_matches_oracle():
    rope = _rope()
    rng = np.random.default_rng(3)
    s, n, hq, hkv, d = 700, 45, 8, 2, 128
    K, V = (f64(bf(rng.standard_normal((s, hkv, d)))) for _ in range(2))
    q = f64(bf(rng.standard_normal((n, hq, d))))
    k, v = (f64(bf(rng.standard_normal((n, hkv, d)))) for _ in range(2))
    rec = rope.KvRecord(K, V).truncated(200, s)
    got = f64(rope.attention_with_decoupled_cache(rec, q, k, v, np.arange(s - 200)))
    want = rope_ref.decoupled_attention_mh(K[200:], V[200:], q, k, v, np.arange(s - 200))
    assert rope_ref.rel_err(got, want) < 1e-2
