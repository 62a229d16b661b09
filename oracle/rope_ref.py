"""float64 restatement of the reference's decoupled-positional-encoding numerics.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference: /root/reference/pkg/src/kvsim/rope.py.  Semantics kept exactly:

* RoPE pairs are *interleaved*: (x[2i], x[2i+1]) rotated by
  angle = pos * theta ** (-2i/d)                     (rope.py:55-60, 63-74)
* attention = softmax(q k^T / sqrt(d)) v with query row r seeing key columns
  c <= n_cached + r                                  (rope.py:94-105)
* decoupled attention re-embeds the cached (pre-RoPE) keys at ``positions``
  and the new tokens at positions[-1]+1 .. +N         (rope.py:118-144)
* truncation keeps rows [start, end) (rope.py:48-52)

Extensions for the multi-head hot path (no reference counterpart; composed
from the per-head primitives, which the reference broadcasts identically over
leading dims):

* ``decoupled_attention_mh``  — (S,Hkv,d) cache, (N,Hq,d) queries, GQA
  group = Hq // Hkv, one call of the per-head function per q-head.
* empty cache (seq_len == 0) is special-cased: the reference crashes in
  ``rotate_matrix`` on a size-0 reshape (rope.py:69) although
  SPEC.md:451 calls it valid; here it is plain causal prefill.
"""

from __future__ import annotations

import numpy as np

THETA_BASE = 10000.0  # rope.py:22


def inv_freq(head_dim: int, theta_base: float = THETA_BASE) -> np.ndarray:
    """theta ** (-2i/d) for i in [0, d/2)  (rope.py:59)."""
    if head_dim % 2:
        raise ValueError("head_dim must be even")
    i = np.arange(head_dim // 2, dtype=np.float64)
    return theta_base ** (-(2.0 * i) / head_dim)


def angles(head_dim: int, positions, theta_base: float = THETA_BASE) -> np.ndarray:
    """(len(positions), d/2) rotation angles  (rope.py:55-60)."""
    pos = np.asarray(positions, dtype=np.float64).reshape(-1)
    return np.outer(pos, inv_freq(head_dim, theta_base))


def rotate(x, positions, theta_base: float = THETA_BASE) -> np.ndarray:
    """Rotate rows of x (..., S, d) at per-row positions (S,)  (rope.py:63-74).

    Broadcasts over leading dims like the reference.  Size-0 inputs return an
    empty array (the reference raises on them, rope.py:69).
    """
    x = np.asarray(x, dtype=np.float64)
    d = x.shape[-1]
    if x.size == 0:
        return x.copy()
    a = angles(d, positions, theta_base)
    c, s = np.cos(a), np.sin(a)
    ev = x[..., 0::2]
    od = x[..., 1::2]
    out = np.empty_like(x)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    return out


def causal_attention(q_rot, k_rot, v, n_cached: int) -> np.ndarray:
    """softmax(q k^T/sqrt(d)) v, row r sees cols <= n_cached + r  (rope.py:94-105)."""
    q_rot = np.asarray(q_rot, dtype=np.float64)
    k_rot = np.asarray(k_rot, dtype=np.float64)
    v = np.asarray(v, dtype=np.float64)
    d = q_rot.shape[-1]
    s = (q_rot @ k_rot.T) / np.sqrt(d)
    rows = np.arange(q_rot.shape[0])[:, None]
    cols = np.arange(k_rot.shape[0])[None, :]
    s = np.where(cols > n_cached + rows, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    w = np.exp(s)
    w /= w.sum(axis=-1, keepdims=True)
    return w @ v


def attention_weights(q_rot, k_rot, n_cached: int) -> np.ndarray:
    """Normalised causal weights (rope.py:108-115)."""
    q_rot = np.asarray(q_rot, dtype=np.float64)
    k_rot = np.asarray(k_rot, dtype=np.float64)
    d = q_rot.shape[-1]
    s = (q_rot @ k_rot.T) / np.sqrt(d)
    rows = np.arange(q_rot.shape[0])[:, None]
    cols = np.arange(k_rot.shape[0])[None, :]
    s = np.where(cols > n_cached + rows, -np.inf, s)
    s = s - s.max(axis=-1, keepdims=True)
    w = np.exp(s)
    return w / w.sum(axis=-1, keepdims=True)


def truncate(keys, values, start: int, end: int):
    """Keep rows [start, end) of a pre-RoPE record (rope.py:48-52)."""
    keys = np.asarray(keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if not 0 <= start <= end <= keys.shape[0]:
        raise ValueError("bad keep range")
    return keys[start:end].copy(), values[start:end].copy()


def decoupled_attention(keys, values, new_q, new_k, new_v, positions,
                        theta_base: float = THETA_BASE) -> np.ndarray:
    """One-head reuse step  (rope.py:118-144).

    ``keys``/``values`` (S, d) are the cached pre-RoPE rows, ``positions`` (S,)
    their current indices; the N new tokens take positions[-1]+1 .. (or 0..
    when the cache is empty).
    """
    keys = np.asarray(keys, dtype=np.float64).reshape(-1, np.shape(new_q)[-1])
    values = np.asarray(values, dtype=np.float64).reshape(keys.shape)
    new_q = np.asarray(new_q, dtype=np.float64)
    new_k = np.asarray(new_k, dtype=np.float64)
    new_v = np.asarray(new_v, dtype=np.float64)
    positions = np.asarray(positions, dtype=np.int64).reshape(-1)
    if positions.shape[0] != keys.shape[0]:
        raise ValueError(
            f"positions length {positions.shape[0]} != cached length {keys.shape[0]}")
    n_cached = keys.shape[0]
    start = int(positions[-1]) + 1 if n_cached else 0
    new_pos = start + np.arange(new_q.shape[0])
    k_all = np.concatenate([rotate(keys, positions, theta_base),
                            rotate(new_k, new_pos, theta_base)], axis=0)
    v_all = np.concatenate([values, new_v], axis=0)
    return causal_attention(rotate(new_q, new_pos, theta_base), k_all, v_all, n_cached)


def decoupled_attention_mh(keys, values, new_q, new_k, new_v, positions,
                           theta_base: float = THETA_BASE) -> np.ndarray:
    """Multi-head / GQA composition of ``decoupled_attention``.

    keys, values: (S, Hkv, d) pre-RoPE cache; new_q: (N, Hq, d);
    new_k/new_v: (N, Hkv, d).  q-head h uses kv-head h // (Hq // Hkv).
    Returns (N, Hq, d).
    """
    new_q = np.asarray(new_q, dtype=np.float64)
    n, hq, d = new_q.shape
    new_k = np.asarray(new_k, dtype=np.float64).reshape(n, -1, d)
    new_v = np.asarray(new_v, dtype=np.float64).reshape(n, -1, d)
    hkv = new_k.shape[1]
    keys = np.asarray(keys, dtype=np.float64).reshape(-1, hkv, d)
    values = np.asarray(values, dtype=np.float64).reshape(-1, hkv, d)
    if hq % hkv:
        raise ValueError("Hq must be a multiple of Hkv")
    g = hq // hkv
    out = np.empty((n, hq, d), dtype=np.float64)
    for h in range(hq):
        kh = h // g
        out[:, h, :] = decoupled_attention(keys[:, kh], values[:, kh], new_q[:, h],
                                           new_k[:, kh], new_v[:, kh], positions,
                                           theta_base)
    return out


# --- NKVT negative control (rope.py:147-173) --------------------------------

def bake(keys, positions, theta_base: float = THETA_BASE) -> np.ndarray:
    """Keys with rotations burned in (the coupled cache)  (rope.py:147-151)."""
    return rotate(keys, positions, theta_base)


def naive_truncate_coupled(baked_keys, values, keep_start: int, keep_end: int,
                           new_q, new_k, new_v, theta_base: float = THETA_BASE):
    """Attend over a truncated coupled cache with stale rotations (rope.py:154-173)."""
    baked_keys = np.asarray(baked_keys, dtype=np.float64)
    values = np.asarray(values, dtype=np.float64)
    if not 0 <= keep_start <= keep_end <= baked_keys.shape[0]:
        raise ValueError("bad keep range")
    kept = keep_end - keep_start
    new_pos = kept + np.arange(np.shape(new_q)[0])
    k_all = np.concatenate([baked_keys[keep_start:keep_end],
                            rotate(new_k, new_pos, theta_base)], axis=0)
    v_all = np.concatenate([values[keep_start:keep_end],
                            np.asarray(new_v, dtype=np.float64)], axis=0)
    return causal_attention(rotate(new_q, new_pos, theta_base), k_all, v_all, kept)


# --- loop oracle (rope.py:181-223) ------------------------------------------

def _rotate_one(vec, pos, theta_base):
    d = len(vec)
    out = [0.0] * d
    for i in range(d // 2):
        a = pos * theta_base ** (-2.0 * i / d)
        c, s = np.cos(a), np.sin(a)
        x0, x1 = vec[2 * i], vec[2 * i + 1]
        out[2 * i] = c * x0 - s * x1
        out[2 * i + 1] = s * x0 + c * x1
    return out


def loop_attention(raw_q, raw_k, raw_v, q_positions, k_positions, n_cached: int,
                   theta_base: float = THETA_BASE) -> np.ndarray:
    """Unvectorised from-scratch attention, structurally independent of BLAS
    (rope.py:192-223).  Small shapes only."""
    raw_q = np.asarray(raw_q, dtype=np.float64)
    raw_k = np.asarray(raw_k, dtype=np.float64)
    raw_v = np.asarray(raw_v, dtype=np.float64)
    d = raw_q.shape[1]
    kr = [_rotate_one(r, p, theta_base) for r, p in zip(raw_k, k_positions)]
    out = []
    for i, (qr, qp) in enumerate(zip(raw_q, q_positions)):
        q = _rotate_one(qr, qp, theta_base)
        vis = n_cached + i + 1
        sc = [sum(a * b for a, b in zip(q, kr[j])) / d ** 0.5 for j in range(vis)]
        m = max(sc)
        e = [np.exp(x - m) for x in sc]
        z = sum(e)
        row = [0.0] * d
        for j in range(vis):
            w = e[j] / z
            for c in range(d):
                row[c] += w * raw_v[j][c]
        out.append(row)
    return np.asarray(out)


def rel_err(got, want) -> float:
    """||got - want|| / ||want||  (rope.py:231-233)."""
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    den = np.linalg.norm(want)
    return float(np.linalg.norm(got - want) / (den if den else 1.0))


def random_instance(rng: np.random.Generator, *, min_seq: int = 8, max_seq: int = 64,
                    max_dim: int = 32):
    """Same draw order as rope.py:236-243 so seeded suites line up."""
    seq = int(rng.integers(min_seq, max_seq + 1))
    d = 2 * int(rng.integers(2, max_dim // 2 + 1))
    n_new = int(rng.integers(1, 5))
    mk = lambda n: rng.standard_normal((n, d))  # noqa: E731
    keys, values = mk(seq), mk(seq)
    return keys, values, mk(n_new), mk(n_new), mk(n_new)


def equivalence_report(n_instances: int = 100, seed: int = 2024) -> dict:
    """full / truncated / NKVT suite  (rope.py:246-286)."""
    rng = np.random.default_rng(seed)
    full, trunc, naive = [], [], []
    for _ in range(n_instances):
        keys, values, q, k, v = random_instance(rng)
        seq = keys.shape[0]
        n = q.shape[0]
        pos = np.arange(seq)
        want = loop_attention(q, np.concatenate([keys, k]), np.concatenate([values, v]),
                              seq + np.arange(n), np.arange(seq + n), seq)
        full.append(rel_err(decoupled_attention(keys, values, q, k, v, pos), want))
        cut = seq // 2
        kk, vv = truncate(keys, values, cut, seq)
        kept = seq - cut
        got_t = decoupled_attention(kk, vv, q, k, v, np.arange(kept))
        want_t = loop_attention(q, np.concatenate([kk, k]), np.concatenate([vv, v]),
                                kept + np.arange(n), np.arange(kept + n), kept)
        trunc.append(rel_err(got_t, want_t))
        got_n = naive_truncate_coupled(bake(keys, pos), values, cut, seq, q, k, v)
        naive.append(float(np.max(np.abs(got_n - want_t))))
    return {
        "instances": n_instances,
        "seed": seed,
        "full_max_rel_err": max(full),
        "truncated_max_rel_err": max(trunc),
        "naive_min_deviation": min(naive),
        "naive_median_deviation": float(np.median(naive)),
        "naive_diverging": sum(1 for x in naive if x > 0.01),
    }
