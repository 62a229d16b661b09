"""float64 forward of the LLaMA-shaped model the GPU runner executes, with
AttentionStore KV reuse (config C1 and small parity cases).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The reference has no model (SURVEY.md §2.3 last row); its numerics contract
is the per-head decoupled attention of rope.py:118-144 and the paper's save
order "cache k, v *before* apply_pos_emb".  This module
wraps oracle.rope_ref.decoupled_attention_mh in a standard pre-norm LLaMA
block so the GPU runner's end-to-end outputs can be checked:

    h  = rmsnorm(x) * w_in
    q,k,v = h @ Wqkv                       (k, v saved pre-RoPE)
    a  = decoupled_attention_mh(cache_k, cache_v, q, k, v, positions)
    x += a @ Wo
    h  = rmsnorm(x) * w_post
    x += (silu(h @ Wg) * (h @ Wu)) @ Wd
    logits = rmsnorm(x) * w_final @ Wlm

Weights are passed in (the GPU runner draws them with torch; the test hands
the exact bf16 values over as float64 arrays).
"""

from __future__ import annotations

import numpy as np

from oracle.rope_ref import THETA_BASE, decoupled_attention_mh

RMS_EPS = 1e-5


def rmsnorm(x, w, eps: float = RMS_EPS):
    x = np.asarray(x, dtype=np.float64)
    return x / np.sqrt(np.mean(x * x, axis=-1, keepdims=True) + eps) * w


def silu(x):
    return x / (1.0 + np.exp(-x))


def forward(weights: dict, tokens, cache, cache_positions, *, n_heads: int,
            n_kv_heads: int, head_dim: int, theta_base: float = THETA_BASE):
    """Prefill ``tokens`` (N,) over a per-layer pre-RoPE cache.

    cache: list over layers of (K (S,Hkv,d), V (S,Hkv,d)); may have S == 0.
    cache_positions: (S,) current positions of the cached rows.
    Returns (logits (N, vocab), new_cache: list over layers of (K_new, V_new)
    pre-RoPE for the N new tokens).
    """
    x = np.asarray(weights["embed"], dtype=np.float64)[np.asarray(tokens)]
    n = x.shape[0]
    hq, hkv, d = n_heads, n_kv_heads, head_dim
    new_cache = []
    for li, lw in enumerate(weights["layers"]):
        h = rmsnorm(x, lw["w_in"])
        qkv = h @ lw["wqkv"]
        q = qkv[:, : hq * d].reshape(n, hq, d)
        k = qkv[:, hq * d: (hq + hkv) * d].reshape(n, hkv, d)
        v = qkv[:, (hq + hkv) * d:].reshape(n, hkv, d)
        new_cache.append((k.copy(), v.copy()))
        ck, cv = cache[li]
        a = decoupled_attention_mh(ck, cv, q, k, v, cache_positions, theta_base)
        x = x + a.reshape(n, hq * d) @ lw["wo"]
        h = rmsnorm(x, lw["w_post"])
        x = x + (silu(h @ lw["wg"]) * (h @ lw["wu"])) @ lw["wd"]
    logits = rmsnorm(x, weights["w_final"]) @ weights["lm_head"]
    return logits, new_cache
