"""Analytical pre-load / async-save timelines (the modeled counterpart of the
measured timelines the GPU engine produces).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Reference: /root/reference/pkg/src/kvsim/overlap.py:69-123 (plan_preload) and
:126-200 (plan_async_save); model.py:259-263 (prefill_time), :273-287
(preload_buffer_size).  Returned as plain dicts with the Timeline fields
(overlap.py:31-66).
"""

from __future__ import annotations

import math


def plan_preload(hist: int, new: int, *, kv_bytes_per_token: float,
                 prefill_s_per_token: float, layers: int, bandwidth: float,
                 read_buffer: float, prev_job_running: bool = True) -> dict:
    """overlap.py:69-123.  Layer k's KV must be resident by the *end* of its
    compute slot (the loader may lag one layer, overlap.py:9-13)."""
    if hist < 0 or new < 0:
        raise ValueError("token counts must be >= 0")
    if read_buffer < 0:
        raise ValueError("read_buffer must be >= 0")
    kv = hist * kv_bytes_per_token
    load_total = kv / bandwidth
    comp_total = new * prefill_s_per_token
    tl_load, tl_comp = load_total / layers, comp_total / layers
    head = min(read_buffer, kv) / bandwidth if (prev_job_running and hist > 0) else 0.0
    loads = ([(k * tl_load - head, (k + 1) * tl_load - head) for k in range(layers)]
             if hist > 0 else [])
    comps, gaps = [], []
    cur = 0.0
    if new > 0:
        for k in range(1, layers + 1):
            ready = max(0.0, k * tl_load - head) if hist else 0.0
            st = max(cur, ready - tl_comp)
            if st > cur:
                gaps.append(st - cur)
            cur = st + tl_comp
            comps.append((st, cur))
        makespan = cur
    else:
        makespan = max(0.0, load_total - head)
        if makespan > 0:
            gaps.append(makespan)
    stall = makespan - comp_total
    if abs(stall) < 1e-12:
        stall = 0.0
    return {"load_intervals": loads, "compute_intervals": comps, "save_intervals": [],
            "stall_total": stall, "max_gap": max(gaps, default=0.0),
            "makespan": makespan}


def plan_async_save(prompt: int, steps: int, *, kv_bytes_per_token: float,
                    prefill_s_per_token: float, decode_s_per_step: float,
                    bandwidth: float, write_buffer: float) -> dict:
    """overlap.py:126-200."""
    if prompt < 0 or steps < 0:
        raise ValueError("token counts must be >= 0")
    if write_buffer < 0:
        raise ValueError("write_buffer must be >= 0")
    b = bandwidth
    pre = prompt * prefill_s_per_token
    dec = steps * decode_s_per_step
    end = pre + dec
    pbytes = prompt * kv_bytes_per_token
    sbytes = kv_bytes_per_token
    total = pbytes + steps * sbytes
    comps = ([(0.0, pre)] if pre > 0 else []) + ([(pre, end)] if dec > 0 else [])
    tl = {"load_intervals": [], "compute_intervals": comps, "save_intervals": [],
          "stall_total": 0.0, "max_gap": 0.0, "makespan": end}
    if total == 0:
        return tl
    w = sbytes / b
    flush_end = pre + pbytes / b
    saves = tl["save_intervals"]
    if flush_end >= end:
        unwritten = total - b * dec
        if pbytes > 0:
            saves.append((pre, flush_end))
    else:
        late = 0
        if steps > 0:
            ok1 = math.floor((end - flush_end) / w + 1e-9)
            late1 = steps - min(steps, max(0, ok1))
            if w <= decode_s_per_step:
                ok2 = math.floor(steps - w / decode_s_per_step + 1e-9)
            else:
                ok2 = math.floor((end - pre - decode_s_per_step) / w + 1e-9)
            late2 = steps - min(steps, max(0, ok2))
            late = max(late1, late2)
        unwritten = late * sbytes
        if pbytes > 0:
            saves.append((pre, flush_end))
        if steps > 0:
            first = max(flush_end, pre + decode_s_per_step)
            saves.append((first, max(end, first) + late * w))
    spill = min(unwritten, write_buffer)
    over = (unwritten - spill) / b
    tl["makespan"] = end + over
    tl["stall_total"] = over
    tl["max_gap"] = over
    if over > 0 and flush_end >= end:
        saves.append((end, tl["makespan"]))
    return tl


def preload_buffer_size(hist: int, new: int, *, kv_bytes_per_token: float,
                        prefill_s_per_token: float, bandwidth: float) -> float:
    """S_buf = max(0, B (T_load L_hist - T_pref L_new))  (model.py:273-287)."""
    if hist < 0 or new < 0:
        raise ValueError("token counts must be >= 0")
    gap = (kv_bytes_per_token / bandwidth) * hist - prefill_s_per_token * new
    return max(0.0, bandwidth * gap)
