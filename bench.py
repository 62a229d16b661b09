#!/usr/bin/env python
"""Benchmark of the B200 AttentionStore KV-reuse prefill path.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config c3] [--turns B]

Workload (BASELINE.json configs[2], the north-star target "LLaMA-2-13B-shaped
multi-turn synthetic sessions"): the reference generator's 512 ShareGPT-shaped
sessions (trace.generate_poisson(512, 1.0, seed=7), committed as
tests/golden/workload_c3.json) replayed through the reference truncation rules
(W = 4096, ratio 0.5).  Sessions are sharded across ranks by a stable hash of
the session id (no collective on the path); each rank takes B hit turns of its
shard (seeded sample), random-init LLaMA-2-13B weights and random bf16
pre-RoPE KV history of the right size per turn.  One step = prefill of those B
turns back to back.

Modes (same turns, same kernels):
  e2e   "host": each turn's kept KV streamed from the pinned host arena by the
        layer-wise pre-loader (K1), re-embedded (K2), attended (K3, tcgen05),
        new-token KV saved back to host (K4); token ids H2D and the first token
        D2H every step.                       -> the JSON "e2e" (headline)
  value "hbm": the same with the session KV resident in an HBM arena (inputs
        already in HBM: SURVEY.md §8f item 1).  -> the JSON "value"
  recompute: full prompt prefill, no reuse, no save (sim.py:432-435 baseline).
Metric = prefill tokens/s = sum(kept + new) / seconds (metrics.py:118-119, 142).
"""

from __future__ import annotations

import argparse
import json
import platform
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
METRIC = "multi-turn prefill tokens/s and p50 TTFT vs recompute; H2D GB/s per GPU"
CONFIGS = {
    "c2": ("llama2-7b", "workload_c2.json"),
    "c3": ("llama2-13b", "workload_c3.json"),
    "c4": ("llama2-7b", None),   # long-context overflow: 32K history at W = 4096
    "c5": ("llama2-70b", "workload_c3.json"),  # tensor-parallel over the launch's ranks
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--turns", type=int, default=16, help="hit turns per GPU per step")
    ap.add_argument("--block-tokens", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--batch-prefill", type=int, default=1,
                    help="value mode: run each step's turns as one batched layer pass "
                         "(askv_prefill_layers_batch); 0 = one turn after another")
    ap.add_argument("--fragmented", action="store_true",
                    help="scatter every turn's blocks over the arena (random permutation) "
                         "instead of the allocator's contiguous runs")
    ap.add_argument("--serve-dram-gb", type=float, default=96.0,
                    help="host DRAM of the measured serving replay (0 = skip it)")
    ap.add_argument("--serve-hbm-gb", type=float, default=64.0,
                    help="HBM session tier of the serving replay's third mode (0 = off)")
    ap.add_argument("--disk-dir", default="/tmp",
                    help="directory for the disk-tier probe ('none' = skip)")
    ap.add_argument("--decode-steps", type=int, default=32,
                    help="greedy decode steps measured after the prefill legs (0 = skip)")
    ap.add_argument("--tp-rank-of", type=int, default=0,
                    help="c5 on one GPU: run one rank of a TP-K shard (weights, heads and KV "
                         "slice of rank 0), collective excluded -- a per-rank compute probe")
    ap.add_argument("--k2-overlap", type=int, default=0,
                    help="1: K2 of layer l+1 on a side stream alongside K3 of layer l")
    ap.add_argument("--profile-attn", action="store_true",
                    help="run only a few hbm steps (for ncu captures)")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# workload
# ---------------------------------------------------------------------------

def long_context_turns(rank: int, n: int, history: int = 32768, new: int = 256,
                       output: int = 64, window: int = 4096):
    """Config C4: sessions with a stored 32K-token history, then
    turns of 256 in / 64 out at W = 4096.  Turn k reuses kept_k rows after the
    reference truncation rules (sim.py:468-483, 576-581): 2048, 2368, ... 3648."""
    from paper_2403_19708_b200.engine import overflow_kept, save_truncate

    cut = window // 2
    shapes = []
    ctx = history
    for k in range(6):
        kept = overflow_kept(ctx, new, window, cut)
        shapes.append((k, kept))
        ctx = save_truncate(kept + new + output, window, cut)
    out = []
    i = 0
    while len(out) < n:
        k, kept = shapes[i % len(shapes)]
        out.append((f"long{rank}_{i // len(shapes)}", k, kept, new))
        i += 1
    return out, len(out)


def select_turns(cfg: str, rank: int, world: int, n: int):
    """Hit turns of this rank's session shard (stable crc32 hash), seeded sample."""
    from paper_2403_19708_b200.engine import overflow_kept, save_truncate

    if cfg == "c4":
        return long_context_turns(rank, n)

    wl = json.loads((ROOT / "tests" / "golden" / CONFIGS[cfg][1]).read_text())
    w, ratio = wl["window"], wl["truncation_ratio"]
    cut = max(1, int(ratio * w))
    from paper_2403_19708_b200.dist import shard_of

    hits = []
    for s in wl["sessions"]:
        if shard_of(s["id"], world) != rank:
            continue
        ctx = 0
        for k, (new, out) in enumerate(s["turns"]):
            kept = overflow_kept(ctx, new, w, cut)
            if k > 0 and kept > 0:
                hits.append((s["id"], k, kept, new))
            ctx = save_truncate(kept + new + out, w, cut)
    rng = np.random.default_rng(1234 + rank)
    pick = sorted(rng.choice(len(hits), size=min(n, len(hits)), replace=False))
    return [hits[i] for i in pick], len(hits)


# ---------------------------------------------------------------------------
# clocks (nvidia-smi sampled during the timed region)
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap,"
              "timestamp")
    # nvidia-smi is started before the warm-up (its NVML start-up stalls CUDA
    # host calls for a moment) and only the samples whose timestamp falls in
    # the timed window [window[0], window[1]] (host clock) are summarised.

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, window=None) -> dict:
        import datetime
        rows = []
        try:
            for line in open(self.path):
                parts = [p.strip() for p in line.split(",")]
                if len(parts) >= 10 and parts[1].replace(".", "").isdigit():
                    if window is not None:
                        try:
                            ts = datetime.datetime.strptime(
                                parts[9], "%Y/%m/%d %H:%M:%S.%f").timestamp()
                        except ValueError:
                            ts = None
                        if ts is not None and not window[0] <= ts <= window[1]:
                            continue
                    rows.append(parts)
        except OSError:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in rows]
        mx = max(float(r[2]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4)
                          if r[5 + i].lower().startswith("active")})
        loaded = [x for x in sm if x > 0.5 * mx] or sm
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": mx, "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference numeric path (oracle port of rope.py:118-144)
# ---------------------------------------------------------------------------

def _cpu_task(args):
    kept, new, hd, seed = args
    from oracle import rope_ref
    rng = np.random.default_rng(seed)
    keys, values = rng.standard_normal((kept, hd)), rng.standard_normal((kept, hd))
    q, k, v = (rng.standard_normal((new, hd)) for _ in range(3))
    t = time.perf_counter()
    rope_ref.decoupled_attention(keys, values, q, k, v, np.arange(kept))
    return time.perf_counter() - t


def cpu_reference(turns, shape, pairs_per_turn: int, seed: int = 0):
    """Time attention_with_decoupled_cache (float64 numpy, one (layer, head) per
    task) on all host cores; extrapolate to whole turns (L x Hq pairs each)."""
    import multiprocessing as mp

    os.environ["OPENBLAS_NUM_THREADS"] = "1"
    os.environ["OMP_NUM_THREADS"] = "1"
    cores = len(os.sched_getaffinity(0))
    tasks = [(kept, new, shape.head_dim, seed + 97 * i + j)
             for i, (_, _, kept, new) in enumerate(turns) for j in range(pairs_per_turn)]
    ctx = mp.get_context("spawn")
    t0 = time.perf_counter()
    with ctx.Pool(cores) as pool:
        times = pool.map(_cpu_task, tasks, chunksize=1)
    wall = time.perf_counter() - t0
    per_turn = []
    for i in range(len(turns)):
        mean_pair = statistics.fmean(times[i * pairs_per_turn:(i + 1) * pairs_per_turn])
        per_turn.append(mean_pair * shape.layers * shape.n_heads / cores)
    tokens = sum(kept + new for _, _, kept, new in turns)
    return {"value": tokens / sum(per_turn), "cores": cores, "cpu_seconds": sum(times),
            "wall_seconds": wall, "tasks": len(tasks)}


def run_reference(args, shape, turns, config):
    """--impl reference: the reference's CPU implementation of the path (oracle
    port of kvsim.rope.attention_with_decoupled_cache), all host cores."""
    pairs = 4
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_reference(turns, shape, pairs, seed=i)
        if i >= args.warmup:
            vals.append(r)
    value = statistics.median(v["value"] for v in vals)
    ms = statistics.fmean(v["wall_seconds"] for v in vals) * 1e3
    sample = (f"attention_with_decoupled_cache (float64 numpy, rope.py:118-144) on {pairs} "
              f"(layer, head) pairs of each of {len(turns)} hit turns per step, extrapolated "
              f"to {shape.layers}x{shape.n_heads} pairs per turn; projections excluded "
              f"(the reference has none)")
    return {"impl": "reference", "metric": METRIC, "value": value, "unit": "tokens/s",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config,
            "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": vals[0]["cores"],
                             "kind": "port", "sample": sample},
            "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}


def make_config(args, shape, turns, n_hits, world, tp, rank_probe) -> dict:
    """The workload description both arms print (ours and --impl reference)."""
    from paper_2403_19708_b200.metrics import percentile

    kept_l = [kept for *_, kept, _ in turns]
    new_l = [new for *_, new in turns]
    kv_bytes = sum(kept_l) * shape.kv_bytes_per_token
    return {
        "workload": (f"{args.config}: {shape.name}-shaped, reference generate_poisson "
                     f"sessions sharded by crc32(session) over {world} GPU(s); "
                     f"{len(turns)} hit turns/GPU/step (of {n_hits} in shard)"
                     if args.config != "c4" else
                     f"c4: {shape.name}-shaped, W=4096, 32768-token stored histories "
                     f"truncated by the reference rules to kept 2048..3648 (block-table "
                     f"edit; only the kept blocks are materialised and loaded), 256 new "
                     f"tokens per turn, {len(turns)} turns/GPU/step"),
        "turns_per_gpu": len(turns), "kept_p50": percentile(kept_l, 0.5),
        "new_p50": percentile(new_l, 0.5), "block_tokens": args.block_tokens,
        "value_mode": ("KV resident in an HBM arena (no host link); the step's turns in one "
                       "batched layer pass" if getattr(args, "batch_prefill", 0) else
                       "KV resident in an HBM arena (no host link)"),
        "e2e_mode": "KV streamed from pinned host DRAM by the layer-wise pre-loader; "
                    "new-token KV saved back asynchronously",
        "l2": f"inputs larger than L2 (per-step KV {kv_bytes / 1e9:.1f} GB)",
        "parallelism": (f"tensor-parallel tp{tp} (NCCL all-reduce of W_o / W_down "
                        f"partials over NVLink)" if tp > 1 else
                        f"one rank of a tp{args.tp_rank_of} shard, all-reduce excluded "
                        f"(per-rank compute probe; outputs are partial sums)"
                        if rank_probe else
                        f"sessions sharded, no collective ({world} independent ranks)")}


def run_serving(args, rank: int, device: int) -> dict:
    import gc

    import torch

    from paper_2403_19708_b200 import serve
    # every rank of the node pins its own arena: stay within 60 % of the
    # available host memory across the node's ranks
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    dram_gb = min(args.serve_dram_gb, host_mem_available() * 0.6 / local_world / 1e9)
    sa = serve.parse(["--config", args.config, "--shard", str(rank), "--of", "8",
                      "--device", str(device), "--dram-gb", f"{dram_gb:.1f}",
                      "--hbm-gb", str(args.serve_hbm_gb)])
    t0 = time.perf_counter()
    out = serve.run(sa)
    out["wall_s"] = time.perf_counter() - t0
    gc.collect()
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
    if hasattr(torch._C, "_host_emptyCache"):
        torch._C._host_emptyCache()   # return the serving arena's pinned pages
    r, c = out["reuse"], out["recompute"]
    return {"workload": f"{args.config} shard {rank} of 8 ({out['sessions']} sessions, "
                        f"{out['turns']} turns, arrival order)",
            "dram_gb": out["dram_bytes"] / 1e9, "read_buffer_gb": out["read_buffer_bytes"] / 1e9,
            "p50_ttft_s": {"reuse": r["p50_ttft_s"], "recompute": c["p50_ttft_s"]},
            "p99_ttft_s": {"reuse": r["p99_ttft_s"], "recompute": c["p99_ttft_s"]},
            "speedup_p50_ttft": out.get("speedup_p50_ttft"),
            "prefill_tokens_per_s": {"reuse": r["prefill_tokens_per_s"],
                                     "recompute": c["prefill_tokens_per_s"]},
            "exposed_transfer_frac": r["exposed_transfer_frac"],
            "hit_rate": r["overall_hit_rate"], "evict_out": r["evict_out"],
            "hits_with_head_start": r["hits_with_head_start"], "h2d_gbs": r["h2d_gbs"],
            "hbm_tier": ({"gb": out["hbm_tier_bytes"] / 1e9,
                          "p50_ttft_s": out["reuse_hbm_tier"]["p50_ttft_s"],
                          "speedup_p50_ttft": out.get("speedup_p50_ttft_hbm_tier"),
                          "exposed_transfer_frac": out["reuse_hbm_tier"]["exposed_transfer_frac"],
                          "tier_hits": out["reuse_hbm_tier"]["tier_hits"]}
                         if "reuse_hbm_tier" in out else None),
            "by_hit_class": r["by_hit_class"], "wall_s": out["wall_s"],
            "note": "queue-inclusive TTFT (sim.py:489) with every prefill measured on this "
                    "GPU; read-buffer head start min(S_buf, B*wait) from real queue waits; "
                    "decode modeled at 1 ms/step (reference llama-13b profile)"}


def host_info() -> dict:
    """CPU model and the numpy / BLAS build the CPU path runs on."""
    model = platform.processor() or ""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    blas = ""
    try:
        cfg = np.show_config(mode="dicts")
        b = cfg.get("Build Dependencies", {}).get("blas", {})
        blas = f"{b.get('name', '')} {b.get('version', '')}".strip()
    except Exception:  # noqa: BLE001 - informational only
        pass
    return {"cpu_model": model, "numpy": np.__version__, "blas": blas}


def cpu_with_projections(turns, shape, cb) -> dict:
    """The attention-only CPU value plus the model's projections for the same
    turns: one layer's QKV / O / MLP GEMMs (float64 numpy, all cores through
    BLAS threads) timed for each of 2 sample turns and scaled by L."""
    import threading  # noqa: F401  (BLAS threads only)

    rng = np.random.default_rng(0)
    d, f = shape.d_model, shape.ffn
    hq, hkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    w = {"qkv": rng.standard_normal(((hq + 2 * hkv) * hd, d)),
         "o": rng.standard_normal((d, hq * hd)),
         "gu": rng.standard_normal((2 * f, d)), "down": rng.standard_normal((d, f))}
    per_tok = []
    for _, _, _, new in turns[:2]:
        x = rng.standard_normal((new, d))
        t = time.perf_counter()
        qkv = x @ w["qkv"].T
        o = qkv[:, :hq * hd] @ w["o"].T
        gu = o @ w["gu"].T
        _ = gu[:, :f] @ w["down"].T
        per_tok.append((time.perf_counter() - t) * shape.layers / new)
    proj_s_per_tok = statistics.fmean(per_tok)
    tokens = sum(kept + new for _, _, kept, new in turns)
    new_total = sum(new for *_, new in turns)
    attn_s = tokens / cb["value"]
    total_s = attn_s + proj_s_per_tok * new_total
    return {"value": tokens / total_s, "unit": "tokens/s",
            "projection_s_per_new_token": proj_s_per_tok,
            "sample": "attention (above) + numpy float64 QKV/O/gate-up/down GEMMs of one "
                      "layer for 2 sample turns, scaled by L, BLAS threads on all cores"}


def cpu_c1_whole_turns() -> dict:
    """Config C1 end to end on the CPU path: all 12 turns of the reference's
    4 tiny sessions through the float64 oracle forward (projections, RoPE,
    attention over the whole conversation, as kvsim would recompute it)."""
    from oracle import llama_ref
    from paper_2403_19708_b200 import model
    wl = json.loads((ROOT / "tests" / "golden" / "workload_c1.json").read_text())
    shape = model.shape("tiny")
    rng = np.random.default_rng(0)
    sd = 0.02
    L, d, f = shape.layers, shape.d_model, shape.ffn
    hq, hkv, hd = shape.n_heads, shape.n_kv_heads, shape.head_dim
    w = {"embed": rng.standard_normal((shape.vocab, d)) * sd,   # oracle [in, out] layout
         "layers": [{"w_in": np.ones(d),
                     "wqkv": rng.standard_normal((d, (hq + 2 * hkv) * hd)) * sd,
                     "wo": rng.standard_normal((hq * hd, d)) * sd, "w_post": np.ones(d),
                     "wg": rng.standard_normal((d, f)) * sd,
                     "wu": rng.standard_normal((d, f)) * sd,
                     "wd": rng.standard_normal((f, d)) * sd} for _ in range(L)],
         "w_final": np.ones(d), "lm_head": rng.standard_normal((d, shape.vocab)) * sd}
    empty = [(np.zeros((0, hkv, hd)),) * 2] * L
    tokens = 0
    t = time.perf_counter()
    for k in range(3):
        for s in wl["sessions"]:
            hist = sum(a + b for a, b in s["turns"][:k])
            ids = rng.integers(0, shape.vocab, hist + s["turns"][k][0])
            llama_ref.forward(w, ids, empty, np.arange(0), n_heads=hq, n_kv_heads=hkv,
                              head_dim=hd)
            tokens += len(ids)
    dt = time.perf_counter() - t
    return {"value": tokens / dt, "unit": "tokens/s", "turns": 12, "prompt_tokens": tokens,
            "seconds": dt, "cores": 1,
            "sample": "C1 (tiny, 4 sessions x 3 turns): every turn's whole prompt through "
                      "the float64 oracle forward (oracle/llama_ref.py), one process"}


# ---------------------------------------------------------------------------
# GPU arm
# ---------------------------------------------------------------------------

def host_mem_available() -> int:
    try:
        for line in open("/proc/meminfo"):
            if line.startswith("MemAvailable:"):
                return int(line.split()[1]) * 1024
    except OSError:
        pass
    return 1 << 62


def link_peak(host_u8: torch.Tensor, dev_u8: torch.Tensor, nbytes: int = 1 << 30) -> dict:
    """Host-link peak of this box: one plain pinned-host <-> HBM cudaMemcpyAsync
    of `nbytes` per direction (best of 3, CUDA events).  The roofline the
    pre-loader (K1) and saver (K4) are judged against."""
    import torch
    n = min(nbytes, host_u8.numel(), dev_u8.numel())
    s = torch.cuda.Stream()
    out = {}
    for name, dst, src in (("h2d", dev_u8[:n], host_u8[:n]), ("d2h", host_u8[:n], dev_u8[:n])):
        best = None
        for _ in range(3):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record()
                dst.copy_(src, non_blocking=True)
                e1.record()
            e1.synchronize()
            t = e0.elapsed_time(e1) * 1e-3
            best = t if best is None else min(best, t)
        out[name] = n / best / 1e9
    # each direction while the other runs for the whole interval (K1 pre-loads
    # and K4 saves share the link in e2e): the measured copy moves n/4, the
    # background one n/2
    s2 = torch.cuda.Stream()
    q = n // 4
    for name, fg in (("h2d_concurrent", "h2d"), ("d2h_concurrent", "d2h")):
        best = None
        for _ in range(3):
            e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
            torch.cuda.synchronize()
            with torch.cuda.stream(s2):   # background: the other direction, 2x longer
                if fg == "h2d":
                    host_u8[q:3 * q].copy_(dev_u8[q:3 * q], non_blocking=True)
                else:
                    dev_u8[q:3 * q].copy_(host_u8[q:3 * q], non_blocking=True)
            with torch.cuda.stream(s):
                e[0].record()
                if fg == "h2d":
                    dev_u8[:q].copy_(host_u8[:q], non_blocking=True)
                else:
                    host_u8[:q].copy_(dev_u8[:q], non_blocking=True)
                e[1].record()
            torch.cuda.synchronize()
            t = e[0].elapsed_time(e[1]) * 1e-3
            best = t if best is None else min(best, t)
        out[name] = q / best / 1e9
    # the saver's own shape: D2H in 2 MB pieces (a layer's new rows of one
    # turn split at block boundaries) while an H2D streams -- per-DMA setup
    # and the shared link cap small pieces well below the large-copy rate
    piece = 2 << 20
    best = None
    for _ in range(3):
        e = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        torch.cuda.synchronize()
        with torch.cuda.stream(s2):
            dev_u8[q:3 * q].copy_(host_u8[q:3 * q], non_blocking=True)
        with torch.cuda.stream(s):
            e[0].record()
            for off in range(0, q - piece + 1, piece):
                host_u8[off:off + piece].copy_(dev_u8[off:off + piece], non_blocking=True)
            e[1].record()
        torch.cuda.synchronize()
        t = e[0].elapsed_time(e[1]) * 1e-3
        best = t if best is None else min(best, t)
    out["d2h_concurrent_2mb"] = (q // piece) * piece / best / 1e9
    return out


def disk_probe(root, arena, bids, block_bytes, rows):
    """Disk tier (§8f-4): write one session's blocks from the pinned arena to
    a file and read them back (IO-thread pool, O_DIRECT when the file system
    allows); GB/s of each direction on this box's disk."""
    import shutil
    import tempfile
    from paper_2403_19708_b200.disk import DiskTier
    d = tempfile.mkdtemp(prefix="askv-disk-", dir=root)
    fs = "?"
    try:
        best = ""
        for line in open("/proc/mounts"):
            parts = line.split()
            if len(parts) > 2 and d.startswith(parts[1]) and len(parts[1]) > len(best):
                best, fs = parts[1], parts[2]
    except OSError:
        pass
    tier = DiskTier(d, block_bytes)
    try:
        nbytes = len(bids) * block_bytes
        t0 = time.perf_counter()
        tier.write("probe", arena, bids, 0, rows, 0).result()
        os.sync()
        t_w = time.perf_counter() - t0
        t0 = time.perf_counter()
        tier.read("probe", arena, bids).result()
        t_r = time.perf_counter() - t0
        direct = tier.direct
    finally:
        tier.close()
        shutil.rmtree(d, ignore_errors=True)
    return {"session_bytes": nbytes, "write_gbs": nbytes / t_w / 1e9,
            "read_gbs": nbytes / t_r / 1e9, "read_s": t_r, "fs": fs,
            "o_direct_requested": direct,
            "note": "one C3 session's blocks, pinned DRAM <-> file; a disk hit adds read_s "
                    "before the layer-wise pre-load"}


def main():
    args = parse()
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    sys.path.insert(0, str(ROOT))
    from paper_2403_19708_b200 import model

    shape = model.shape(CONFIGS[args.config][0])
    tp = world if args.config == "c5" else 1
    rank_probe = args.config == "c5" and world == 1 and args.tp_rank_of > 1
    if rank_probe:   # one TP rank's shard on this GPU, no all-reduce partner
        shape = shape.tp_shard(args.tp_rank_of)
    if tp > 1:
        # C5: one model replica tensor-parallel over all ranks (head-parallel
        # attention + KV store slice per rank, NCCL all-reduce after W_o / W_down)
        shape = shape.tp_shard(tp)
        turns, n_hits = select_turns("c3", 0, 1, args.turns)
    else:
        turns, n_hits = select_turns("c3" if args.config == "c5" else args.config, rank,
                                     world, args.turns)

    if args.impl == "reference":
        if rank == 0:
            tp_ref = world if args.config == "c5" else 1
            probe_ref = args.config == "c5" and world == 1 and args.tp_rank_of > 1
            cfg = make_config(args, shape, turns, n_hits, world, tp_ref, probe_ref)
            print(json.dumps(run_reference(args, shape, turns, cfg)), flush=True)
        return

    import torch
    import torch.distributed as dist

    if not torch.cuda.is_available():
        raise SystemExit("bench.py needs a CUDA device (no CPU fallback)")
    # ASKV_BENCH_ONE_GPU=1 (test hook): every rank on cuda:0 with a gloo group,
    # to exercise the N>1 path (sharding, barriers, max/sum over ranks) on a
    # 1-GPU box; never used for reported numbers
    one_gpu = os.environ.get("ASKV_BENCH_ONE_GPU") == "1"
    local = 0 if one_gpu else local
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    from paper_2403_19708_b200 import dist as pdist
    if world > 1:
        pdist.init("gloo" if one_gpu else "nccl", dev)


    from paper_2403_19708_b200 import build as _build
    from paper_2403_19708_b200.metrics import percentile

    # measured serving replay: this rank's
    # shard (1 of 8 -- the shard a GPU of an 8-GPU node serves) of the
    # reference workload in arrival order through the reference serving loop,
    # every prefill / save run on this GPU; before the bench's own arena so
    # the two pinned arenas never coexist
    serving = None
    if (args.config in ("c2", "c3") and args.serve_dram_gb > 0 and tp == 1 and not rank_probe
            and rank < 8):
        serving = run_serving(args, rank, local)
    from paper_2403_19708_b200.runner import Job, Runner, attention_flops
    from paper_2403_19708_b200.store import HostArena

    _build.build()
    tb = args.block_tokens
    block_bytes = tb * shape.kv_bytes_per_token
    nbs = [-(-(kept + new) // tb) for _, _, kept, new in turns]
    # every rank pins its turns' blocks in host DRAM (13B: ~1.9 GB per turn);
    # keep all ranks of the node within half the available memory
    host_budget = host_mem_available() // 2 // int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    while len(turns) > 4 and sum(nbs) * block_bytes > host_budget:
        turns, nbs = turns[:-1], nbs[:-1]
    dec_steps = args.decode_steps
    # decode probe (§8f-2): the first sampled turn gets its own blocks with room
    # for the decoded tokens
    dec_nb = -(-(turns[0][2] + turns[0][3] + dec_steps) // tb) if dec_steps else 0
    n_blocks = sum(nbs) + dec_nb
    max_new = max(new for *_, new in turns)
    max_kept = max(kept for *_, kept, _ in turns)
    # arenas: the same block ids in the pinned host arena and the HBM arena
    # this rank's pinned arena on its GPU's NUMA node
    from paper_2403_19708_b200 import numa as _numa
    numa_node = _numa.gpu_numa_node(local)
    arena = HostArena(n_blocks, block_bytes, pin=True, numa_node=numa_node)
    hbm = torch.empty(n_blocks * block_bytes // 2, dtype=torch.bfloat16, device=dev)
    g = torch.Generator(device=dev).manual_seed(7 + rank)
    chunk = 1 << 28
    host_bf = arena.buffer.view(torch.bfloat16)
    for off in range(0, hbm.numel(), chunk):
        m = min(chunk, hbm.numel() - off)
        hbm[off:off + m].normal_(generator=g)
        host_bf[off:off + m].copy_(hbm[off:off + m])
    torch.cuda.synchronize()
    tp_hook = None
    if tp > 1:
        tp_hook = pdist.NcclComm(rank, world)   # native: ncclAllReduce inside the layer graph
    runner = Runner(shape, device=dev, seed=rank if tp > 1 else 0, block_tokens=tb,
                    host_arena=arena, tp_reduce=tp_hook,
                    hbm_arena=hbm, read_buffer_bytes=4 << 30,
                    # batched value mode: every (job, layer) of a step holds its
                    # own write-buffer slot while the batch runs
                    write_buffer_bytes=max(1 << 30, (len(turns) * shape.layers
                                                     * max(max_new, 1) * shape.row_bytes
                                                     if args.batch_prefill else 0)),
                    max_new=max(max_new, 1), max_ctx=max(shape.context_window, max_kept + 1),
                    # tune the GEMMs over the recompute baseline's prompt lengths too
                    autotune=max(shape.context_window, max_kept + 1) + max(max_new, 1),
                    overlap=bool(args.k2_overlap))
    # block placement: the arena allocator's contiguous runs (what a session
    # gets in serving, store.HostArena) or, with --fragmented, a random
    # permutation (every block of a layer its own DMA)
    if args.fragmented:
        ids_perm = np.random.default_rng(99 + rank).permutation(n_blocks)
    else:
        ids_perm = np.concatenate([np.asarray(arena.alloc(nb), dtype=np.int64) for nb in nbs]
                                  + ([np.asarray(arena.alloc(dec_nb), dtype=np.int64)]
                                     if dec_nb else []))
    jobs = {"host": [], "hbm": [], "recompute": []}
    pos = 0
    trng = np.random.default_rng(5 + rank)
    elems_per_block = block_bytes // 2
    for (sid0, k, kept, new), nb in zip(turns, nbs):
        sid = f"{sid0}#{k}"  # each sampled turn owns its own synthetic blocks
        bids = [int(b) for b in ids_perm[pos:pos + nb]]
        pos += nb
        new_ids = torch.as_tensor(trng.integers(0, shape.vocab, new)).pin_memory()
        prompt_ids = torch.as_tensor(trng.integers(0, shape.vocab, kept + new)).pin_memory()
        off = torch.as_tensor([b * elems_per_block for b in bids], dtype=torch.int64,
                              device=dev)
        jobs["host"].append(Job(sid, new_ids, kept=kept, source="host", block_ids=bids,
                                save=True))
        jobs["hbm"].append(Job(sid, new_ids.to(dev), kept=kept, source="hbm", block_ids=bids,
                               save=True, dev_block_off=off))
        jobs["recompute"].append(Job(sid, prompt_ids.to(dev)))
    dec_bids = [int(b) for b in ids_perm[pos:pos + dec_nb]]
    prompt_tokens = sum(kept + new for *_, kept, new in turns)
    new_tokens = sum(new for *_, new in turns)

    def barrier():
        if world > 1:
            dist.barrier()

    red_dev = torch.device("cpu") if one_gpu else dev

    def max_over_ranks(x: float) -> float:
        return pdist.max_over_ranks(x, red_dev)

    def sum_over_ranks(x: float) -> float:
        return pdist.sum_over_ranks(x, red_dev)

    def timed(mode: str, steps: int, warmup: int, probe: bool = False, clocks=None,
              batch: bool = False):
        js = jobs[mode]
        sampler = ClockSampler(local) if clocks is not None and \
            os.environ.get("ASKV_BENCH_CLOCKS", "1") != "0" else None
        if sampler:
            sampler.__enter__()
        runner.probe = [] if probe else None   # same graph shapes as the timed steps
        for _ in range(warmup):
            runner.run(js, batch=batch)
            runner.join()
        torch.cuda.synchronize()
        barrier()
        runner.probe = [] if probe else None
        launches0 = runner.launches
        cs = runner.s_compute
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        w0 = time.time()
        e0.record(cs)
        res = None
        for _ in range(steps):
            res = runner.run(js, batch=batch)
            runner.join()
        e1.record(cs)
        torch.cuda.synchronize()
        w1 = time.time()
        if sampler:
            sampler.__exit__(None, None, None)
            clocks.update(sampler.summary((w0, w1)))
        barrier()
        ms = e0.elapsed_time(e1)
        launches = runner.launches - launches0
        Runner.finalize(res)
        probe_rec = runner.probe
        runner.probe = None
        return ms, res, launches, probe_rec

    clocks: dict = {}
    if args.profile_attn:
        timed("hbm", 2, 1)
        return

    # e2e (headline) — KV from the pinned host arena, clocks sampled here
    ms_host, res_host, launches, _ = timed("host", args.steps, args.warmup, clocks=clocks)
    # value — KV resident in HBM; probe the attention / re-embed launches
    clocks_value: dict = {}
    ms_hbm, res_hbm, _, probe = timed("hbm", args.steps, args.warmup,
                                      probe=not args.batch_prefill, clocks=clocks_value)
    # value, batched (scheduler knob): the step's turns in one pass over the
    # layers -- GEMMs over all their new tokens, K2 / K3 / saves per turn
    ms_batch = None
    if args.batch_prefill:
        clocks_batch: dict = {}
        # the headline configuration: the kernel probes (K3 / K2 rooflines) ride here
        ms_batch, _, _, probe = timed("hbm", args.steps, args.warmup, probe=True,
                                      clocks=clocks_batch, batch=True)
    # recompute baseline
    ms_re, res_re, _, _ = timed("recompute", max(2, args.steps // 2), 1)
    # prestaged TTFT: each turn starts once its whole KV sits in the read buffer
    for j in jobs["host"]:
        j.prestage = True
    _, res_pre, _, _ = timed("host", 1, 1)
    for j in jobs["host"]:
        j.prestage = False

    # isolated requests: one job on an idle GPU, wall clock from the host call
    # to the first token on the host, with a prompt length the runner has not
    # seen (n - 1): includes GEMM-plan / graph-update host work and launch
    # latency, i.e. what a lone request waits (HBM-resident KV)
    iso = []
    for j in jobs["hbm"][:8]:
        if j.n_new < 3:
            continue
        for cut, timed_run in ((2, False), (1, True)):   # warm server, then an unseen length
            jj = Job(j.session_id + "/iso", j.token_ids[:-cut], kept=j.kept, source="hbm",
                     block_ids=j.block_ids, save=False, dev_block_off=j.dev_block_off)
            torch.cuda.synchronize()
            w0 = time.perf_counter()
            r = runner.run([jj])
            r[0].first_token.numpy()
            torch.cuda.synchronize()
            if timed_run:
                iso.append(time.perf_counter() - w0)
            Runner.finalize(r)

    decode = None
    if dec_steps:
        from paper_2403_19708_b200.runner import ResidentKv
        _, _, d_kept, d_new = turns[0]
        kvres = ResidentKv(shape, d_kept + d_new + dec_steps, dev)
        d_ids = torch.as_tensor(trng.integers(0, shape.vocab, d_new)).pin_memory()

        def decode_turn():
            # prompt from host DRAM into the resident cache, then greedy steps;
            # every step's K|V row is saved to host DRAM on the save stream
            kvres.rows = 0
            r0 = runner.run([Job("decode", d_ids, kept=d_kept, source="host", block_ids=dec_bids,
                                 save=True, kv_cache=kvres)])[0]
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(runner.s_compute)
            tok, steps_res = r0.next_token, []
            for s in range(dec_steps):
                r = runner.run([Job("decode", tok, kept=d_kept + d_new + s, source="resident",
                                    block_ids=dec_bids, save=True, kv_cache=kvres)])[0]
                steps_res.append(r)
                tok = r.next_token
            e1.record(runner.s_compute)
            runner.join()
            torch.cuda.synchronize()
            Runner.finalize([r0] + steps_res)
            return e0.elapsed_time(e1), steps_res

        decode_turn()  # warm-up
        d_ms, d_res = decode_turn()
        spans = [r.timeline.makespan for r in d_res]
        saves = [b - a for r in d_res for a, b in r.timeline.save_intervals]
        decode = {"steps": dec_steps, "context": d_kept + d_new,
                  "tpot_ms": d_ms / dec_steps,
                  "tpot_makespan_p50_ms": percentile(spans, 0.5) * 1e3,
                  "tokens_per_s": dec_steps / (d_ms * 1e-3),
                  "d2h_bytes_per_token": shape.kv_bytes_per_token,
                  "save_busy_ms_per_token": sum(saves) / dec_steps * 1e3,
                  "note": "batch-1 greedy decode with every layer's rotated KV resident in "
                          "HBM; per-token K|V saved to pinned host DRAM asynchronously "
                          "(overlap.py:126-200 decode branch); weight-bandwidth bound"}

    # host-link roofline (plain 1 GB copies each way, after the timed regions)
    link = link_peak(arena.buffer, hbm.view(torch.uint8))
    disk = None
    if args.disk_dir != "none" and rank == 0:
        disk = disk_probe(args.disk_dir, arena, [int(b) for b in ids_perm[:nbs[0]]],
                          block_bytes, turns[0][2] + turns[0][3])

    steps_re = max(2, args.steps // 2)
    t_host = max_over_ranks(ms_host) * 1e-3
    t_hbm = max_over_ranks(ms_hbm) * 1e-3
    t_re = max_over_ranks(ms_re) * 1e-3
    # weak scaling: ranks serve disjoint sessions (sum); C5 TP: one replica (its tokens)
    tok_all = prompt_tokens if tp > 1 else sum_over_ranks(prompt_tokens)
    new_all = new_tokens if tp > 1 else sum_over_ranks(new_tokens)
    turns_all = len(turns) if tp > 1 else sum_over_ranks(len(turns))
    value_unbatched = tok_all * args.steps / t_hbm
    t_batch = max_over_ranks(ms_batch) * 1e-3 if ms_batch is not None else None
    value = tok_all * args.steps / t_batch if t_batch else value_unbatched
    e2e = tok_all * args.steps / t_host
    recompute = tok_all * steps_re / t_re

    # roofline of the dominant kernel (K3 attention), live CUDA-event durations
    # device timestamps (globaltimer) around each K3 / K2 launch inside the layer graphs
    dur = runner.probe_durations(probe)
    att = [(t, w) for kind, t, w, _ in dur if kind == "attention"]
    emb = [(t, w) for kind, t, w, _ in dur if kind == "reembed"]
    emb_moved = sum(m for kind, _, _, m in dur if kind == "reembed")
    peaks = json.loads((ROOT / "MEASURED_PEAKS.json").read_text()) \
        if (ROOT / "MEASURED_PEAKS.json").exists() else {}
    tflops_peak = peaks.get("bf16_tflops_sustained", 1400.0)
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    att_tflops = sum(w for _, w in att) / sum(t for t, _ in att) / 1e12
    emb_gbs = sum(w for _, w in emb) / sum(t for t, _ in emb) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "ncu_attn_traffic.json"
    if tf.exists():
        traffic = json.loads(tf.read_text()).get("bytes_per_launch")

    # TTFT / exposed transfer / link GB/s from the measured timelines
    def ttfts(res):
        return [r.timeline.makespan for r in res]

    ttft_host = percentile(ttfts(res_host), 0.5)
    ttft_hbm = percentile(ttfts(res_hbm), 0.5)
    ttft_re = percentile(ttfts(res_re), 0.5)
    ttft_pre = percentile(ttfts(res_pre), 0.5)
    stall_host = sum(r.timeline.stall_total for r in res_host)
    span_host = sum(r.timeline.makespan for r in res_host)
    stall_pre = sum(r.timeline.stall_total for r in res_pre)
    span_pre = sum(r.timeline.makespan for r in res_pre)
    load_busy = sum(r.timeline.load_total for r in res_host)
    save_busy = sum(r.timeline.save_total for r in res_host)
    h2d_bytes = sum(r.bytes_loaded for r in res_host)
    d2h_bytes = sum(r.bytes_saved for r in res_host)
    h2d_step = h2d_bytes + sum(j.n_new * 8 for j in jobs["host"])
    d2h_step = d2h_bytes + 8 * len(jobs["host"])

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:   # N=1 only (contract)
        cb = cpu_reference(turns, shape, pairs_per_turn=24)
        cpu = {"value": cb["value"], "unit": "tokens/s", "cores": cb["cores"], "kind": "port",
               **host_info(),
               "with_projections": cpu_with_projections(turns, shape, cb),
               "c1_whole_turns": cpu_c1_whole_turns(),
               "sample": (f"oracle port of attention_with_decoupled_cache (rope.py:118-144, "
                          f"float64 numpy, 1 thread/process) on 24 (layer, head) pairs of each "
                          f"of the {len(turns)} rank-0 turns ({cb['cpu_seconds']:.1f} CPU-s), "
                          f"extrapolated to {shape.layers}x{shape.n_heads} pairs per turn; "
                          f"projections excluded")}

    kept_l = [kept for *_, kept, _ in turns]
    new_l = [new for *_, new in turns]
    line = {
        "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": (ms_batch if ms_batch is not None else ms_hbm) / args.steps,
        "value_unbatched": {"value": value_unbatched, "ms_per_step": ms_hbm / args.steps,
                            "note": "value mode with one turn after another (each turn its "
                                    "own layer pass: the TTFT-optimal schedule)"},
        "batch_prefill": ({"turns_per_batch": len(turns), "ms_per_step": ms_batch / args.steps,
                           "clocks": clocks_batch,
                           "note": "the step's turns in one pass over the layers: norms, "
                                   "projections and MLP over all their new tokens, pre-load "
                                   "wait / K2 / K3 / saves per turn (scheduler knob "
                                   "--batch-prefill; trades TTFT for throughput)"}
                          if ms_batch is not None else None),
        "higher_is_better": True, "scaling": "strong" if tp > 1 else "weak",
        "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (reference ShareGPT-shaped session generator; random-init weights "
                "and KV)",
        "config": make_config(args, shape, turns, n_hits, world, tp, rank_probe),
        "e2e": {"value": e2e, "unit": "tokens/s", "h2d_bytes_per_step": h2d_step,
                "d2h_bytes_per_step": d2h_step, "ms_per_step": ms_host / args.steps},
        # SURVEY.md §8d/§8e companions: new-token throughput and sessions (turns)/s,
        # whole job (all ranks), HBM-resident and host-link modes
        "new_tokens_per_s": {"value_mode": new_all * args.steps / t_hbm,
                             "e2e_mode": new_all * args.steps / t_host},
        "sessions_per_s": {"value_mode": turns_all * args.steps / t_hbm,
                           "e2e_mode": turns_all * args.steps / t_host},
        "recompute": {"value": recompute, "unit": "tokens/s",
                      "ms_per_step": ms_re / steps_re},
        "speedup_vs_recompute": {"value_mode": value / recompute, "e2e_mode": e2e / recompute},
        "ttft_p50_s": {"reuse_host_saturated": ttft_host, "reuse_host_prestaged": ttft_pre,
                       "reuse_hbm": ttft_hbm, "recompute": ttft_re,
                       "speedup_prestaged": ttft_re / ttft_pre if ttft_pre else None,
                       "speedup_saturated": ttft_re / ttft_host if ttft_host else None},
        "ttft_isolated_hbm_s": {"p50": percentile(iso, 0.5) if iso else None,
                                "turns": len(iso),
                                "note": "one request on an idle, warm server (GPU idle), host "
                                        "wall time from the call to the first token on the "
                                        "host, prompt length not seen before"},
        "exposed_transfer_frac": {"host_saturated": stall_host / span_host,
                                  "host_prestaged": stall_pre / span_pre},
        "link_gbs_per_gpu": {"h2d": h2d_bytes / load_busy / 1e9 if load_busy else None,
                             "d2h": d2h_bytes / save_busy / 1e9 if save_busy else None,
                             "h2d_bytes_per_step": h2d_bytes},
        "roofline": {"kernel": "askv_prefill_attn (K3, tcgen05)", "bound": "tensor",
                     "achieved": att_tflops, "peak": tflops_peak, "unit": "TFLOP/s",
                     "frac": att_tflops / tflops_peak, "traffic": traffic,
                     "peak_source": "MEASURED_PEAKS.json bf16_tflops_sustained",
                     "flops_per_launch": statistics.fmean(w for _, w in att),
                     "launches": len(att)},
        "roofline_link": {"kernel": "K1 askv_preload_layer (H2D copy-engine DMAs: strided "
                                    "2-D runs of contiguous arena blocks)",
                          "bound": "host link",
                          "achieved": h2d_bytes / load_busy / 1e9 if load_busy else None,
                          "peak": link["h2d"], "unit": "GB/s",
                          "frac": (h2d_bytes / load_busy / 1e9) / link["h2d"] if load_busy else None,
                          "e2e_frac": (h2d_step / (ms_host / args.steps * 1e-3) / 1e9) / link["h2d"],
                          "d2h_peak": link["d2h"],
                          "h2d_peak_with_d2h_running": link["h2d_concurrent"],
                          "block_placement": "random permutation" if args.fragmented
                                             else "arena allocator (contiguous runs)",
                          "peak_source": "measured in this run: one 1 GB pinned-host->HBM "
                                         "cudaMemcpyAsync, best of 3"},
        # K4: the saver's D2H runs while K1 streams the next layers in (e2e),
        # so its roofline is the D2H rate measured under a concurrent H2D
        "roofline_save": {"kernel": "K4 askv_save_layer (D2H of the new tokens' rows)",
                          "bound": "host link (D2H with H2D running)",
                          "achieved": d2h_bytes / save_busy / 1e9 if save_busy else None,
                          "peak": link["d2h_concurrent"], "unit": "GB/s",
                          "frac": ((d2h_bytes / save_busy / 1e9) / link["d2h_concurrent"]
                                   if save_busy else None),
                          "d2h_peak_alone": link["d2h"],
                          "d2h_peak_2mb_pieces": link["d2h_concurrent_2mb"],
                          "frac_of_2mb_pieces": ((d2h_bytes / save_busy / 1e9)
                                                 / link["d2h_concurrent_2mb"]
                                                 if save_busy else None),
                          "peak_source": "measured in this run: 256 MB D2H while a 512 MB "
                                         "H2D runs on another stream, best of 3; the 2 MB-"
                                         "piece figure is the same D2H cut into the saver's "
                                         "piece size"},
        "roofline_reembed": {"kernel": "askv_reembed (K2)", "bound": "hbm",
                             "achieved": emb_gbs, "peak": hbm_peak, "unit": "GB/s",
                             "frac": emb_gbs / hbm_peak,
                             "bytes_per_launch": statistics.fmean(w for _, w in emb),
                             "bytes_moved_per_launch": emb_moved / max(1, len(emb)),
                             "us_per_launch": sum(t for t, _ in emb) / max(1, len(emb)) * 1e6,
                             "work": "SURVEY §8(d): read + write of the kept rows' K "
                                     "(kept x Hkv x hd x 2 B each way); V rows stay in "
                                     "place except the last partial 128-row tile"},
        "decode": decode,
        "disk": disk,
        "gpu_launches": launches,
        # during the headline `value` timed region (the batched one when batching)
        "clocks": clocks_batch if ms_batch is not None else clocks_value,
        "clocks_value_unbatched": clocks_value if ms_batch is not None else None,
        "clocks_e2e": clocks,            # during the `e2e` timed region
        "cpu_baseline": cpu,
        "serving": serving,
        "host_arena": {"numa_node": arena.numa_node, "numa_nodes": _numa.node_count(),
                       "bytes": arena.n_blocks * arena.block_bytes},
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
