"""Serve a reference workload on one GPU in measured mode and report the
reference's metrics: every turn of the rank's session shard, in arrival
order, through the reference serving loop (job queue, continuous batching,
truncation, scheduler-aware eviction / prefetch) with each prefill and save
run on this GPU (measured.MeasuredExecutor).  Queue waits give the
read-buffer head start min(S_buf, B * wait) (sim.py:436-442); the read buffer
S_buf is sized by the reference's preload_buffer_size (model.py:273-287) over
the workload's hit turns.

    python -m paper_2403_19708_b200.serve --config c3 --shard 0 --of 8 --json out.json
    python -m paper_2403_19708_b200.serve --config c3 --of 8 --load 8   # 8x the arrival rate

Reports, for reuse and for the recompute comparator (Mode.RECOMPUTE):
queue-inclusive p50 / p99 TTFT (sim.py:489), isolated prefill p50
(Timeline.makespan), prefill tokens/s (metrics.py:118-119), hit rates and the
exposed-transfer fraction sum(stall) / sum(prefill) (overlap.py:118).
"""

from __future__ import annotations

import argparse
import json
import os
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent

CONFIGS = {  # workload fixture (the reference generator's sessions), model shape
    "c2": ("workload_c2.json", "7b"),
    "c3": ("workload_c3.json", "13b"),
}


def read_buffer_bytes(workload, prof, tiers, block_tokens: int, row_bytes: int,
                      layers: int, cap: float) -> int:
    """S_buf for this workload: the largest preload_buffer_size over its
    turns (model.py:273-287, paper PAPER.md:298-299), capped at `cap`, and at
    least L + 1 slots of the largest kept history (the ring's minimum)."""
    from .model import preload_buffer_size

    w, cut = prof.context_window, prof.cut_tokens
    from .engine import overflow_kept, save_truncate

    need, max_kept = 0.0, 0
    for s in workload.sessions:
        ctx = 0
        for k, t in enumerate(s.turns):
            kept = overflow_kept(ctx, t.new_input_tokens, w, cut)
            if k and kept:
                need = max(need, preload_buffer_size(kept, t.new_input_tokens, prof, tiers))
                max_kept = max(max_kept, kept)
            ctx = save_truncate(kept + t.new_input_tokens + t.output_tokens, w, cut)
    slot = (-(-(max_kept + block_tokens) // block_tokens) * block_tokens) * row_bytes
    return int(max(min(need, cap), (layers + 1) * slot))


def run(args) -> dict:
    import torch

    from . import build as _build
    from . import engine as E
    from . import measured, model, sim
    from .dist import shard_of
    from .metrics import summarize
    from .policy import PolicyConfig

    _build.build()
    torch.cuda.set_device(args.device)
    dev = torch.device("cuda", args.device)
    fixture, shape_name = CONFIGS[args.config]
    raw = json.loads((ROOT / "tests" / "golden" / fixture).read_text())
    ids = None
    if args.of > 1:
        ids = [s["id"] for s in raw["sessions"] if shard_of(s["id"], args.of) == args.shard]
    wl = sim.workload_from_dict(raw, ids)
    if args.max_sessions:
        wl.sessions = wl.sessions[:args.max_sessions]
    if args.load != 1.0:
        # k x the reference's offered load: session starts and think times
        # (the gaps between a session's generator arrivals, sim.py:493) / k
        wl.sessions = [sim.Session(x.session_id, x.turns,
                                   tuple(a / args.load for a in x.arrival_times))
                       for x in wl.sessions]
    shape = model.shape(shape_name)
    tb = args.block_tokens
    bb = tb * shape.kv_bytes_per_token
    # the reference's per-token prefill slope only feeds preload_buffer_size;
    # decode stays modeled (batched decode, 1 ms/step: the reference's
    # llama-13b profile, model.py:167-175) -- it is outside the prefill path
    prof0 = model.profile_for(shape, prefill_seconds_per_token=args.prefill_s_per_token,
                              decode_seconds_per_step=args.decode_s_per_step)
    tiers0 = model.TierConfig(pcie_bandwidth=args.link_gbs * 1e9, disk_capacity=0,
                              dram_capacity=int(args.dram_gb * 1e9))
    rb = read_buffer_bytes(wl, prof0, tiers0, tb, shape.row_bytes, shape.layers,
                           cap=args.read_buffer_gb * 1e9)
    dram = int(args.dram_gb * 1e9) // bb * bb
    # physical spare beyond the accounting capacity: rows of the job in flight
    # and of its append before save() trims (2 windows of blocks)
    spare = 2 * (-(-(shape.context_window + 4096) // tb))
    host_blocks = dram // bb + spare
    from . import numa
    node = numa.gpu_numa_node(args.device) if args.numa_node < 0 else args.numa_node
    t_alloc = time.perf_counter()
    hbm_blocks = int(args.hbm_gb * 1e9) // bb
    eng = E.Engine(shape, host_blocks=host_blocks, block_tokens=tb, device=dev, seed=0,
                   read_buffer_bytes=rb, max_new=4096, dram_bytes=dram, hbm_blocks=hbm_blocks,
                   autotune=True if args.autotune < 0 else args.autotune, policy=PolicyConfig(),
                   numa_node=node)
    t_alloc = time.perf_counter() - t_alloc
    tiers = model.TierConfig(hbm_read_buffer=rb, hbm_write_buffer=int(2e9),
                             dram_capacity=eng.store.mem_capacity, disk_capacity=0,
                             pcie_bandwidth=args.link_gbs * 1e9)
    cfg = sim.SimConfig(profile=prof0, tiers=tiers, block_bytes=bb,
                        batch_size=args.batch_size)
    out = {"config": args.config, "model": shape_name, "shard": [args.shard, args.of],
           "load": args.load,
           "sessions": len(wl.sessions), "turns": sum(len(s.turns) for s in wl.sessions),
           "dram_bytes": eng.store.mem_capacity, "read_buffer_bytes": rb,
           "block_tokens": tb, "batch_size": args.batch_size,
           "decode_s_per_step": args.decode_s_per_step, "setup_s": t_alloc,
           "numa_node": eng.arena.numa_node,
           "data": "synthetic: reference generator sessions, random-init weights, random ids"}
    modes = ["reuse", "recompute"] if not args.reuse_only else ["reuse"]
    tier = eng.hbm
    if tier is not None:
        modes.append("reuse_hbm_tier")
        out["hbm_tier_bytes"] = hbm_blocks * bb
    for mode in modes:
        # the HBM session tier only in its own mode
        eng.hbm = tier if mode == "reuse_hbm_tier" else None
        eng.store.on_release = tier.drop if eng.hbm is not None else None
        if tier is not None:
            for sid in list(tier.tab):
                tier.drop(sid)
        t0 = time.perf_counter()
        log, ex = measured.serve(wl, eng, cfg, recompute=mode == "recompute")
        wall = time.perf_counter() - t0
        s = summarize(log)
        s["host_wall_s"] = wall
        s["jobs"] = ex.jobs
        if mode == "reuse_hbm_tier":
            s["tier_hits"], s["tier_promotions"] = tier.hits, tier.promotions
        if mode.startswith("reuse"):
            loads = [t.timeline for t in log.turns
                     if t.timeline is not None and t.hit_class != "miss"]
            lb = sum(t.bytes_loaded for t in log.turns if t.hit_class != "miss")
            busy = sum(tl.load_total for tl in loads)
            s["h2d_gbs"] = lb / busy / 1e9 if busy else 0.0
            waited = [t for t in log.turns if t.hit_class != "miss"
                      and t.timeline is not None and t.timeline.load_intervals
                      and min(a for a, _ in t.timeline.load_intervals) < 0]
            s["hits_with_head_start"] = len(waited)
            if args.turns_out:
                s["turn_records"] = [
                    {"session": t.session_id, "turn": t.turn_index, "hit": t.hit_class,
                     "prompt": t.prompt_tokens, "new": t.new_tokens, "ttft": t.ttft_s,
                     "prefill": t.prefill_s, "stall": t.stall_s} for t in log.turns]
        out[mode] = s
    eng.runner.close()
    if "recompute" in out:
        r, c = out["reuse"], out["recompute"]
        out["speedup_p50_ttft"] = c["p50_ttft_s"] / r["p50_ttft_s"] if r["p50_ttft_s"] else None
        out["speedup_p50_prefill"] = (c["p50_prefill_s"] / r["p50_prefill_s"]
                                      if r["p50_prefill_s"] else None)
        if "reuse_hbm_tier" in out:
            h = out["reuse_hbm_tier"]
            out["speedup_p50_ttft_hbm_tier"] = (c["p50_ttft_s"] / h["p50_ttft_s"]
                                                if h["p50_ttft_s"] else None)
    return out


def parse(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n\n")[0])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--shard", type=int, default=0)
    ap.add_argument("--of", type=int, default=1, help="session shards (ranks of a node)")
    ap.add_argument("--max-sessions", type=int, default=0)
    ap.add_argument("--load", type=float, default=1.0,
                    help="offered load relative to the reference workload: arrival "
                         "times and think times divided by this factor")
    ap.add_argument("--device", type=int, default=0)
    ap.add_argument("--dram-gb", type=float, default=96.0)
    ap.add_argument("--hbm-gb", type=float, default=0.0,
                    help="also serve with an HBM session tier of this size (0 = off)")
    ap.add_argument("--read-buffer-gb", type=float, default=10.0,
                    help="cap of S_buf (TierConfig.hbm_read_buffer default 10 GB)")
    ap.add_argument("--link-gbs", type=float, default=55.0)
    ap.add_argument("--block-tokens", type=int, default=128)
    ap.add_argument("--batch-size", type=int, default=24)
    ap.add_argument("--prefill-s-per-token", type=float, default=1.92e-4)
    ap.add_argument("--decode-s-per-step", type=float, default=1.0e-3)
    ap.add_argument("--numa-node", type=int, default=-1,
                    help="arena NUMA node (-1: the GPU's own node when the host reports one)")
    ap.add_argument("--autotune", type=int, default=-1,
                    help="GEMM autotune up to this many rows (0 = off, -1 = every "
                         "prompt length the run can see)")
    ap.add_argument("--reuse-only", action="store_true")
    ap.add_argument("--turns-out", action="store_true")
    ap.add_argument("--json", default="")
    return ap.parse_args(argv)


def main(argv=None):
    args = parse(argv)
    res = run(args)
    line = json.dumps(res)
    if args.json:
        Path(args.json).write_text(line + "\n")
    print(line, flush=True)
    os._exit(0)   # skip interpreter teardown of the pinned arena / IO threads


if __name__ == "__main__":
    main()
