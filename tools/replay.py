"""Measured-mode replay of a reference workload.

Every turn of a committed reference workload (tests/golden/workload_<cfg>.json,
the sessions of trace.generate_poisson) goes through the real B200 engine in
arrival order: overflow truncation, store lookup, layer-wise pre-load from the
pinned host arena, re-embed, tcgen05 attention, async save, teacher-forced
append of the output tokens, save-time truncation (engine.Engine.turn, the
sim._start_job/_finish_job semantics).  Each prefill's makespan is measured
with CUDA events; queue-inclusive TTFT follows a FIFO single-prefill-stream
server fed at the workload's arrival times (sim.py:212-222, 485-489), using the
measured makespans as service times.  The same turns are replayed in
recompute mode (sim Mode.RECOMPUTE: no store, the whole prompt is prefilled).

    python tools/replay.py --config c2 [--sessions 64]
"""
import argparse
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def fifo_ttft(arrivals, service):
    """Queue-inclusive TTFT of a serial prefill server (completion - arrival)."""
    order = np.argsort(arrivals, kind="stable")
    free = 0.0
    out = np.empty(len(arrivals))
    for i in order:
        start = max(free, arrivals[i])
        free = start + service[i]
        out[i] = free - arrivals[i]
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--sessions", type=int, default=0)
    ap.add_argument("--host-gb", type=float, default=120.0)
    ap.add_argument("--hbm-gb", type=float, default=0.0,
                    help="HBM session tier capacity (SURVEY.md §8f item 1); 0 = DRAM only")
    ap.add_argument("--disk-gb", type=float, default=0.0,
                    help="disk tier capacity (SURVEY.md §8f item 4); 0 = no disk tier")
    ap.add_argument("--disk-dir", default="/tmp/askv-replay-disk")
    ap.add_argument("--prefetch", type=int, default=0,
                    help="scheduler-aware prefetch window: disk->DRAM reads for the "
                         "sessions of the next N turns (policy.py:122-150)")
    ap.add_argument("--out", default="")
    a = ap.parse_args()
    from paper_2403_19708_b200 import engine, metrics, model
    from paper_2403_19708_b200.runner import Job, LlamaWeights, Runner

    wl = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                     f"workload_{a.config}.json")))
    shape = model.shape({"c1": "tiny", "c2": "7b", "c3": "13b"}[a.config])
    sessions = wl["sessions"][: a.sessions or None]
    tb = 128 if shape.layers > 2 else 16
    block_bytes = tb * shape.kv_bytes_per_token
    host_blocks = int(a.host_gb * 1e9 // block_bytes)
    weights = LlamaWeights(shape, seed=0)
    eng = engine.Engine(shape, host_blocks=host_blocks, block_tokens=tb, weights=weights,
                        max_new=2048, read_buffer_bytes=4 << 30,
                        hbm_blocks=int(a.hbm_gb * 1e9 // block_bytes),
                        disk_dir=a.disk_dir if a.disk_gb else None,
                        disk_blocks=int(a.disk_gb * 1e9 // block_bytes))
    turns = sorted(((s["arrivals"][k], s["id"], k, s["turns"][k][0], s["turns"][k][1])
                    for s in sessions for k in range(len(s["turns"]))))
    rng = np.random.default_rng(0)
    recs = []
    t_wall = time.time()
    for i, (arr, sid, k, new, out) in enumerate(turns):
        ids = torch.as_tensor(rng.integers(0, shape.vocab, new)).pin_memory()
        oids = torch.as_tensor(rng.integers(0, shape.vocab, out)) if out else None
        if a.prefetch and eng.store.disk is not None:
            ahead = [t[1] for t in turns[i + 1:i + 1 + a.prefetch] if t[1] != sid]
            eng.store.pinned.add(sid)
            eng.prefetch(ahead)
            eng.store.pinned.discard(sid)
        o = eng.turn(sid, k, ids, oids, now=arr)
        torch.cuda.synchronize()
        eng.runner.finalize(o.results)
        # a disk hit's read (or the unfinished part of its prefetch) precedes the
        # layer-wise pre-load: it is part of the prefill service time
        recs.append(dict(arrival=arr, session=sid, turn=k, hit=o.hit, kept=o.kept, new=new,
                         prompt=o.prompt, makespan=o.ttft_s() + eng.last_disk_wait_s,
                         disk_wait=eng.last_disk_wait_s,
                         stall=sum(r.timeline.stall_total for r in o.results)))
    reuse_wall = time.time() - t_wall
    # recompute mode: the same prompts, whole prompt prefilled, no store
    rec_runner = Runner(shape, weights=weights, block_tokens=tb, max_new=2048,
                        max_ctx=shape.context_window + 2048)
    for r in recs:
        # the (truncated) prompt the reference would recompute; prompts beyond the
        # window are capped at W (the engine's rolling window keeps <= W rows)
        n = min(r["prompt"], shape.context_window)
        ids = torch.as_tensor(rng.integers(0, shape.vocab, n))
        res = rec_runner.run([Job(r["session"], ids.cuda())])[0]
        torch.cuda.synchronize()
        Runner.finalize([res])
        r["recompute_makespan"] = res.timeline.makespan
    arr = np.array([r["arrival"] for r in recs])
    ms_re = np.array([r["makespan"] for r in recs])
    ms_rc = np.array([r["recompute_makespan"] for r in recs])
    tt_re, tt_rc = fifo_ttft(arr, ms_re), fifo_ttft(arr, ms_rc)
    prompt = [r["prompt"] for r in recs]
    elig = [r for r in recs if r["turn"] > 0]
    hits = [r for r in elig if r["hit"] != "miss"]
    hit_ms = np.array([r["makespan"] for r in hits])
    hit_rc = np.array([r["recompute_makespan"] for r in hits])
    out = {
        "config": a.config, "shape": shape.name, "sessions": len(sessions), "turns": len(recs),
        "hit_rate": len(hits) / max(1, len(elig)),
        "reuse": {"p50_ttft_s": metrics.percentile(tt_re, 0.5),
                  "p99_ttft_s": metrics.percentile(tt_re, 0.99),
                  "prefill_tok_s": metrics.prefill_throughput(prompt, ms_re),
                  "exposed_transfer_frac": float(sum(r["stall"] for r in recs) / ms_re.sum())},
        "recompute": {"p50_ttft_s": metrics.percentile(tt_rc, 0.5),
                      "p99_ttft_s": metrics.percentile(tt_rc, 0.99),
                      "prefill_tok_s": metrics.prefill_throughput(prompt, ms_rc)},
        "hit_turns_p50_makespan_s": {"reuse": metrics.percentile(hit_ms, 0.5),
                                     "recompute": metrics.percentile(hit_rc, 0.5)},
        "store": {"mem_used": eng.store.mem_used, "items": len(eng.store.items),
                  "arena_blocks": host_blocks},
        "hbm_tier": ({"gb": a.hbm_gb, "hits": eng.hbm.hits, "promotions": eng.hbm.promotions}
                     if eng.hbm else None),
        "disk_tier": ({"gb": a.disk_gb, "prefetch_window": a.prefetch,
                       "disk_hits": sum(r["hit"] == "disk_hit" for r in recs),
                       "evictions_to_disk": eng.disk_evictions,
                       "promotions": eng.disk_promotions,
                       "read_gb": eng.store.disk.bytes_read / 1e9,
                       "write_gb": eng.store.disk.bytes_written / 1e9,
                       "exposed_disk_wait_s": float(sum(r["disk_wait"] for r in recs))}
                      if eng.store.disk else None),
        "wall_s_reuse_replay": reuse_wall,
        "note": "TTFT = FIFO serial-prefill queue on measured makespans at the workload's "
                "arrival times (no read-buffer head start: the load starts with the job)",
    }
    out["ttft_reduction_p50"] = 1 - out["reuse"]["p50_ttft_s"] / out["recompute"]["p50_ttft_s"]
    out["prefill_speedup"] = out["reuse"]["prefill_tok_s"] / out["recompute"]["prefill_tok_s"]
    js = json.dumps(out, indent=1)
    print(js)
    if a.out:
        open(a.out, "w").write(js)


if __name__ == "__main__":
    main()
