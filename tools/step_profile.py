"""Per-kernel breakdown + GPU idle fraction of a bench step (torch.profiler /
CUPTI; nsys is not in the image).  Diagnostics only, never a bench number.

    python tools/step_profile.py [--mode hbm|host|recompute] [--turns 4]
"""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="hbm")
    ap.add_argument("--turns", type=int, default=4)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--bg-h2d", action="store_true",
                    help="stream a background pinned H2D copy during the profiled step")
    ap.add_argument("--no-save", action="store_true", help="jobs without the K4 save")
    ap.add_argument("--no-graph", action="store_true", help="stream-issue the layer loop")
    ap.add_argument("--overlap", action="store_true", help="K2(l+1) alongside K3(l)")
    ap.add_argument("--batch", action="store_true",
                    help="the turns as one batched layer pass (askv_prefill_layers_batch)")
    ap.add_argument("--no-profiler", action="store_true",
                    help="skip torch.profiler (for running under ncu)")
    a = ap.parse_args()
    import bench
    from paper_2403_19708_b200 import model
    from paper_2403_19708_b200.runner import Job, Runner
    from paper_2403_19708_b200.store import HostArena

    shape = model.shape(bench.CONFIGS[a.config][0])
    turns, _ = bench.select_turns(a.config, 0, 1, a.turns)
    tb = 128
    bb = tb * shape.kv_bytes_per_token
    nbs = [-(-(k + n) // tb) for _, _, k, n in turns]
    arena = HostArena(sum(nbs), bb, pin=True)
    hbm = torch.zeros(sum(nbs) * bb // 2, dtype=torch.bfloat16, device="cuda")
    max_new = max(n for *_, n in turns)
    runner = Runner(shape, host_arena=arena, hbm_arena=hbm, read_buffer_bytes=4 << 30,
                    write_buffer_bytes=max(1 << 30, len(turns) * shape.layers * max_new
                                           * shape.row_bytes if a.batch else 0),
                    max_new=max_new,
                    max_ctx=4096, timeline=True, graph=not a.no_graph, overlap=a.overlap)
    jobs, pos = [], 0
    rng = np.random.default_rng(0)
    for (sid, k, kept, new), nb in zip(turns, nbs):
        ids = list(range(pos, pos + nb))
        pos += nb
        toks = torch.as_tensor(rng.integers(0, shape.vocab, new))
        if a.mode == "hbm":
            off = torch.as_tensor([b * bb // 2 for b in ids], dtype=torch.int64, device="cuda")
            jobs.append(Job(f"{sid}#{k}", toks.cuda(), kept=kept, source="hbm", block_ids=ids,
                            save=not a.no_save, dev_block_off=off))
        elif a.mode in ("host", "prestage"):
            jobs.append(Job(f"{sid}#{k}", toks.pin_memory(), kept=kept, source="host",
                            block_ids=ids, save=True, prestage=a.mode == "prestage"))
        else:
            jobs.append(Job(f"{sid}#{k}",
                            torch.as_tensor(rng.integers(0, shape.vocab, kept + new)).cuda()))
    for _ in range(2):
        runner.run(jobs, batch=a.batch)
        runner.join()
    torch.cuda.synchronize()
    if a.no_profiler:   # one more step (the ncu capture window), then stop
        runner.run(jobs, batch=a.batch)
        runner.join()
        torch.cuda.synchronize()
        return
    from torch.profiler import ProfilerActivity, profile
    bg = None
    if a.bg_h2d:   # isolate copy-engine interference: 1 GB H2D chunks on their own stream
        import threading
        src = torch.empty(1 << 30, dtype=torch.uint8).pin_memory()
        dst = torch.empty(1 << 30, dtype=torch.uint8, device="cuda")
        stop = threading.Event()
        bs = torch.cuda.Stream()

        def loop():
            while not stop.is_set():
                with torch.cuda.stream(bs):
                    dst.copy_(src, non_blocking=True)
                bs.synchronize()
        bg = threading.Thread(target=loop, daemon=True)
        bg.start()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    import time
    with profile(activities=[ProfilerActivity.CUDA, ProfilerActivity.CPU]) as prof:
        e0.record(runner.s_compute)
        h0 = time.perf_counter()
        runner.run(jobs, batch=a.batch)
        runner.join()
        host_issue_ms = (time.perf_counter() - h0) * 1e3
        e1.record(runner.s_compute)
        torch.cuda.synchronize()
    # host issue rate without the profiler attached
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    runner.run(jobs, batch=a.batch)
    runner.join()
    host_issue_ms_noprof = (time.perf_counter() - h0) * 1e3
    torch.cuda.synchronize()
    gpu_ms_noprof = (time.perf_counter() - h0) * 1e3
    wall_us = e0.elapsed_time(e1) * 1e3
    res = runner.run(jobs, batch=a.batch)
    runner.join()
    torch.cuda.synchronize()
    Runner.finalize(res)
    if bg is not None:
        stop.set()
        bg.join()
    tls = [{"makespan_ms": r.timeline.makespan * 1e3, "stall_ms": r.timeline.stall_total * 1e3,
            "layer_ms": [round((b - a) * 1e3, 3) for a, b in r.timeline.compute_intervals[:6]]}
           for r in res]
    agg = collections.defaultdict(lambda: [0, 0.0])
    busy = []
    for ev in prof.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA and ev.time_range.elapsed_us() > 0:
            name = ev.name
            for key in ("attn_fwd", "attn_combine", "reembed", "rope_new", "rmsnorm", "silu_mul",
                        "nvjet", "gemm", "Memcpy", "elementwise", "embedding", "argmax",
                        "reduce"):
                if key.lower() in name.lower():
                    name = key
                    break
            agg[name][0] += 1
            agg[name][1] += ev.time_range.elapsed_us()
            busy.append((ev.time_range.start, ev.time_range.end, name))
    # compute-stream kernels only (exclude memcpy) for the idle estimate
    ker = sorted((s, e) for s, e, n in busy if n != "Memcpy")
    merged = 0.0
    cs, ce = None, None
    for s, e in ker:
        if cs is None or s > ce:
            if cs is not None:
                merged += ce - cs
            cs, ce = s, e
        else:
            ce = max(ce, e)
    if cs is not None:
        merged += ce - cs
    cpu_total = sum(ev.cpu_time_total for ev in prof.events()
                    if ev.device_type == torch.autograd.DeviceType.CPU and ev.name == "aten::linear")
    out = {"mode": a.mode, "batch": a.batch, "turns": len(jobs), "wall_us": wall_us,
           "timelines": tls,
           "host_issue_ms": host_issue_ms, "host_issue_ms_noprof": host_issue_ms_noprof,
           "wall_ms_noprof": gpu_ms_noprof,
           "kernel_busy_us": merged, "gpu_idle_frac": 1 - merged / wall_us,
           "kernels": {k: {"n": v[0], "us": round(v[1], 1), "avg_us": round(v[1] / v[0], 2)}
                       for k, v in sorted(agg.items(), key=lambda x: -x[1][1])}}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
