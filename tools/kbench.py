"""Kernel micro-benchmarks (CUDA events, warm-up, L2 flushed between reps).

    python tools/kbench.py attn [--kernel 1|2]
    python tools/kbench.py reembed
"""
import argparse
import json
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402


def timeit(fn, reps=20, flush=True, batch=1):
    buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush:
            buf.zero_()
        else:  # keep the queue busy so e0 does not time the host launch latency
            torch.cuda._sleep(200000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(batch):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e-3 / batch)
    ts.sort()
    return ts[len(ts) // 2]


def attn(args):
    from paper_2403_19708_b200 import ops
    from paper_2403_19708_b200.runner import attention_flops
    shapes = [(2142, 237, 40, 40), (2869, 301, 40, 40), (2048, 256, 32, 32), (1000, 100, 40, 40),
              (3600, 700, 40, 40), (0, 2379, 40, 40), (2048, 256, 8, 1)]
    if args.shape:
        shapes = [tuple(int(x) for x in args.shape.split(","))]
    out = []
    for kept, n, hq, hkv in shapes:
        d = 128
        q = torch.randn(n, hq, d, device="cuda").to(torch.bfloat16)
        kv = torch.randn(kept + n, 2, hkv, d, device="cuda").to(torch.bfloat16)
        o = torch.empty(n, hq, d, device="cuda", dtype=torch.bfloat16)
        s = args.splits or ops.attn_num_splits(kept, n, hq, n_kv_heads=hkv)
        ws = torch.empty(max(1, ops.attn_workspace_bytes(kept, n, hq, d, s)), dtype=torch.uint8,
                         device="cuda")
        t = timeit(lambda: ops.prefill_attn(q, kv, kept, n, hq, hkv, d, o, ws, num_splits=s),
                   reps=args.reps, flush=not args.warm, batch=args.batch)
        fl = attention_flops(kept, n, hq, d)
        row = dict(kept=kept, n=n, hq=hq, hkv=hkv, splits=s, us=t * 1e6, tflops=fl / t / 1e12,
                   l2="warm" if args.warm else "flushed")
        out.append(row)
        print(json.dumps(row))
    return out


def reembed(args):
    from paper_2403_19708_b200 import ops
    for kept, hkv in [(2869, 40), (2142, 40), (4000, 32), (2048, 1)]:
        d = 128
        src = torch.randn(kept, 2, hkv, d, device="cuda").to(torch.bfloat16)
        dst = torch.empty_like(src)
        table = ops.rope_table(8192, d)
        t = timeit(lambda: ops.reembed(src, kept, hkv, d, table, dst))
        by = 2 * src.numel() * 2
        print(json.dumps(dict(kept=kept, hkv=hkv, us=t * 1e6, gbs=by / t / 1e9)))


def sweep(args):
    """Time every split count for a few shapes (tunes choose_splits)."""
    from paper_2403_19708_b200 import ops
    from paper_2403_19708_b200.runner import attention_flops
    shapes = [(2142, 237, 40, 40), (2869, 301, 40, 40), (1000, 100, 40, 40), (3600, 700, 40, 40),
              (2048, 256, 8, 1), (500, 60, 40, 40), (3800, 120, 40, 40), (2000, 400, 32, 32)]
    for kept, n, hq, hkv in shapes:
        d = 128
        q = torch.randn(n, hq, d, device="cuda").to(torch.bfloat16)
        kv = torch.randn(kept + n, 2, hkv, d, device="cuda").to(torch.bfloat16)
        o = torch.empty(n, hq, d, device="cuda", dtype=torch.bfloat16)
        auto = ops.attn_num_splits(kept, n, hq)
        res = {}
        for s in (1, 2, 3, 4, 5, 6, 8, 10, 12, 16):
            if s > (kept + n + 127) // 128:
                continue
            ws = torch.empty(max(1, ops.attn_workspace_bytes(kept, n, hq, d, s)),
                             dtype=torch.uint8, device="cuda")
            t = timeit(lambda: ops.prefill_attn(q, kv, kept, n, hq, hkv, d, o, ws, num_splits=s),
                       reps=10)
            res[s] = round(t * 1e6, 1)
        best = min(res, key=res.get)
        print(json.dumps(dict(kept=kept, n=n, hq=hq, hkv=hkv, auto=auto, best=best, us=res,
                              best_tflops=attention_flops(kept, n, hq, d) / res[best] / 1e6)))


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("what")
    ap.add_argument("--kernel", default="2")
    ap.add_argument("--splits", type=int, default=0)
    ap.add_argument("--shape", default="", help="kept,n,hq,hkv")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--warm", action="store_true", help="no L2 flush between reps")
    ap.add_argument("--batch", type=int, default=1, help="launches per timed rep (averaged)")
    a = ap.parse_args()
    os.environ["ASKV_ATTN_KERNEL"] = a.kernel
    {"attn": attn, "reembed": reembed, "sweep": sweep}[a.what](a)
