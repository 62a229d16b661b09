"""Host cost of a batched layer pass (16 C3 turns, HBM-resident KV): Python
plan building vs the native issue path (capture / graph update / launch,
askv_issue_stats) against the GPU time.  Diagnostics only.

    python tools/host_batch.py [--turns 16] [--no-batch]
"""
import argparse
import cProfile
import ctypes as C
import io
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--turns", type=int, default=16)
    ap.add_argument("--no-batch", action="store_true")
    a = ap.parse_args()
    import bench
    from paper_2403_19708_b200 import _lib, model
    from paper_2403_19708_b200.runner import Job, Runner
    shape = model.shape("13b")
    turns, _ = bench.select_turns("c3", 0, 1, a.turns)
    tb = 128
    bb = tb * shape.kv_bytes_per_token
    nbs = [-(-(k + n) // tb) for _, _, k, n in turns]
    hbm = torch.zeros(sum(nbs) * bb // 2, dtype=torch.bfloat16, device="cuda")
    max_new = max(n for *_, n in turns)
    runner = Runner(shape, hbm_arena=hbm, read_buffer_bytes=1 << 30,
                    write_buffer_bytes=len(turns) * shape.layers * max_new * shape.row_bytes,
                    max_new=max_new, max_ctx=4096)
    jobs, pos = [], 0
    rng = np.random.default_rng(0)
    for (sid, k, kept, new), nb in zip(turns, nbs):
        ids = list(range(pos, pos + nb))
        pos += nb
        off = torch.as_tensor([b * bb // 2 for b in ids], dtype=torch.int64, device="cuda")
        jobs.append(Job(f"{sid}#{k}", torch.as_tensor(rng.integers(0, shape.vocab, new)).cuda(),
                        kept=kept, source="hbm", block_ids=ids, save=True, dev_block_off=off))
    batch = not a.no_batch
    for _ in range(3):
        runner.run(jobs, batch=batch)
        runner.join()
    torch.cuda.synchronize()
    st0 = (C.c_double * 4)()
    st1 = (C.c_double * 4)()
    lib = _lib.lib()
    reps = 5
    lib.askv_issue_stats(st0)
    prof = cProfile.Profile()
    t0 = time.perf_counter()
    prof.enable()
    for _ in range(reps):
        runner.run(jobs, batch=batch)
        runner.join()
    prof.disable()
    host = (time.perf_counter() - t0) / reps
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / reps
    lib.askv_issue_stats(st1)
    d = [(st1[i] - st0[i]) / reps for i in range(4)]
    print(f"batch={batch} turns={len(jobs)} host issue {host * 1e3:.1f} ms/step, wall "
          f"{wall * 1e3:.1f} ms/step; native: {d[0]:.0f} calls, capture {d[1] / 1e3:.1f} ms, "
          f"update {d[2] / 1e3:.1f} ms, launch {d[3] / 1e3:.1f} ms")
    s = io.StringIO()
    pstats.Stats(prof, stream=s).sort_stats("tottime").print_stats(18)
    print(s.getvalue())


if __name__ == "__main__":
    main()
