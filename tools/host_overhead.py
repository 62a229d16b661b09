"""Host issue cost of one reuse job (graph capture + update / instantiate +
launch) against its GPU makespan, 13B shapes.  Diagnostics only.

    python tools/host_overhead.py [--graph 0|1]
"""
import argparse
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import numpy as np  # noqa: E402
import torch  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--graph", type=int, default=1)
    ap.add_argument("--kept", type=int, default=2869)
    ap.add_argument("--new", type=int, default=301)
    a = ap.parse_args()
    from paper_2403_19708_b200 import model
    from paper_2403_19708_b200.runner import Job, Runner
    shape = model.shape("llama2-13b")
    tb = 128
    bb = tb * shape.kv_bytes_per_token
    nb = -(-(a.kept + a.new) // tb)
    hbm = torch.zeros(nb * bb // 2, dtype=torch.bfloat16, device="cuda")
    runner = Runner(shape, hbm_arena=hbm, read_buffer_bytes=1 << 30, write_buffer_bytes=1 << 30,
                    max_new=1024, max_ctx=4096, graph=bool(a.graph))
    off = torch.as_tensor([b * bb // 2 for b in range(nb)], dtype=torch.int64, device="cuda")
    rng = np.random.default_rng(0)
    out = {}
    for label, new in (("same shape", a.new), ("new shape each call", None)):
        host, wall, span = [], [], []
        for i in range(8):
            n = new if new is not None else a.new - 8 + i   # distinct n -> graph cache miss
            ids = torch.as_tensor(rng.integers(0, shape.vocab, n)).cuda()
            job = Job(f"s{i}", ids, kept=a.kept, source="hbm", block_ids=list(range(nb)),
                      save=False, dev_block_off=off)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            res = runner.run([job])
            t1 = time.perf_counter()
            res[0].first_token.numpy()   # host-visible first token (the copy was async)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            Runner.finalize(res)
            host.append((t1 - t0) * 1e3)
            wall.append((t2 - t0) * 1e3)
            span.append(res[0].timeline.makespan * 1e3)
        out[label] = {"host_issue_ms": np.median(host[2:]), "wall_to_first_token_ms":
                      np.median(wall[2:]), "gpu_makespan_ms": np.median(span[2:])}
    print({"graph": a.graph, **out})


if __name__ == "__main__":
    main()
