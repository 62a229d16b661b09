"""Batched prefill (scheduler knob, askv_prefill_layers_batch): several
sessions' turns in one pass over the layers -- projections / norms / MLP over
the concatenated new tokens, pre-load wait / K2 / K3 / saves per job.  Every
job's first-token logits match the float64 oracle on that job's own stored
rows, and the saved rows match the job run alone."""

import numpy as np
import pytest
import torch

from oracle import llama_ref, rope_ref

pytestmark = pytest.mark.gpu
TOL = 2e-2


def _setup(bt=16, nb=40, max_new=64):
    from paper_2403_19708_b200 import model, runner
    from paper_2403_19708_b200.store import HostArena
    shape = model.shape("tiny")
    arena = HostArena(nb, bt * shape.kv_bytes_per_token, pin=True)
    hbm = torch.empty(nb * bt * shape.kv_bytes_per_token // 2, dtype=torch.bfloat16,
                      device="cuda")
    g = torch.Generator(device="cuda").manual_seed(3)
    hbm.normal_(generator=g)
    arena.buffer.view(torch.bfloat16).copy_(hbm.cpu())
    r = runner.Runner(shape, seed=4, block_tokens=bt, host_arena=arena, hbm_arena=hbm,
                      read_buffer_bytes=8 << 20, write_buffer_bytes=16 << 20, max_new=max_new,
                      max_ctx=512, autotune=False)
    return shape, r, arena, hbm


MIXES = {
    # host-sourced jobs read V from their own read-buffer slots: one K3 launch per job
    "mixed": [("a", 40, 17, "host", [0, 1, 2, 3]), ("b", 0, 23, "none", [4, 5]),
              ("c", 33, 9, "hbm", [6, 7, 8]), ("d", 64, 31, "host", [9, 10, 11, 12, 13, 14])],
    # HBM-resident / new sessions only: one varlen K3 launch for the batch
    "varlen": [("a", 40, 17, "hbm", [0, 1, 2, 3]), ("b", 0, 23, "none", [4, 5]),
               ("c", 33, 9, "hbm", [6, 7, 8]), ("d", 64, 31, "hbm", [9, 10, 11, 12, 13, 14]),
               ("e", 130, 60, "hbm", list(range(15, 27)))],
    # 128-token blocks: K3 also reads the kept tiles' V straight from the HBM arena
    "varlen_vsrc128": [("a", 200, 17, "hbm", [0, 1]), ("b", 0, 23, "none", [2]),
                       ("c", 256, 9, "hbm", [3, 4, 5]), ("d", 300, 31, "hbm", [6, 7, 8])],
}
# more than one query tile per job: with ASKV_ATTN_PAIR=1 (test below) the
# varlen launch pairs a job's tiles per CTA, odd last tiles running alone
LONG = {"varlen_long": [("a", 40, 300, "hbm", list(range(0, 22))),
                        ("b", 0, 150, "none", list(range(55, 65))),
                        ("c", 130, 257, "hbm", list(range(23, 48))),
                        ("d", 64, 40, "hbm", list(range(48, 55)))]}
# truncated sessions (store.head_row > 0: the session's token 0 sits inside
# its first block) in the batched K2 launch, next to an aligned one
LONG["varlen_head"] = [("a", 40, 17, "hbm", [0, 1, 2, 3], 5), ("b", 0, 23, "none", [4, 5]),
                       ("c", 33, 9, "hbm", [6, 7, 8, 15], 11), ("d", 64, 31, "hbm", [9, 10, 11, 12, 13, 14])]
MIXES.update(LONG)
BT = {"mixed": 16, "varlen": 16, "varlen_vsrc128": 128, "varlen_long": 16, "varlen_head": 16}
SETUP = {"varlen_long": dict(nb=66, max_new=320)}


def _jobs(shape, r, bt, rng, mix):
    from paper_2403_19708_b200.runner import Job
    specs = MIXES[mix]
    jobs = []
    elems = bt * shape.kv_bytes_per_token // 2
    for sid, kept, n, src, bids, *rest in specs:
        ids = torch.as_tensor(rng.integers(0, shape.vocab, n))
        off = torch.as_tensor([b * elems for b in bids], dtype=torch.int64, device="cuda")
        jobs.append(Job(sid, ids, kept=kept, source=src, block_ids=bids, save=True,
                        dev_block_off=off if src == "hbm" else None,
                        head=rest[0] if rest else 0))
    return jobs


def _stored(shape, buf_bf16, bids, bt, rows, head=0):
    """Pre-RoPE K/V rows [0, rows) of a block list (session token 0 at row
    `head` of the first block), per layer, float64."""
    L, rb = shape.layers, shape.row_elems
    blk = bt * rb * L
    out = []
    for layer in range(L):
        rws = []
        for t in range(head, head + rows):
            b = bids[t // bt]
            base = b * blk + layer * bt * rb + (t % bt) * rb
            rws.append(buf_bf16[base:base + rb])
        kv = torch.stack(rws).float().cpu().numpy().astype(np.float64)
        kv = kv.reshape(rows, 2, shape.n_kv_heads, shape.head_dim)
        out.append((kv[:, 0], kv[:, 1]))
    return out


@pytest.mark.parametrize("mix", sorted(MIXES))
def test_batched_prefill_matches_oracle_and_single_runs(mix):
    from paper_2403_19708_b200.runner import Runner
    bt = BT[mix]
    shape, r, arena, hbm = _setup(bt, **SETUP.get(mix, {}))
    wnp = r.w.to_numpy()
    rng = np.random.default_rng(5)
    jobs = _jobs(shape, r, bt, rng, mix)
    # oracle inputs: each job's stored rows before the run
    caches = {}
    for j in jobs:
        if j.kept:
            src = hbm if j.source == "hbm" else arena.buffer.view(torch.bfloat16)
            caches[j.session_id] = _stored(shape, src, j.block_ids, bt, j.kept, j.head)
    res = r.run(jobs, want_logits=True, batch=True)
    r.join()
    torch.cuda.synchronize()
    Runner.finalize(res)
    batched_saved = {j.session_id: _stored(shape, hbm if j.source == "hbm" else
                                           arena.buffer.view(torch.bfloat16),
                                           j.block_ids, bt, j.kept + j.n_new, j.head)
                     for j in jobs}
    for j, o in zip(jobs, res):
        empty = [(np.zeros((0, shape.n_kv_heads, shape.head_dim)),) * 2] * shape.layers
        cache = caches.get(j.session_id, empty)
        want, _ = llama_ref.forward(wnp, j.token_ids.numpy(), cache, np.arange(j.kept),
                                    n_heads=shape.n_heads, n_kv_heads=shape.n_kv_heads,
                                    head_dim=shape.head_dim)
        got = o.logits.cpu().double().numpy()
        assert rope_ref.rel_err(got, want[-1]) <= TOL, j.session_id
        assert o.timeline is not None and o.timeline.makespan > 0
    # the same jobs one at a time write the same new rows (the batched GEMMs
    # may round differently: within one bf16 ulp)
    for j in jobs:
        single = r.run([j], want_logits=True)
        r.join()
        torch.cuda.synchronize()
        Runner.finalize(single)
        got = _stored(shape, hbm if j.source == "hbm" else arena.buffer.view(torch.bfloat16),
                      j.block_ids, bt, j.kept + j.n_new, j.head)
        for layer in range(shape.layers):
            for a, b in zip(got[layer], batched_saved[j.session_id][layer]):
                assert np.allclose(a, b, rtol=1e-2, atol=1e-2), (j.session_id, layer)


def test_batched_prefill_paired_varlen():
    """The long mix with paired query tiles forced on (csrc/attention.cu
    use_pairs, read once per process: run in a subprocess)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "from test_batch_gpu import *;"
            "test_batched_prefill_matches_oracle_and_single_runs('varlen_long')")
    r = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                       env=dict(os.environ, ASKV_ATTN_PAIR="1"))
    assert r.returncode == 0, r.stderr[-3000:]
