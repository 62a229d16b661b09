"""World-size-2 gloo test of the multi-GPU host plumbing on CPU: disjoint and
complete session shards, bench turn selection per shard, max/sum-over-ranks."""

import json
import os
import socket
from pathlib import Path

import pytest
import torch.multiprocessing as mp

ROOT = Path(__file__).resolve().parent.parent


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank),
                      WORLD_SIZE=str(world), LOCAL_RANK=str(rank))
    import sys
    sys.path.insert(0, str(ROOT))
    import torch.distributed as dist

    from paper_2403_19708_b200 import dist as pdist
    import bench

    pdist.init("gloo")
    wl = json.loads((ROOT / "tests" / "golden" / "workload_c3.json").read_text())
    ids = [s["id"] for s in wl["sessions"]]
    mine = pdist.shard(ids, rank, world)
    turns, n_hits = bench.select_turns("c3", rank, world, 16)
    got = [None] * world
    dist.all_gather_object(got, {"mine": mine, "turns": [t[0] for t in turns],
                                 "n_hits": n_hits})
    mx = pdist.max_over_ranks(10.0 + rank)
    sm = pdist.sum_over_ranks(1.0 + rank)
    if rank == 0:
        (Path(out_dir) / "res.json").write_text(json.dumps(
            {"gathered": got, "max": mx, "sum": sm, "all": ids}))
    dist.destroy_process_group()


def test_two_rank_gloo_sharding(tmp_path):
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    res = json.loads((tmp_path / "res.json").read_text())
    a, b = (set(g["mine"]) for g in res["gathered"])
    assert not (a & b) and (a | b) == set(res["all"])
    assert 150 < len(a) < 360 and 150 < len(b) < 360       # roughly balanced hash
    for r, g in enumerate(res["gathered"]):
        assert len(g["turns"]) == 16
        assert all((sid in (a if r == 0 else b)) for sid in g["turns"])
    assert res["max"] == 11.0 and res["sum"] == 3.0
    assert res["gathered"][0]["n_hits"] + res["gathered"][1]["n_hits"] == 2373
