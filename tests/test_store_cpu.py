"""KvStore mirror (paper_2403_19708_b200.store) against the reference's golden
dump_state sequence, plus block-table invariants of the physical arena, plus
the closed-form truncation arithmetic against the oracle and golden grid."""

import json
from pathlib import Path

import numpy as np
import pytest
from hypothesis import given, settings, strategies as st

from oracle import layout_ref
from paper_2403_19708_b200 import model
from paper_2403_19708_b200.engine import overflow_kept, save_truncate
from paper_2403_19708_b200.store import (HitClass, HostArena, ItemNotFoundError, KvStore,
                                         StoreSizeError, Tier)

G = Path(__file__).resolve().parent / "golden"


def _profile(kvb, layers=2):
    return model.ModelProfile(name="p", kv_bytes_per_token=float(kvb),
                              prefill_seconds_per_token=1e-4, decode_seconds_per_step=1e-3,
                              context_window=4096, layers=layers)


@pytest.mark.parametrize("physical", [False, True])
def test_store_matches_reference_dump_sequence(physical):
    for case in json.loads((G / "store.json").read_text()):
        prof = _profile(case["kv_bytes_per_token"])
        tiers = model.TierConfig(dram_capacity=10**15, disk_capacity=10**15)
        kw = {}
        if physical:
            if case["block_tokens"] > 64:   # keep the CPU arena small
                continue
            kw = dict(arena=HostArena(1200, case["block_bytes"], pin=False),
                      block_tokens=case["block_tokens"])
        stor = KvStore(prof, tiers, block_bytes=case["block_bytes"], **kw)
        for (op, sid, tok, now), want in zip(case["ops"], case["dumps"]):
            if op == "save":
                if physical:
                    stor.reserve_rows(sid, tok)
                    stor.mark_written(sid, tok)
                stor.save(sid, tok, now)
            elif op == "truncate":
                stor.truncate_item(sid, tok, now)
            else:
                stor.remove(sid)
            stor.check_invariants()
            assert json.loads(stor.dump_state()) == want


def test_block_table_truncation_drops_front_blocks():
    tb = 16
    prof = model.ModelProfile(name="p", kv_bytes_per_token=1024.0, prefill_seconds_per_token=1e-4,
                              decode_seconds_per_step=1e-3, context_window=64, layers=2)
    arena = HostArena(64, tb * 1024, pin=False)
    stor = KvStore(prof, model.TierConfig(dram_capacity=64 * tb * 1024, disk_capacity=0),
                   block_bytes=tb * 1024, arena=arena, block_tokens=tb)
    tab = stor.reserve_rows("s", 60)
    stor.mark_written("s", 60)
    stor.save("s", 60, 0.0)
    assert len(tab) == 4
    # load-time truncation: W=64, cut=32; hist 60 + new 10 -> kept 28 (drops 32 = 2 blocks)
    kept = overflow_kept(60, 10, 64, 32)
    assert kept == 28
    stor.truncate_item("s", kept, 1.0)
    assert stor.block_table("s") == tab[2:]
    stor.check_invariants()
    # the next save appends in place
    tab2 = stor.reserve_rows("s", kept + 10)
    assert tab2[:2] == tab[2:]
    stor.mark_written("s", kept + 10)
    stor.save("s", kept + 10, 2.0)
    stor.check_invariants()
    stor.remove("s")
    assert arena.free_blocks == 64
    with pytest.raises(ItemNotFoundError):
        stor.remove("s")


def test_physical_store_rejects_misaligned_blocks():
    prof = _profile(100)
    with pytest.raises(ValueError):
        KvStore(prof, model.TierConfig(), block_bytes=3000 * 100,
                arena=HostArena(1, 3000 * 100, pin=False), block_tokens=3000)


def test_store_errors_and_ttl():
    prof = _profile(1000)
    stor = KvStore(prof, model.TierConfig(dram_capacity=10**9, disk_capacity=10**9),
                   block_bytes=10**6, ttl=10.0)
    with pytest.raises(ValueError):
        stor.save("a", 0, 0.0)
    with pytest.raises(StoreSizeError):
        stor.save("a", 10**7, 0.0)
    stor.save("a", 100, 0.0)
    assert stor.lookup("a", 5.0) is HitClass.MEMORY_HIT
    assert stor.lookup("a", 16.0) is HitClass.MISS       # expired and removed
    assert stor.peek("a") is None
    stor.save("b", 100, 0.0)
    assert stor.move("b", Tier.DISK) == 100 * 1000
    assert stor.lookup("b", 1.0) is HitClass.DISK_HIT


@settings(max_examples=300, deadline=None)
@given(hist=st.integers(0, 40000), new=st.integers(1, 9000),
       w=st.sampled_from([64, 100, 2048, 4096]), ratio=st.sampled_from([0.25, 0.5, 0.75]))
def test_closed_form_truncation_equals_reference_loops(hist, new, w, ratio):
    cut = max(1, int(ratio * w))
    assert overflow_kept(hist, new, w, cut) == layout_ref.overflow_kept(hist, new, w, ratio)
    assert save_truncate(hist + new, w, cut) == layout_ref.save_truncate(hist + new, w, ratio)


def test_closed_form_truncation_golden_grid():
    for r in json.loads((G / "truncation.json").read_text()):
        cut = max(1, int(r["ratio"] * r["W"]))
        if "kept" in r:
            assert overflow_kept(r["hist"], r["new"], r["W"], cut) == r["kept"]
        else:
            assert save_truncate(r["save_tokens"], r["W"], cut) == r["saved"]


def test_block_counts_equal_reference_charge():
    """charge(tokens * kvb) / block_bytes == ceil(tokens / T_b) for the LLaMA shapes."""
    for name, tb in (("llama2-13b", 128), ("llama2-7b", 256), ("llama2-70b", 128)):
        s = model.shape(name)
        bb = tb * s.kv_bytes_per_token
        for tok in (1, tb - 1, tb, tb + 1, 2142, 4096):
            ch = layout_ref.charge(layout_ref.kv_size(tok, s.kv_bytes_per_token), bb)
            assert ch // bb == -(-tok // tb)


def test_shapes_kv_bytes():
    assert model.shape("13b").kv_bytes_per_token == 819200
    assert model.shape("7b").kv_bytes_per_token == 524288
    assert model.shape("70b").kv_bytes_per_token == 327680
    assert model.shape("70b").tp_shard(8).kv_bytes_per_token == 40960


@settings(max_examples=400, deadline=None)
@given(kept=st.integers(0, 4096), sizes=st.lists(st.integers(1, 2048), min_size=1, max_size=12),
       w=st.sampled_from([4096, 2048]))
def test_rolling_window_chunks_equal_save_truncation(kept, sizes, w):
    """Chunked prefill/append with a rolling window (chunks <= cut) ends at the
    reference's save-time truncation of the whole turn (sim.py:576-581)."""
    from paper_2403_19708_b200.engine import rolling_kept
    cut = w // 2
    sizes = [min(c, cut) for c in sizes]
    kept = min(kept, w)
    assert rolling_kept(kept, sizes, w, cut) == layout_ref.save_truncate(kept + sum(sizes), w,
                                                                          0.5)


@pytest.mark.parametrize("ratio", [0.1, 0.25, 0.5, 0.75, 0.9])
@pytest.mark.parametrize("w", [64, 100, 4096])
def test_rolling_window_engine_chunk_any_ratio(ratio, w):
    """The engine's chunk bound min(max_new, cut, W - cut) keeps the rolling
    window equal to the reference's save-time truncation (sim.py:576-581) for
    every truncation ratio, not only 0.5 (ratio 0.75 with chunks
    > W - cut overflowed).  Exhaustive over kept / turn length on a grid."""
    from paper_2403_19708_b200.engine import rolling_kept
    cut = max(1, int(ratio * w))
    chunk = max(1, min(2048, cut, w - cut))
    for kept in range(0, w + 1, max(1, w // 32)):
        for total in range(1, 3 * w, max(1, w // 40)):
            sizes = [chunk] * (total // chunk) + ([total % chunk] if total % chunk else [])
            assert rolling_kept(kept, sizes, w, cut) == \
                layout_ref.save_truncate(kept + total, w, ratio), (kept, total)
    # the bound is what makes it hold: ratio 0.75 with a chunk of W/2 breaks it
    if ratio == 0.75 and w == 4096:
        assert rolling_kept(2000, [3072], w, cut) != \
            layout_ref.save_truncate(2000 + 3072, w, ratio)


def _disk_store(tmp_path, blocks=16, tb=16, kvb=1024, disk_blocks=64):
    from paper_2403_19708_b200.disk import DiskTier
    prof = model.ModelProfile(name="p", kv_bytes_per_token=float(kvb),
                              prefill_seconds_per_token=1e-4, decode_seconds_per_step=1e-3,
                              context_window=4096, layers=2)
    bb = tb * kvb
    arena = HostArena(blocks, bb, pin=False)
    disk = DiskTier(str(tmp_path / "kv"), bb, io_threads=4, chunk_bytes=4096)
    stor = KvStore(prof, model.TierConfig(dram_capacity=blocks * bb, disk_capacity=disk_blocks * bb),
                   block_bytes=bb, arena=arena, block_tokens=tb, disk=disk)
    return stor, arena, disk


def _fill(stor, arena, sid, rows, seed):
    tab = stor.reserve_rows(sid, rows)
    stor.mark_written(sid, rows)
    buf = arena.buffer.numpy()
    rng = np.random.default_rng(seed)
    for b in tab:
        buf[b * arena.block_bytes:(b + 1) * arena.block_bytes] = rng.integers(
            0, 256, arena.block_bytes, dtype=np.uint8)
    return [bytes(buf[b * arena.block_bytes:(b + 1) * arena.block_bytes]) for b in tab]


def test_disk_tier_round_trip_is_bit_exact(tmp_path):
    """move(sid, DISK) writes the session's blocks to its file and frees them
    from the arena; move(sid, MEMORY) reads them back into fresh blocks, bytes
    identical.  Accounting stays the reference's."""
    stor, arena, disk = _disk_store(tmp_path)
    want = _fill(stor, arena, "a", 70, 0)            # 5 blocks of 16 rows
    stor.save("a", 70, 0.0)
    free0 = arena.free_blocks
    moved = stor.move("a", Tier.DISK)
    assert moved == stor.peek("a").bytes and stor.peek("a").tier is Tier.DISK
    assert arena.free_blocks == free0 + 5 and stor.block_table("a") == []
    assert (tmp_path / "kv").exists() and disk.bytes_written == 5 * arena.block_bytes
    stor.check_invariants()
    assert stor.lookup("a", 1.0) is HitClass.DISK_HIT
    _fill(stor, arena, "b", 64, 1)                    # reuse the freed blocks meanwhile
    stor.save("b", 64, 1.0)
    stor.move("a", Tier.MEMORY, wait=False)           # async prefetch
    stor.wait("a")
    buf = arena.buffer.numpy()
    got = [bytes(buf[b * arena.block_bytes:(b + 1) * arena.block_bytes])
           for b in stor.block_table("a")]
    assert got == want and not stor.on_disk("a")
    stor.check_invariants()


def test_disk_tier_truncation_and_remove(tmp_path):
    """Truncating an item while it sits on disk is a file front-offset edit;
    after promotion the table holds exactly the kept suffix's blocks."""
    stor, arena, disk = _disk_store(tmp_path)
    want = _fill(stor, arena, "t", 80, 2)             # 5 blocks
    stor.save("t", 80, 0.0)
    stor.move("t", Tier.DISK)
    stor.truncate_item("t", 40, 1.0)                  # drop 40 rows = 2 whole blocks + 8
    assert disk.meta["t"].nblocks == 3 and disk.meta["t"].head == 8
    stor.check_invariants()
    stor.move("t", Tier.MEMORY)
    buf = arena.buffer.numpy()
    got = [bytes(buf[b * arena.block_bytes:(b + 1) * arena.block_bytes])
           for b in stor.block_table("t")]
    assert got == want[2:] and stor.head_row("t") == 8
    stor.move("t", Tier.DISK)
    path = disk.path("t")
    stor.remove("t")
    assert not Path(path).exists() and "t" not in disk.meta
    stor.check_invariants()


def test_hbm_tier_block_reuse_is_fenced():
    """HBM session tier bookkeeping (engine.HbmTier, host-side only): a block
    that moves from one session to another records the previous owner, so the
    new owner's next job orders its tier writes after that session's saves; a
    session re-taking its own freed blocks needs no fence; the mirror tracks
    the host table's front drops and growth one-to-one."""
    from paper_2403_19708_b200.engine import HbmTier
    tier = HbmTier(4, 64, "cpu")
    assert tier.sync("a", [10, 11], 0, set()) and tier.tab["a"] == [0, 1]
    assert tier.sync("b", [20, 21], 0, set()) and tier.tab["b"] == [2, 3]
    assert tier.fence == {}
    # c needs a block: the LRU session (a) is evicted, its blocks go to c
    assert tier.sync("c", [30], 0, set()) and tier.tab["c"] == [0]
    assert "a" not in tier.tab and tier.fence == {"c": {"a"}}
    # front drop of b's first block, then growth: b takes back its own block
    # first (no fence) and a's remaining one (fenced on a)
    assert tier.sync("b", [21, 22, 23], 1, set())
    assert tier.tab["b"] == [3, 1, 2] and tier.fence["b"] == {"a"}
    # pinned sessions are never evicted; with nothing evictable the sync fails
    # and the session is dropped from the tier
    assert not tier.sync("d", [40, 41], 0, {"b", "c"})
    assert "d" not in tier.tab


def test_arena_allocator_runs_and_no_double_allocation():
    """HostArena hands out contiguous runs (a session's growth continues its
    last block when free) and never gives out a block twice."""
    import random

    from paper_2403_19708_b200.store import CapacityError, HostArena
    a = HostArena(64, 8, pin=False)
    x = a.alloc(10)
    assert x == list(range(10))
    y = a.alloc(4, after=x[-1])
    assert y == list(range(10, 14))
    a.release(x[:5])
    z = a.alloc(6)              # the freed 5-run is too short: first run of 6
    assert z == list(range(14, 20))
    rng = random.Random(3)
    held = {"x": x[5:], "y": y, "z": z}
    for step in range(400):
        k = rng.choice("abcdefgh")
        if k in held and rng.random() < 0.5:
            a.release(held.pop(k))
        else:
            n = rng.randint(1, 6)
            try:
                got = a.alloc(n, after=held[k][-1] if held.get(k) else None)
            except CapacityError:
                continue
            held.setdefault(k, []).extend(got)
        used = [b for v in held.values() for b in v]
        assert len(used) == len(set(used)) and a.free_blocks == 64 - len(used)
    with pytest.raises(ValueError):
        b = held[next(iter(held))][0]
        a.release([b])
        a.release([b])
