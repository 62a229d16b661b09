"""The C-ABI library loads without a GPU and exports every symbol include/askv.h
declares; the ctypes signature table covers exactly those symbols."""

import ctypes
import json
import os
import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def declared():
    text = (ROOT / "include" / "askv.h").read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(askv_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def built():
    from paper_2403_19708_b200 import build
    return build.build()


def test_header_declares_hot_path_entry_points():
    names = declared()
    for fn in ("askv_reembed", "askv_prefill_attn", "askv_preload_layer", "askv_save_layer",
               "askv_rope_new", "askv_version"):
        assert fn in names


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(str(built))
    for name in declared():
        assert hasattr(lib, name), name


def test_ctypes_table_matches_header(built):
    from paper_2403_19708_b200 import _lib
    assert sorted(_lib.SIGNATURES) == declared()
    lib = _lib.lib()
    assert lib.askv_version() == 100
    assert lib.askv_last_error() == b""
    # the ctypes mirror of askv_prefill_plan has the C layout
    assert ctypes.sizeof(_lib.PrefillPlan) == lib.askv_prefill_plan_size()


def _sk_slots(n_cached, n_new, hq, hkv, sms=148, bm=128, bn=128):
    """Python restatement of K3's stream-K schedule (csrc/attention.cu sk_plan):
    (units, max partial slots of a unit)."""
    pack = hq // hkv if hq > hkv and 128 % (hq // hkv) == 0 and hq // hkv <= 16 else 1
    q_rows = n_new * pack
    qt = -(-q_rows // bm)
    tiles = [-(-(n_cached + (min((q + 1) * bm, q_rows) - 1) // pack + 1) // bn)
             for q in range(qt)]
    heads = hkv if pack > 1 else hq
    units = [(h, q, t) for h in range(heads) for q, t in enumerate(tiles)]
    total = sum(t for *_, t in units)
    min_per = -(-max(tiles) // 23)
    ctas = max(1, min(sms, total // min_per))
    owner = lambda g: ((g + 1) * ctas - 1) // total  # noqa: E731
    slots, ub = 1, 0
    for h, q, t in units:
        slots = max(slots, owner(ub + t - 1) - owner(ub) + 1)
        ub += t
    return len(units), slots


def test_split_policy_without_gpu(built):
    from paper_2403_19708_b200 import _lib
    lib = _lib.lib()
    # one query tile x 40 heads = 40 CTAs: split the 18 KV tiles 3 ways (one wave)
    assert lib.askv_attn_num_splits(2142, 100, 40, 148) == 3
    # 13B p50 turn (2 query tiles x 40 heads = 80 CTAs) already fills a wave
    assert lib.askv_attn_num_splits(2142, 237, 40, 148) == 1
    # 70B TP8 rank (8 q-heads): split while >= 6 KV tiles per split remain
    assert lib.askv_attn_num_splits(2048, 256, 8, 148) == 3
    # short history: 9 KV tiles would leave 5 per split -- not worth a combine
    assert lib.askv_attn_num_splits(1000, 100, 40, 148) == 1
    # full recompute of 2379 tokens fills the machine without splitting
    assert lib.askv_attn_num_splits(0, 2379, 40, 148) == 1
    assert lib.askv_attn_workspace_bytes(2142, 237, 40, 128, 4) == 4 * 237 * 40 * 129 * 4


def test_stream_k_schedule_without_gpu(built):
    """Opt-in stream-K schedule (ASKV_ATTN_SK=1, read once per process): one
    launch, no uniform split; its partial slabs are slots x units x 128 rows x
    (d + 1) fp32 with the slot count of the python restatement, none when no
    unit is cut (148 SMs when no GPU is visible)."""
    import subprocess
    import sys
    cases = [(2142, 237, 40, 40), (2142, 100, 40, 40), (2869, 301, 8, 1), (1000, 60, 2, 2),
             (100, 5, 4, 4), (4000, 90, 1, 1)]
    code = ("import sys, json; sys.path.insert(0, %r)\n"
            "from paper_2403_19708_b200 import _lib\n"
            "lib = _lib.lib()\n"
            "print(json.dumps([[lib.askv_attn_num_splits_gqa(k, n, h, v, 148),"
            " lib.askv_attn_workspace_bytes_gqa(k, n, h, v, 128, 0)] for k, n, h, v in %r]))"
            % (str(Path(__file__).resolve().parent.parent), cases))
    env = dict(os.environ, ASKV_ATTN_SK="1")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, env=env,
                         check=True).stdout
    got = json.loads(out.strip().splitlines()[-1])
    for (kept, n, hq, hkv), (splits, ws) in zip(cases, got):
        units, slots = _sk_slots(kept, n, hq, hkv)
        assert splits == 1
        assert ws == (slots * units * 128 * 129 * 4 if slots > 1 else 0), (kept, n)


def test_argument_errors_without_gpu(built):
    """Validation happens before any CUDA call, so it is testable on CPU."""
    from paper_2403_19708_b200 import _lib
    lib = _lib.lib()
    rc = lib.askv_prefill_attn(None, None, 256, 0, 4, 3, 2, 128, 1.0, None, None, 0, 0, None)
    assert rc == _lib.ASKV_EINVAL
    assert b"multiple" in lib.askv_last_error()
    rc = lib.askv_save_layer(None, None, 1, 100, 0, 16, 8, 0, 40, None, None, None)
    assert rc == _lib.ASKV_EINVAL


def test_attention_kernel_does_not_spill(built):
    """K3's softmax warpgroups run with 224 registers (setmaxnreg); before the
    register split the 168-register cap spilled ~100 B per thread inside the
    tile loop.  Guard the split: the fused kernels keep (almost) no stack."""
    import shutil
    import subprocess
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(tool).exists():
        pytest.skip("cuobjdump not available")
    out = subprocess.run([tool, "-res-usage", str(built)], capture_output=True, text=True,
                         check=True).stdout
    stacks = {}
    name = None
    for line in out.splitlines():
        m = re.search(r"Function (\S+):", line)
        if m:
            name = m.group(1)
            continue
        m = re.search(r"STACK:(\d+)", line)
        if m and name and ("attn_fwd_kernel" in name or "attn_sk_kernel" in name):
            stacks[name] = int(m.group(1))
    assert len(stacks) == 6, stacks  # HD 64 / 128 x unpaired / paired / stream-K
    assert max(stacks.values()) <= 16, stacks


def test_attention_build_knobs_default_to_the_measured_kernel():
    """K3's build-time A/B knobs must default to the measured
    product configuration: the experiment variants (pipeline probes, column
    split, per-warp arrival, evict_first) are opt-in only."""
    src = (ROOT / "paper_2403_19708_b200" / "csrc" / "attention.cu").read_text()
    want = {"ASKV_ATTN_PROBE": "0", "ASKV_ATTN_COLSPLIT": "0", "ASKV_ATTN_WARP_ARRIVE": "0",
            "ASKV_ATTN_LAST_OFULL": "1", "ASKV_ATTN_LAST_OFULL_ALL": "0",
            "ASKV_ATTN_EARLY_VFREE": "1", "ASKV_ATTN_KV_POLICY": "1", "ASKV_ATTN_INTERLEAVE": "0", "ASKV_ATTN_ELECT_ISSUE": "1",
            "ASKV_ATTN_SUMCHECK": "1", "ASKV_ATTN_POLY_Q": "1", "ASKV_ATTN_L2_PREFETCH": "0"}
    for knob, val in want.items():
        m = re.search(r"#define %s (\S+)" % knob, src)
        assert m and m.group(1) == val, (knob, m and m.group(1))
