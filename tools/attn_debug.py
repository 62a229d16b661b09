"""Per-row error map of K3 vs a torch fp32 reference (diagnostics only).
    python tools/attn_debug.py kept n hq hkv d [splits]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2403_19708_b200 import ops  # noqa: E402


def ref(q, kv, kept, n, hq, hkv):
    g = hq // hkv
    k = kv[:, 0].float().repeat_interleave(g, dim=1)  # [T, hq, d]
    v = kv[:, 1].float().repeat_interleave(g, dim=1)
    s = torch.einsum("nhd,thd->hnt", q.float(), k) / q.shape[-1] ** 0.5
    t = torch.arange(kept + n, device=q.device)
    mask = t[None, :] > (kept + torch.arange(n, device=q.device))[:, None]
    s = s.masked_fill(mask[None], float("-inf"))
    return torch.einsum("hnt,thd->nhd", s.softmax(-1), v)


def main():
    kept, n, hq, hkv, d = (int(x) for x in sys.argv[1:6])
    splits = int(sys.argv[6]) if len(sys.argv) > 6 else 0
    g = torch.Generator(device="cuda").manual_seed(0)
    q = torch.randn(n, hq, d, device="cuda", generator=g).to(torch.bfloat16)
    kv = torch.randn(kept + n, 2, hkv, d, device="cuda", generator=g).to(torch.bfloat16)
    out = torch.empty(n, hq, d, device="cuda", dtype=torch.bfloat16)
    s = splits or ops.attn_num_splits(kept, n, hq)
    ws = torch.empty(max(1, ops.attn_workspace_bytes(kept, n, hq, d, s)), dtype=torch.uint8,
                     device="cuda")
    ops.prefill_attn(q, kv, kept, n, hq, hkv, d, out, ws, num_splits=s)
    torch.cuda.synchronize()
    want = ref(q, kv, kept, n, hq, hkv)
    err = (out.float() - want).abs().amax(dim=2)  # [n, hq]
    print(f"shape kept={kept} n={n} hq={hq} hkv={hkv} d={d} splits={s}: "
          f"max err {err.max().item():.3e}")
    bad = (err > 2e-2).nonzero().tolist()
    rows = sorted({r for r, _ in bad})
    print("bad rows:", len(rows), rows[:40], "...", rows[-10:] if rows else "")
    print("bad heads:", sorted({h for _, h in bad}))


if __name__ == "__main__":
    main()
