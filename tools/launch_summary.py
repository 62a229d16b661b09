"""Summarise an ncu launch list (`ncu --metrics gpu__time_duration.sum --csv
--log-file X.csv ...`) as a markdown table of per-kernel shares.

    python tools/launch_summary.py gpurun_out/r01d_launches.csv

Set-up launches (weight init, arena fill, GEMM autotune) are skipped: the table
starts at the first device timestamp (stamp_kernel) of the first bench job.
ncu serialises kernels and runs them cold, so shares, not absolute times, carry
over to the bench.
"""
import collections
import csv
import sys

GROUPS = [("nvjet", "cuBLASLt GEMM (nvjet)"), ("attn_fwd", "askv attn_fwd (K3)"),
          ("attn_combine", "askv attn_combine (K3 split-KV merge)"),
          ("reembed", "askv reembed (K2)"), ("rope_new", "askv rope_new"),
          ("rmsnorm", "askv rmsnorm"), ("silu_mul", "askv silu_mul"),
          ("stamp_kernel", "askv stamp (device timeline)"), ("copy_sm", "askv copy_sm")]


def label(name: str) -> str:
    for key, lab in GROUPS:
        if key in name:
            return lab
    return "torch: " + name[:60]


def main():
    lines = [ln for ln in open(sys.argv[1]) if not ln.startswith("==")]  # ncu notes
    rows = list(csv.DictReader(lines))
    rows = [r for r in rows if r.get("Metric Name") == "gpu__time_duration.sum"]
    start = next((i for i, r in enumerate(rows) if "stamp_kernel" in r["Kernel Name"]), 0)
    agg = collections.OrderedDict()
    total = 0.0
    for r in rows[start:]:
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "ns")
        us = v / 1e3 if unit in ("ns", "nsecond") else v * 1e3 if unit in ("ms", "msecond") else v
        key = label(r["Kernel Name"])
        n, t = agg.get(key, (0, 0.0))
        agg[key] = (n + 1, t + us)
        total += us
    print(f"Step kernels captured: {sum(n for n, _ in agg.values())} launches, "
          f"{total:.1f} us (set-up launches before the first job excluded)\n")
    print("| kernel | launches | total us | share | avg us |\n|---|---|---|---|---|")
    for key, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"| {key} | {n} | {t:.1f} | {100 * t / total:.1f}% | {t / n:.2f} |")


if __name__ == "__main__":
    main()
