"""Summarise an `ncu --set full` report (read here with `ncu -i ... --page raw --csv`).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [--traffic-json profiles/ncu_attn_traffic.json]

Prints one markdown table per captured kernel (duration, DRAM / L2 bytes,
tensor-pipe and issue utilisation, occupancy) and optionally writes the DRAM
traffic of the first captured launch for bench.py's `roofline.traffic`.
"""
import argparse
import csv
import io
import json
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__cycles_elapsed.avg.per_second", "SM clock"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("lts__t_bytes.sum", "L2 bytes (all)"),
    ("lts__t_sector_hit_rate.pct", "L2 hit rate"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM throughput"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory throughput"),
    ("TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
     "tensor pipe active (elapsed)"),
    ("TPC.TriageCompute.sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg",
     "tensor (hmma/tcgen05) subpipe active cycles per SM"),
    ("sm__cycles_elapsed.avg", "SM cycles elapsed"),
    ("sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
     "tensor memory (TMEM) active, % of active cycles"),
    ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU) pipe"),
    ("sm__issue_active.avg.pct_of_peak_sustained_elapsed", "issue slots busy (elapsed)"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "registers/thread"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy"),
]


def load(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units = rows[0], rows[1]
    return head, units, rows[2:]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--traffic-json", default="")
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    head, units, rows = load(a.report)
    idx = {h: i for i, h in enumerate(head)}
    first = None
    for r in rows:
        name = r[idx["Kernel Name"]] if "Kernel Name" in idx else "?"
        print(f"\n### {name[:110]}\n")
        print("| metric | value |\n|---|---|")
        for key, label in METRICS:
            if key in idx and r[idx[key]] not in ("", "n/a"):
                print(f"| {label} (`{key}`) | {r[idx[key]]} {units[idx[key]]} |")
        if first is None:
            first = r
    if a.traffic_json and first is not None:
        def num(key):
            v = first[idx[key]].replace(",", "")
            u = units[idx[key]]
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
            return float(v) * scale
        traffic = num("dram__bytes_read.sum") + num("dram__bytes_write.sum")
        json.dump({"bytes_per_launch": traffic, "report": a.report, "note": a.note,
                   "kernel": first[idx["Kernel Name"]][:160],
                   "grid": first[idx["launch__grid_size"]]},
                  open(a.traffic_json, "w"), indent=1)
        print(f"\nwrote {a.traffic_json}: {traffic:.3e} B/launch", file=sys.stderr)


if __name__ == "__main__":
    main()
