#!/usr/bin/env python
"""Summarise ncu evidence for profiles/: key raw metrics + stall breakdown of a
--set full report, or per-kernel averages of a gpu__time_duration launch list.

    python tools/ncu_summary.py report.ncu-rep > profiles/<name>.txt
    python tools/ncu_summary.py launches.csv   > profiles/<name>.txt
"""
import collections
import csv
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "lts__t_bytes.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
]


def report(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for vals in rows[2:]:
        name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
        print(f"kernel: {name}")
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                print(f"  {k:75s} {vals[i]:>18s} {units[i]}")
        st = [(float(v), h) for h, v in zip(hdr, vals)
              if h.startswith("smsp__pcsamp_warps_issue_stalled") and not h.endswith("not_issued")
              and v not in ("", "0")]
        tot = sum(s for s, _ in st) or 1.0
        print("  stall reasons (pc sampling):")
        for s, h in sorted(st, reverse=True)[:8]:
            print(f"    {100 * s / tot:5.1f}%  {h.replace('smsp__pcsamp_warps_issue_stalled_', '')}")


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr = rows[hi]
    ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg.setdefault(r[ki].split("(")[0], []).append((float(r[vi].replace(",", "")), r[ui]))
    print(f"{'kernel':45s} {'launches':>8s} {'avg':>12s}")
    for k, v in agg.items():
        avg = sum(x for x, _ in v) / len(v)
        print(f"{k[:45]:45s} {len(v):8d} {avg:12.1f} {v[0][1]}")


if __name__ == "__main__":
    p = sys.argv[1]
    (report if p.endswith(".ncu-rep") else launches)(p)
