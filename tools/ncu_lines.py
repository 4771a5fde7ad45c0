#!/usr/bin/env python
"""Per-CUDA-source-line stall samples and executed instructions of one kernel in an ncu
report (source page, cuda,sass view): the top lines, and totals over line ranges.

    python tools/ncu_lines.py report.ncu-rep [top] [a-b a-b ...]

NCU_KERNEL=<regex> selects one kernel of a multi-kernel report.
"""
import os
import csv
import subprocess
import sys


def load(path):
    sel = ["-k", "regex:" + os.environ["NCU_KERNEL"]] if os.environ.get("NCU_KERNEL") else []
    out = subprocess.run(["ncu", "-i", path, *sel, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
    h = rows[hi]
    # SASS rows (empty line number, an address) carry the metrics in fixed columns; a CUDA
    # line row (its source text may contain unquoted commas) sets the current line
    i_s, i_e = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    lines = {}
    src = {}
    cur = None
    for r in rows[hi + 1:]:
        if r and r[0]:
            if not r[0].isdigit():   # a new file / function header
                cur = None
                continue
            cur = int(r[0])
            src[cur] = ",".join(r[1:-6])
            continue
        if cur is None or len(r) <= i_e or not r[2].startswith("0x"):
            continue
        s = int(r[i_s] or 0)
        e = int(r[i_e] or 0)
        a = lines.setdefault(cur, [0, 0])
        a[0] += s
        a[1] += e
    return lines, src


def main():
    lines, src = load(sys.argv[1])
    top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
    ts = sum(v[0] for v in lines.values()) or 1
    te = sum(v[1] for v in lines.values()) or 1
    print(f"total samples {ts}, warp-instructions {te}")
    for ln, (s, e) in sorted(lines.items(), key=lambda kv: -kv[1][0])[:top]:
        print(f"{ln:5d} {100 * s / ts:6.2f}% samples {100 * e / te:6.2f}% inst | {src.get(ln, '')[:90]}")
    for rng in sys.argv[3:]:
        a, b = (int(x) for x in rng.split("-"))
        s = sum(v[0] for k, v in lines.items() if a <= k <= b)
        e = sum(v[1] for k, v in lines.items() if a <= k <= b)
        print(f"lines {a}-{b}: {100 * s / ts:6.2f}% samples {100 * e / te:6.2f}% inst")


if __name__ == "__main__":
    main()
