"""Registers and spills per kernel from a ptxas -v log (build/<unit>.ptxas.log).
    python tools/ptxas_summary.py build/mlp_tc.ptxas.log [name-filter]"""
import re
import sys

name, spill = None, None
flt = sys.argv[2] if len(sys.argv) > 2 else ""
for line in open(sys.argv[1]):
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        name = m.group(1)
    m = re.search(r"(\d+) bytes spill stores, (\d+) bytes spill loads", line)
    if m:
        spill = (int(m.group(1)), int(m.group(2)))
    m = re.search(r"Used (\d+) registers", line)
    if m and name and flt in name:
        print(f"{name[:70]:70s} regs {m.group(1):>4s} spill st/ld {spill}")
        name = None
