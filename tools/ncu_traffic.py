#!/usr/bin/env python
"""DRAM bytes per launch of every step kernel in an `ncu --set full` report, as the JSON
bench.py reads for `roofline.traffic` / `kernels[*].dram_bytes_ncu`:

    python tools/ncu_traffic.py report.ncu-rep > profiles/r2_dram_traffic.json
"""
import csv
import json
import subprocess
import sys

STAGE = (("prolongate", "K1_prolong"), ("element_kernel", "K2_residual"),
         ("node_sum", "K2_residual"), ("mlp_tc_kernel", "K3K4_gather_mlp"),
         ("scatter_update", "K5_scatter"))


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    ik = hdr.index("Kernel Name")
    ir, iw = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per, parts = {}, {}
    for v in rows[2:]:
        b = float(v[ir].replace(",", "")) * scale[units[ir]] + float(v[iw].replace(",", "")) * scale[units[iw]]
        for pat, stage in STAGE:
            if pat in v[ik]:
                short = v[ik].split("(")[0].replace("void ", "")
                parts.setdefault(stage, {}).setdefault(short, []).append(b)
    res = {"source": "ncu --set full --clock-control none, config-3 step (tools/gpu/step_run.py "
                     "64x32x32, f16x3); dram__bytes_read.sum + dram__bytes_write.sum per launch "
                     "(mean over the captured launches of each kernel)"}
    for stage, ks in parts.items():
        means = {k: sum(x) / len(x) for k, x in ks.items()}
        per[stage] = int(sum(means.values()))
        if len(means) > 1:
            res[stage + "_parts"] = {k: int(x) for k, x in means.items()}
    res.update(per)
    print(json.dumps(res, indent=2))


if __name__ == "__main__":
    main(sys.argv[1])
