#!/usr/bin/env python
"""Summarise an exported ncu raw page (scripts/ncu_export.sh -> raw.csv.gz)
as a markdown table per kernel: launches, mean duration, DRAM bytes, DRAM /
SM / tensor-pipe utilisation, grid, registers, dynamic smem.

    python scripts/ncu_summary.py gpurun_out/TAG/raw.csv.gz
"""
import csv
import gzip
import sys
from collections import OrderedDict

COLS = {
    "t": "gpu__time_duration.sum",
    "rd": "dram__bytes_read.sum",
    "wr": "dram__bytes_write.sum",
    "dram": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "tc": "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
    "warps": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "grid": "launch__grid_size",
    "regs": "launch__registers_per_thread",
    "smem": "launch__shared_mem_per_block_dynamic",
}


def num(x):
    try:
        return float(str(x).replace(",", ""))
    except ValueError:
        return float("nan")


def main(path):
    with gzip.open(path, "rt") if path.endswith(".gz") else open(path) as f:
        rows = list(csv.reader(f))
    head, units = rows[0], rows[1]
    idx = {k: head.index(v) for k, v in COLS.items() if v in head}
    name_i = head.index("Kernel Name")
    unit = {k: units[i] for k, i in idx.items()}
    agg = OrderedDict()
    for r in rows[2:]:
        if len(r) < len(head):
            continue
        nm = r[name_i].split("(")[0].replace("void ", "")
        a = agg.setdefault(nm, {"n": 0, **{k: 0.0 for k in idx}})
        a["n"] += 1
        for k, i in idx.items():
            a[k] += num(r[i])
    tscale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
              "ms": 1e3}.get(unit.get("t", "ns"), 1e-3)
    bs = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1.0, "Gbyte": 1e3}
    rscale = bs.get(unit.get("rd", "byte"), 1e-6)  # each column carries its own unit
    wscale = bs.get(unit.get("wr", "byte"), 1e-6)
    sscale = 1.0 if unit.get("smem", "").startswith("Kbyte") else 1 / 1024
    print("| kernel | launches | time us (ncu, cold) | DRAM read MB | DRAM write MB | DRAM % peak "
          "| SM thr % | tensor pipe % | warps active % | grid | regs | dyn smem KB |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|")
    for nm, a in agg.items():
        n = a["n"]
        g = lambda k, s=1.0: a[k] / n * s if k in a else float("nan")
        print(f"| {nm} | {n} | {g('t', tscale):.2f} | {g('rd', rscale):.3f} | {g('wr', wscale):.3f} "
              f"| {g('dram'):.1f} | {g('sm'):.1f} | {g('tc'):.1f} | {g('warps'):.1f} | {g('grid'):.0f} "
              f"| {g('regs'):.0f} | {g('smem') * sscale:.0f} |")


if __name__ == "__main__":
    main(sys.argv[1])
