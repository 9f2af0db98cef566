"""Summarise an ncu launch list (CSV of --metrics gpu__time_duration.sum
[,dram__bytes_read.sum,dram__bytes_write.sum]).

python scripts/launch_summary.py <launches.csv> [--json out.json]
Prints per-kernel launch count, average duration (us), share of kernel time
and, when captured, average DRAM bytes per launch; --json writes
{kernel: dram bytes per launch} (the bench's roofline "traffic" table).
"""
import collections
import csv
import json
import sys

SCALE = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3, "ms": 1e3}
BSCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def load(path):
    hdr = None
    launches = collections.OrderedDict()
    with open(path) as f:
        for r in csv.reader(f):
            if "Kernel Name" in r:
                hdr = r
                continue
            if not hdr or len(r) != len(hdr):
                continue
            rec = dict(zip(hdr, r))
            key = rec["ID"]
            ent = launches.setdefault(key, {"name": rec["Kernel Name"], "us": 0.0, "dram": None})
            v = float(rec["Metric Value"].replace(",", ""))
            unit = rec.get("Metric Unit", "")
            mn = rec.get("Metric Name")
            if mn == "gpu__time_duration.sum":
                ent["us"] = v * SCALE.get(unit, 1e-3)
            elif mn in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                ent["dram"] = (ent["dram"] or 0.0) + v * BSCALE.get(unit, 1.0)
    return list(launches.values())


def short(name):
    return name.split("(")[0].replace("void ", "")[:70]


def main():
    recs = load(sys.argv[1])
    d = collections.defaultdict(list)
    for r in recs:
        d[short(r["name"])].append(r)
    tot = sum(r["us"] for r in recs)
    print(f"{'share':>6} {'n':>5} {'avg_us':>8} {'dram_MB':>8}  kernel   "
          f"(total {tot:.1f} us over {len(recs)} launches)")
    traffic = {}
    for k, v in sorted(d.items(), key=lambda kv: -sum(r["us"] for r in kv[1])):
        us = sum(r["us"] for r in v)
        drams = [r["dram"] for r in v if r["dram"] is not None]
        dm = sum(drams) / len(drams) if drams else None
        if dm is not None:
            traffic[k] = dm
        dms = f"{dm / 1e6:8.2f}" if dm is not None else "       -"
        print(f"{us / tot * 100:5.1f}% {len(v):5d} {us / len(v):8.2f} {dms}  {k}")
    if "--json" in sys.argv:
        out = sys.argv[sys.argv.index("--json") + 1]
        with open(out, "w") as f:
            json.dump(traffic, f, indent=1, sort_keys=True)


if __name__ == "__main__":
    main()
