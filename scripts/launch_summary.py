"""Summarise an ncu --metrics gpu__time_duration.sum launch list (CSV).

python scripts/launch_summary.py <launches.csv>
Prints per-kernel launch count, average duration (us) and share of kernel time.
"""
import collections
import csv
import sys


def load(path):
    hdr = None
    out = []
    with open(path) as f:
        for r in csv.reader(f):
            if "Kernel Name" in r:
                hdr = r
                continue
            if hdr and len(r) == len(hdr):
                rec = dict(zip(hdr, r))
                if rec.get("Metric Name") == "gpu__time_duration.sum":
                    v = float(rec["Metric Value"].replace(",", ""))
                    unit = rec.get("Metric Unit", "ns")
                    scale = {"ns": 1e-3, "nsecond": 1e-3, "usecond": 1.0, "us": 1.0,
                             "msecond": 1e3, "ms": 1e3}.get(unit, 1e-3)
                    out.append((rec["Kernel Name"], v * scale, rec.get("Grid Size", "")))
    return out


def main():
    recs = load(sys.argv[1])
    d = collections.defaultdict(list)
    for name, us, grid in recs:
        short = name.split("(")[0].replace("void ", "")[:70]
        d[short].append(us)
    tot = sum(sum(v) for v in d.values())
    print(f"{'share':>6} {'n':>5} {'avg_us':>8}  kernel   (total {tot:.1f} us over {len(recs)} launches)")
    for k, v in sorted(d.items(), key=lambda kv: -sum(kv[1])):
        print(f"{sum(v)/tot*100:5.1f}% {len(v):5d} {sum(v)/len(v):8.2f}  {k}")


if __name__ == "__main__":
    main()
