"""Per-launch DRAM traffic (dram__bytes_read.sum + dram__bytes_write.sum) of
the step's kernels from an exported ncu raw page, keyed by bench.py's op
names: the `traffic` field of the bench line's roofline object.

    python scripts/ncu_traffic.py gpurun_out/TAG/raw.csv.gz profiles/traffic_rNN.json "source note"
"""
import csv
import gzip
import json
import sys

OPS = [("tc2_kernel<0>", "sage_transform_l0"), ("tc2_kernel<1>", "sage_transform_bwd_l0"),
       ("sage_head_kernel", "sage_head"), ("sage_aggregate_parts_kernel", "sage_aggregate_l0"),
       ("sage_scatter_bwd_kernel", "sage_scatter_bwd_l0"), ("adam_kernel", "optimizer"),
       ("gather_q_kernel", "prep_gather"), ("sample_q_kernel", "prep_sample")]


def main(path, out, note):
    rows = list(csv.reader(gzip.open(path, "rt")))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    rd = hdr.index("dram__bytes_read.sum")
    wr = hdr.index("dram__bytes_write.sum")
    units = rows[1]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6}
    acc = {}
    for r in rows[2:]:
        name = r[ki]
        for pat, op in OPS:
            if pat.replace("<", "<").split("<")[0] in name and (("<" not in pat) or pat in name.replace(" ", "")):
                b = (float(r[rd].replace(",", "")) * scale.get(units[rd], 1)
                     + float(r[wr].replace(",", "")) * scale.get(units[wr], 1))
                acc.setdefault(op, []).append(b)
                break
    res = {"source": note}
    res.update({op: sum(v) / len(v) for op, v in acc.items()})
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else "")
