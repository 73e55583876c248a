"""DRAM traffic per launch and kernel class from an ncu CSV capture of
`--metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum`.

usage: python tools/ncu_traffic.py CAPTURE.csv CONFIG > profiles/traffic_CONFIG.json
Kernel classes use the names of tf_timing_class_name (bench.py's roofline key).
"""
import collections, csv, json, sys

CLASSES = [("large_update_kernel<1", "large_update_kernel<1> (schur)"),
           ("large_update_kernel<0", "large_update_kernel<0> (panel)"),
           ("large_update_kernel<2", "large_update_kernel<2> (trsm)"),
           ("factor_small_kernel", "factor_small_kernel"),
           ("large_assemble_kernel", "large_assemble_kernel")]

rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9,
         "B": 1, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "ns": 1e-9, "us": 1e-6}
per = collections.defaultdict(lambda: collections.defaultdict(float))
for r in rows[start + 1:]:
    if len(r) <= vi:
        continue
    key = (r[0], r[ki])
    per[key][r[mi]] += float(r[vi].replace(",", "")) * scale.get(r[ui], 1.0)
out = {"capture": sys.argv[1], "config": sys.argv[2], "kernels": {}}
for pat, name in CLASSES:
    ks = [v for (i, k), v in per.items() if pat in k]
    if not ks:
        continue
    n = len(ks)
    rd = sum(v["dram__bytes_read.sum"] for v in ks)
    wr = sum(v["dram__bytes_write.sum"] for v in ks)
    t = sum(v["gpu__time_duration.sum"] for v in ks)
    out["kernels"][name] = {"launches": n, "dram_bytes_per_launch": (rd + wr) / n,
                            "dram_read_bytes": rd, "dram_write_bytes": wr,
                            "serialized_ms": t * 1e3}
print(json.dumps(out, indent=1))
