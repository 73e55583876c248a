"""Summarise an ncu --csv launch list: per-kernel count and total device time
(rows of gpu__time_duration.sum; other metrics in the capture are ignored)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
start = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[start]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
scale = {"nsecond": 1e-6, "ns": 1e-6, "usecond": 1e-3, "us": 1e-3, "msecond": 1.0, "ms": 1.0,
         "second": 1e3, "s": 1e3}
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[start + 1:]:
    if len(r) <= vi or r[mi] != "gpu__time_duration.sum":
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", "")) * scale[r[ui]]
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total serialized {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} n={n:5d} ms={t:9.3f} share={t / tot:6.1%}")
