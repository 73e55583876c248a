"""Summarise an ncu --csv launch list: per-kernel count and total device time."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
for i, r in enumerate(rows):
    if r and r[0] == "ID":
        hdr, start = r, i + 1
        break
ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
agg = collections.defaultdict(lambda: [0, 0.0])
tot = 0.0
for r in rows[start:]:
    if len(r) <= vi:
        continue
    name = r[ki].split("(")[0][:70]
    v = float(r[vi].replace(",", "")) / 1e6
    agg[name][0] += 1
    agg[name][1] += v
    tot += v
print(f"total {tot:.3f} ms over {sum(a[0] for a in agg.values())} launches")
for k, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{k:70s} n={n:5d} ms={t:9.3f} share={t / tot:6.1%}")
