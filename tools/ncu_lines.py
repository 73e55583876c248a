"""Per-source-line instruction counts and stall samples from an ncu report (cuda,sass view)."""
import collections, csv, subprocess, sys
rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
cur = None; hdr = None
agg = collections.defaultdict(lambda: [0, 0, ""])
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]; continue
    if r[0] == "Line No":
        hdr = r; continue
    if hdr is None or len(r) < 8:
        continue
    try:
        ln, w, n = int(r[0]), int(r[4] or 0), int(r[7] or 0)
    except ValueError:
        continue
    a = agg[(cur, ln)]; a[0] += w; a[1] += n; a[2] = r[1].strip()[:95]
tw = sum(v[0] for v in agg.values()); tn = sum(v[1] for v in agg.values())
print(f"samples {tw}  warp-instructions {tn}")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1])[:top]:
    print(f"{v[1] / tn:6.1%} inst {v[0] / max(tw, 1):6.1%} stall  {k[0]}:{k[1]}  {v[2]}")
