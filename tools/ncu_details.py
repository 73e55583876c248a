"""Print key metrics and top stall reasons from an ncu report (details + raw pages)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
want = ["Duration", "DRAM Throughput", "Compute (SM) Throughput", "Achieved Occupancy",
        "Registers Per Thread", "Grid Size", "Block Size", "Executed Ipc Active",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate"]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
seen = set()
for r in rows[1:]:
    if r[mi] in want and r[mi] not in seen:
        seen.add(r[mi]); print(f"{r[mi]:40s} {r[vi]} {r[ui]}")
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
h = rr[0]
vals = rr[2] if len(rr) > 2 else []
stalls = []
for i, name in enumerate(h):
    if name.startswith("smsp__average_warp_latency_issue_stalled_") or name.startswith("smsp__pcsamp_warps_issue_stalled_"):
        try:
            stalls.append((float(vals[i].replace(",", "")), name))
        except Exception:
            pass
    if name in ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                "dram__bytes_read.sum", "dram__bytes_write.sum",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active"):
        print(f"{name:60s} {vals[i]}")
for v, n in sorted(stalls, reverse=True)[:10]:
    print(f"  stall {n:75s} {v}")
