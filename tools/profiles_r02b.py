"""Copy the round-2 final measurement set (gpurun_out/m3, tools/measure_r02b.sh)
into profiles/: bench lines, same-config anchors, launch summary, traffic."""
import json, shutil, subprocess, sys
from pathlib import Path
R = Path(__file__).resolve().parents[1]
M, P = R / "gpurun_out" / "m3", R / "profiles"
for f in sorted(M.glob("bench_*.json")):
    txt = f.read_text().strip().splitlines()
    if not txt:
        print("empty", f.name); continue
    (P / f.name.replace(".json", "_r02.json")).write_text(txt[-1] + "\n")
lines = ["Same-configuration anchors (both arms run the WHOLE system; no extrapolation)",
         "GPU arm: bench.py --config cfgN (1 B200, one CUDA graph per step); reference arm: "
         "bench.py --impl reference --config cfgN", ""]
for c, lab in (("cfg2", "2D Q2 64x64 (16,641 DoF)"), ("cfg1", "1D 1024 elements (1,025 DoF)")):
    g = json.loads((P / f"bench_{c}_r02.json").read_text())
    r = json.loads((P / f"bench_{c}_reference_r02.json").read_text())
    cb = r["cpu_baseline"]
    lines += [f"{c} {lab}:",
              f"  GPU value {g['value']:.3e} DoF/s ({g['ms_per_step']:.3f} ms/system), e2e {g['e2e']['value']:.3e} DoF/s",
              f"  reference arm {r['value']:.3e} DoF/s aggregate over {cb['cores']} cores "
              f"({r['ms_per_step']:.1f} ms per step); one core {cb.get('single_core_value', float('nan')):.3e} DoF/s",
              f"  ratio value/reference {g['value'] / r['value']:.1f}x, e2e/reference "
              f"{g['e2e']['value'] / r['value']:.1f}x, value/one core "
              f"{g['value'] / cb.get('single_core_value', float('nan')):.1f}x", ""]
(P / "r02_same_config_anchor.txt").write_text("\n".join(lines))
if (M / "cfg5_launches.csv").exists():
    shutil.copy(M / "cfg5_launches.csv", P / "r02_cfg5_launches.csv")
    out = subprocess.run([sys.executable, str(R / "tools" / "ncu_summary.py"), str(M / "cfg5_launches.csv")],
                         capture_output=True, text=True).stdout
    (P / "r02_cfg5_launches_summary.txt").write_text(
        "ncu launch list of `bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-graph` "
        "(every launch of the run: warm-up, timed, diagnostic, per-level and end-to-end "
        "factor+solve passes; ncu serializes the kernels; --clock-control none)\n" + out)
if (M / "cfg5_traffic.csv").exists():
    out = subprocess.run([sys.executable, str(R / "tools" / "ncu_traffic.py"), str(M / "cfg5_traffic.csv"), "cfg5"],
                         capture_output=True, text=True).stdout
    if out.strip():
        (P / "traffic_cfg5.json").write_text(out)
if (M / "gpu_tests.log").exists():
    shutil.copy(M / "gpu_tests.log", P / "r02_gpu_tests.log")
print("ok")
