"""bench.py keeps the driver's JSON contract (both arms)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "e2e"}


def run(args, timeout=900):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK")}
    out = subprocess.run([sys.executable, str(ROOT / "bench.py")] + args, capture_output=True,
                         text=True, timeout=timeout, cwd=str(ROOT), env=env)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_reference_arm_contract():
    d = run(["--impl", "reference", "--config", "cfg1", "--steps", "2", "--warmup", "1"])
    assert KEYS <= set(d) and d["impl"] == "reference"
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["config"]["workload"] == "cfg1"
    c = d["cpu_baseline"]
    assert c["kind"] == "port" and c["cores"] >= 1 and c["value"] == d["value"]
    assert c["cpu_model"] and c["nproc"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    # the reference arm never imports the product package
    code = ("import runpy, sys; sys.argv = ['bench.py', '--impl', 'reference', '--config', 'cfg1',"
            " '--steps', '1', '--warmup', '0']; runpy.run_path('bench.py', run_name='__main__');"
            " bad = [m for m in sys.modules if m.startswith('paper_2306_08994_b200')];"
            " assert not bad, bad")
    out = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=600,
                         cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]


@pytest.mark.gpu
def test_gpu_arm_contract(cuda_ok):
    d = run(["--config", "cfg2", "--steps", "3", "--warmup", "3"])
    assert KEYS <= set(d)
    assert d["value"] > 0 and d["dtype"] == "f64" and d["n_gpus"] == 1
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert {"bound", "achieved", "peak", "unit", "frac", "traffic"} <= set(r) and 0 < r["frac"] < 1.5
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["clocks"]["sm_mhz"] and "reasons" in d["clocks"]
    assert d["cpu_baseline"]["value"] > 0 and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["rel_residual"] < 1e-12
    assert set(d["modelled_scaling"]) == {"2", "4", "8"}
