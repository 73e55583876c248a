"""Generate on-disk-format goldens by running the REFERENCE CLI itself.

Run in the build container only (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_fileio_golden.py

Writes tests/golden/fileio/<case>/{matrix.mtx, rhs.txt, manifest.json,
L.mtx, U.mtx, pivot_order.txt, solution.txt} from `tracefront.cli` (generate,
factorize, solve; cli.py:164-221).
"""
import shutil
import subprocess
import sys
from pathlib import Path

OUT = Path(__file__).resolve().parent / "fileio"
CASES = {"1d_n6_p2": ["--elements", "6", "--degree", "2"],
         "1d_n5_p3_sin": ["--elements", "5", "--degree", "3", "--rhs", "sin_pi"]}

for name, flags in CASES.items():
    d = OUT / name
    shutil.rmtree(d, ignore_errors=True)
    d.mkdir(parents=True)
    for cmd in ("generate", "factorize", "solve"):
        r = subprocess.run([sys.executable, "-m", "tracefront.cli", cmd, *flags, "--out", str(d)],
                           capture_output=True, text=True)
        print(name, cmd, r.returncode, r.stdout.strip().splitlines()[-1:] if r.stdout else r.stderr[-200:])
