"""CLI harness (mirrors tracefront's cli.py:64-356)."""
import subprocess
import sys

import pytest

from paper_2306_08994_b200 import cli


def run(*argv):
    return subprocess.run([sys.executable, "-m", "paper_2306_08994_b200.cli", *argv],
                          capture_output=True, text=True)


def test_plan_1d_matches_reference_depth():
    r = run("plan", "--elements", "1024", "--degree", "1")
    assert r.returncode == 0, r.stderr
    assert "tree_depth=11" in r.stdout and "n_dof=1025" in r.stdout


# `tracefront plan` output of the reference itself (cli.py:184-196), captured with
# PYTHONPATH=/root/reference/pkg/src python -m tracefront.cli plan --elements N --degree P
REF_PLAN = {
    ("1024", "1"): "n_dof=1025 tree_depth=11 tasks_division=2028 tasks_multiplication=4036 "
                   "tasks_subtraction=4036 tasks_assertion=5081 tasks_total=15181 "
                   "foata_classes=50 max_class_width=2560",
    ("64", "3"): "n_dof=193 tree_depth=7 tasks_division=436 tasks_multiplication=1052 "
                 "tasks_subtraction=1052 tasks_assertion=1065 tasks_total=3605 "
                 "foata_classes=40 max_class_width=576",
}


@pytest.mark.parametrize("n,p", sorted(REF_PLAN))
def test_plan_prints_reference_lines(n, p):
    r = run("plan", "--elements", n, "--degree", p)
    assert r.returncode == 0, r.stderr
    want = REF_PLAN[(n, p)].split()
    assert r.stdout.split()[:len(want)] == want


def test_plan_2d():
    r = run("plan", "--mesh", "64x64", "--degree", "2")
    assert r.returncode == 0 and "n_dof=16641" in r.stdout and "tree_depth=13" in r.stdout


@pytest.mark.parametrize("argv", [["plan", "--elements", "0"], ["plan", "--elements", "4", "--degree", "5"],
                                  ["plan", "--mesh", "4x"], ["plan"]])
def test_usage_errors_exit_1(argv):
    assert run(*argv).returncode == 1


@pytest.mark.gpu
def test_verify_and_solve_on_gpu(tmp_path, cuda_ok):
    assert cli.main(["verify", "--elements", "200", "--degree", "2"]) == 0
    assert cli.main(["solve", "--mesh", "8x8", "--degree", "2", "--out", str(tmp_path)]) == 0
    assert (tmp_path / "solution.txt").exists()
    assert cli.main(["bench", "--mesh", "32x32", "--degree", "1", "--nrhs", "4",
                     "--repeats", "2", "--out", str(tmp_path / "b.csv")]) == 0
