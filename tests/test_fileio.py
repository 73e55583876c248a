"""On-disk formats: the CLI exports of the reference
(cli.py:164-221; fileio.py:20-44) against goldens written by the reference
CLI itself (tests/golden/make_fileio_golden.py)."""
from pathlib import Path

import numpy as np
import pytest

from paper_2306_08994_b200 import cli, fileio

GOLD = Path(__file__).resolve().parent / "golden" / "fileio"
CASES = {"1d_n6_p2": ["--elements", "6", "--degree", "2"],
         "1d_n5_p3_sin": ["--elements", "5", "--degree", "3", "--rhs", "sin_pi"]}


def _mm(path):
    lines = Path(path).read_text().splitlines()
    keys = [tuple(int(t) for t in ln.split()[:2]) for ln in lines[2:]]
    vals = np.array([float(ln.split()[2]) for ln in lines[2:]])
    return lines[0], lines[1], keys, vals


@pytest.mark.parametrize("case", sorted(CASES))
def test_generate_byte_identical(case, tmp_path):
    assert cli.main(["generate", *CASES[case], "--out", str(tmp_path)]) == 0
    for f in ("matrix.mtx", "rhs.txt", "manifest.json"):
        assert (tmp_path / f).read_bytes() == (GOLD / case / f).read_bytes(), f


def test_vector_and_csv_writers(tmp_path):
    v = [1.0, -0.1, 1e-300, 12345.678901234567]
    fileio.write_vector(tmp_path / "v.txt", v)
    assert (tmp_path / "v.txt").read_text() == "".join(f"{x!r}\n" for x in v)
    assert fileio.read_vector(tmp_path / "v.txt") == v
    fileio.write_csv_rows(tmp_path / "r.csv", ["a", "b"], [[1, 2.5]])
    assert (tmp_path / "r.csv").read_text().splitlines() == ["a,b", "1,2.5"]
    fileio.write_matrix_market_general(tmp_path / "m.mtx", 3, 3, {(3, 1): 2.0, (1, 1): 1.0})
    assert (tmp_path / "m.mtx").read_text() == (
        "%%MatrixMarket matrix coordinate real general\n3 3 2\n1 1 1.0\n3 1 2.0\n")


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_factorize_and_solve_exports(case, tmp_path, cuda_ok):
    assert cli.main(["factorize", *CASES[case], "--out", str(tmp_path)]) == 0
    assert (tmp_path / "pivot_order.txt").read_bytes() == \
        (GOLD / case / "pivot_order.txt").read_bytes()
    for f in ("L.mtx", "U.mtx"):
        h, dims, keys, vals = _mm(tmp_path / f)
        gh, gdims, gkeys, gvals = _mm(GOLD / case / f)
        assert (h, dims, keys) == (gh, gdims, gkeys), f
        assert np.abs(vals - gvals).max() <= 1e-10 * np.abs(gvals).max(), f
    assert cli.main(["solve", *CASES[case], "--out", str(tmp_path)]) == 0
    x = np.array(fileio.read_vector(tmp_path / "solution.txt"))
    g = np.array(fileio.read_vector(GOLD / case / "solution.txt"))
    assert np.abs(x - g).max() <= 1e-10 * np.abs(g).max()
