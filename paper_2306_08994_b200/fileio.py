"""On-disk formats of the reference (fileio.py:1-60, used by cli.py:160-221, 324):
Matrix Market coordinate files, one-value-per-line vectors and CSV rows.

Byte-compatible with the reference writers: entries sorted by (row, column),
1-based indices, floats rendered with ``repr(float(v))`` (shortest
round-trip), a trailing newline.  Vectorized for large exports.
"""

from __future__ import annotations

import csv
from pathlib import Path
from typing import Iterable

import numpy as np


def _fmt(v) -> str:
    return repr(float(v))


def _mm_lines(header: str, n_rows: int, n_cols: int, rows, cols, vals) -> str:
    rows = np.asarray(rows, dtype=np.int64)
    cols = np.asarray(cols, dtype=np.int64)
    vals = np.asarray(vals, dtype=np.float64)
    order = np.lexsort((cols, rows))
    body = [f"{int(rows[t])} {int(cols[t])} {_fmt(vals[t])}" for t in order]
    return "\n".join([header, f"{n_rows} {n_cols} {len(body)}"] + body) + "\n"


def write_matrix_market_symmetric(path, system) -> None:
    """Coordinate export of the assembled system, symmetric qualifier, lower
    triangle only (fileio.py:20-27)."""
    keys = list(system.entries.keys())
    rows = [i for i, _ in keys]
    cols = [j for _, j in keys]
    vals = [system.entries[k] for k in keys]
    Path(path).write_text(_mm_lines("%%MatrixMarket matrix coordinate real symmetric",
                                    system.n_dof, system.n_dof, rows, cols, vals))


def write_matrix_market_general(path, n_rows: int, n_cols: int, entries: dict) -> None:
    """Coordinate export of a sparse matrix given as {(i, j): v}, 1-based keys
    (fileio.py:30-39)."""
    keys = list(entries.keys())
    rows = [i for i, _ in keys]
    cols = [j for _, j in keys]
    vals = [entries[k] for k in keys]
    Path(path).write_text(_mm_lines("%%MatrixMarket matrix coordinate real general",
                                    n_rows, n_cols, rows, cols, vals))


def write_vector(path, values: Iterable[float]) -> None:
    """One value per line (fileio.py:42-44)."""
    Path(path).write_text("".join(f"{_fmt(v)}\n" for v in np.asarray(values).ravel()))


def read_vector(path) -> list[float]:
    return [float(x) for x in Path(path).read_text().split()]


def write_csv_rows(path, header: list, rows: list) -> None:
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(header)
        w.writerows(rows)


def factor_exports(factors) -> tuple[dict, dict]:
    """L (unit lower, pivot rows carry 1.0) and U (d on the diagonal,
    d_z * q(z, y) off it) in global coordinates, as cli.py:208-215 builds them."""
    lower = dict(factors.l_entries)
    for z in factors.pivot_order:
        lower[(z, z)] = 1.0
    u = factors.u_entries
    upper = {(z, y): (v if z == y else v * u[(z, z)]) for (z, y), v in u.items()}
    return lower, upper
