"""Generate at-scale golden vectors with the C port of the reference arithmetic.

TEST INFRASTRUCTURE.  The reference's own Python path cannot run at these
sizes (cfg3 symbolic ~1 h / 40 GB, task graph ~4e10
tasks), so the goldens come from `oracle/tf_oracle.c`, the C port of
`factorize_nested_loops` + `solve` (engine.py:500-552, 468-493) that
tests/test_oracle.py pins BITWISE to the reference on all 19 reference
goldens (incl. cfg2, 16,641 DoF).  Problem generation is the oracle's own
restatement (oracle/mesh_nd.py), not the product package.

    python tests/golden/make_scale_golden.py 2d_1024x1024_p1 3d_32x32x32_p1 ...

Per instance it stores (tests/golden/scale_<name>.npz):
  pivot_order_sha256, n_piv       the whole pivot order, hashed
  u/l counts, absmax, strided key/value samples (stride SAMPLE)
  diag sample (every SAMPLE-th pivot in pivot order)
  RHS block B = default_rng(0).standard_normal((n, NRHS)); for the columns
  in COLS: the oracle solution at every ROW_STRIDE-th row + its full inf-norm
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
from oracle.mesh_nd import element_matrix, tensor_mesh  # noqa: E402
from oracle.tfo import OracleFactors  # noqa: E402

OUT = Path(__file__).resolve().parent
INSTANCES = {
    "2d_1024x1024_p1": ((1024, 1024), 1),  # BASELINE cfg3 (primary degree)
    "3d_32x32x32_p1": ((32, 32, 32), 1),   # 3D at scale (cfg4 is 64^3: ~9 h in the port)
    "2d_512x512_p2": ((512, 512), 2),      # Q2 at scale (cfg3 p=2 halved per axis)
    "2d_256x256_p1": ((256, 256), 1),
}
NRHS = 64
COLS = (0, 31, 63)
SAMPLE = 1009
ROW_STRIDE = 7


def run(name):
    dims, p = INSTANCES[name]
    t0 = time.time()
    n_dof, elems, _ = tensor_mesh(dims, p)
    emat = element_matrix(dims, p)
    dofs = np.asarray(elems, dtype=np.int32)
    t1 = time.time()
    o = OracleFactors(n_dof, dofs, emat)
    t_factor = time.time() - t1
    assert o.status == 0, o.zero_pivot
    a = o.arrays()
    piv = a["pivot_order"]
    out = {
        "dims": np.array(dims, dtype=np.int64), "degree": np.int64(p), "n_dof": np.int64(n_dof),
        "n_piv": np.int64(len(piv)),
        "pivot_order_sha256": np.frombuffer(
            hashlib.sha256(np.ascontiguousarray(piv, dtype="<i4").tobytes()).digest(), np.uint8),
        "pivot_order_head": piv[:4096].copy(),
        "u_count": np.int64(len(a["u_v"]) + len(piv)), "l_count": np.int64(len(a["l_v"])),
        "sample_stride": np.int64(SAMPLE),
    }
    uab = max(np.abs(a["u_v"]).max(initial=0.0), np.abs(a["diag"]).max())
    out["u_absmax"] = np.float64(uab)
    out["l_absmax"] = np.float64(np.abs(a["l_v"]).max(initial=0.0))
    out["u_keys"] = np.stack([a["u_z"][::SAMPLE], a["u_y"][::SAMPLE]], axis=1).astype(np.int32)
    out["u_vals"] = a["u_v"][::SAMPLE].copy()
    out["l_keys"] = np.stack([a["l_x"][::SAMPLE], a["l_z"][::SAMPLE]], axis=1).astype(np.int32)
    out["l_vals"] = a["l_v"][::SAMPLE].copy()
    out["diag_pos"] = np.arange(0, len(piv), SAMPLE, dtype=np.int64)
    out["diag_vals"] = a["diag"][::SAMPLE].copy()
    del a
    B = np.random.default_rng(0).standard_normal((n_dof, NRHS))
    t1 = time.time()
    rows = np.arange(0, n_dof, ROW_STRIDE, dtype=np.int64)
    out["nrhs"] = np.int64(NRHS)
    out["cols"] = np.array(COLS, dtype=np.int64)
    out["row_stride"] = np.int64(ROW_STRIDE)
    for j in COLS:
        x = o.solve(B[:, j])
        out[f"x{j}_rows"] = x[rows].copy()
        out[f"x{j}_absmax"] = np.float64(np.abs(x).max())
    t_solve = (time.time() - t1) / len(COLS)
    out["t_oracle_factor_s"] = np.float64(t_factor)
    out["t_oracle_solve_s"] = np.float64(t_solve)
    np.savez_compressed(OUT / f"scale_{name}.npz", **out)
    print(f"{name}: n_dof={n_dof} pivots={len(piv)} oracle factor {t_factor:.1f}s "
          f"solve {t_solve:.2f}s/col total {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(INSTANCES):
        run(nm)
