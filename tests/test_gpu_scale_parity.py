"""GPU parity at the BASELINE sizes, on the DEFAULT kernel selection.

The goldens (tests/golden/scale_*.npz, made by tests/golden/make_scale_golden.py)
come from the C port of the reference arithmetic (oracle/tf_oracle.c), which
tests/test_oracle.py pins bitwise to the reference's own outputs.  At these
sizes every production kernel runs with its production thresholds: the
shared-memory small fronts, blocked large fronts with DMMA trailing updates,
lookahead super-blocks (k > 256 with <= 64 fronts), the root dataflow kernel,
the narrow / wave / split single-RHS sweeps and the 64-column wave sweeps.

Contract (BASELINE north_star): identical pivot order;
factor samples within 1e-10 of the reference normwise (max|dU|/max|U_ref|);
solution columns within 1e-10 relative (inf-norm) per right-hand side.
"""
import hashlib
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest

from conftest import GOLDEN

FACTOR_TOL = 1e-10
SOLVE_TOL = 1e-10
ROOT = Path(__file__).resolve().parents[1]
SCALE = sorted(p.stem[len("scale_"):] for p in GOLDEN.glob("scale_*.npz"))


def load(name):
    return dict(np.load(GOLDEN / f"scale_{name}.npz"))


def build(g):
    import paper_2306_08994_b200 as tf
    from paper_2306_08994_b200.tree import EliminationTree
    dims = tuple(int(x) for x in g["dims"])
    mesh = tf.TensorMesh(dims, int(g["degree"]))
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = EliminationTree(fronts, n_dof=mesh.n_dof, keep_lists=True)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    return mesh, system, plan


def check(g, plan, factors, solve_block, single=True):
    po = np.ascontiguousarray(plan.pivot_order_array, dtype="<i4")
    assert len(po) == int(g["n_piv"])
    assert np.array_equal(po[:len(g["pivot_order_head"])], g["pivot_order_head"])
    assert hashlib.sha256(po.tobytes()).digest() == bytes(g["pivot_order_sha256"])
    du = np.abs(factors.u_values(g["u_keys"]) - g["u_vals"]).max() / float(g["u_absmax"])
    dl = np.abs(factors.l_values(g["l_keys"]) - g["l_vals"]).max() / float(g["l_absmax"])
    dd = np.abs(factors.pivot_values(g["diag_pos"]) - g["diag_vals"]).max() / float(g["u_absmax"])
    assert du <= FACTOR_TOL and dl <= FACTOR_TOL and dd <= FACTOR_TOL, (du, dl, dd)
    n, nrhs, rs = int(g["n_dof"]), int(g["nrhs"]), int(g["row_stride"])
    B = np.random.default_rng(0).standard_normal((n, nrhs))
    X = solve_block(B)
    errs = {}
    for j in g["cols"]:
        ref = g[f"x{int(j)}_rows"]
        errs[int(j)] = np.abs(X[::rs, int(j)] - ref).max() / float(g[f"x{int(j)}_absmax"])
    if single:
        x0 = solve_block(np.ascontiguousarray(B[:, 0]))
        errs["single"] = np.abs(x0[::rs] - g["x0_rows"]).max() / float(g["x0_absmax"])
    assert max(errs.values()) <= SOLVE_TOL, errs
    return du, dl, errs


@pytest.mark.gpu
@pytest.mark.parametrize("name", SCALE)
def test_scale_parity_default_kernels(name, cuda_ok):
    import paper_2306_08994_b200 as tf
    g = load(name)
    mesh, system, plan = build(g)
    factors = tf.run_sequential(plan, tf.init_state(system, plan))
    check(g, plan, factors, lambda B: tf.solve(factors, B))


_VARIANT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import paper_2306_08994_b200 as tf
from paper_2306_08994_b200 import device
if {limit}:
    device.set_small_front_limit({limit})
import test_gpu_scale_parity as T
g = T.load({name!r})
mesh, system, plan = T.build(g)
f = tf.run_sequential(plan, tf.init_state(system, plan))
print("ok", T.check(g, plan, f, lambda B: tf.solve(f, B)))
"""

VARIANTS = {
    # CTA-per-front sweeps on every level with k > 64 (production: >= 256 fronts)
    "front": dict(TFB_FRONT_SOLVE="2", TFB_FRONT_MIN_FRONTS="1"),
    # split backward sweep (update-row chunks + pivot rows) on every k > 64 level
    "split": dict(TFB_FRONT_SOLVE="0", TFB_SPLIT_SOLVE="2"),
    # every non-leaf level through the blocked large-front kernels
    "large": dict(_LIMIT="1"),
}


@pytest.mark.gpu
@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("name", [n for n in SCALE if n in ("2d_1024x1024_p1", "3d_32x32x32_p1",
                                                            "2d_256x256_p1")])
def test_scale_parity_forced_variants(name, variant, cuda_ok):
    env = dict(os.environ)
    env.update({k: v for k, v in VARIANTS[variant].items() if not k.startswith("_")})
    limit = int(VARIANTS[variant].get("_LIMIT", "0"))
    code = _VARIANT.format(root=str(ROOT), tests=str(ROOT / "tests"), limit=limit, name=name)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert out.stdout.startswith("ok"), out.stdout[-2000:]
