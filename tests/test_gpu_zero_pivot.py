"""Zero-pivot detection on every front path, against the C port of the reference.

engine.py:527-530 (factorize_nested_loops) raises ZeroPivotError(front, pivot)
at the FIRST pivot in pivot order with |a(z,z)| <= 1e-14 max|A| (engine.py:74);
_extract_factors re-checks every pivot (engine.py:155-159).  A DOF whose row
and column are zero in every element matrix keeps an exactly-zero pivot
through all earlier eliminations, so the failing (node, pivot) pair is exact
on both sides.  The oracle (tf_oracle.c, bitwise = the reference) gives the
expected pair; the GPU must report the same one, including when several
fronts of one level fail (earliest pivot-order position wins) and on the
large-front kernels (diag32 / diag64 / lookahead / root dataflow).
"""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200 import device
from paper_2306_08994_b200.fem import ElementSystem, FrontSet


def zeroed_problem(shape, targets_fn, p=1):
    mesh = tf.TensorMesh(shape, p)
    base = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = tf.build_elimination_tree(base, n_dof=mesh.n_dof)
    plan = tf.symbolic_eliminate(tree, None)
    targets = targets_fn(plan)
    vals = np.broadcast_to(base.values, (len(base),) + base.values.shape).copy()
    for g in targets:
        e, a = np.nonzero(base.dofs == g)
        vals[e, a, :] = 0.0
        vals[e, :, a] = 0.0
    fs = FrontSet(base.dofs, vals)
    peak = tf.assemble_system(mesh, "one").peak
    system = ElementSystem(mesh.n_dof, fs, np.zeros(mesh.n_dof), peak=peak)
    tree2 = tf.build_elimination_tree(fs, n_dof=mesh.n_dof)
    return mesh, fs, system, tf.symbolic_eliminate(tree2, system), targets


def pivot_at(plan, level, front, col):
    """Global index of pivot `col` (clamped to the front's k) of `front` at `level`."""
    lt = plan.native.levels[level]
    col = min(col, int(lt.front_k()[front]) - 1)
    return int(plan.native.pivot_order[int(lt.piv_off[front]) + col])


def expected(mesh, fs):
    from oracle.tfo import OracleFactors
    o = OracleFactors(mesh.n_dof, fs.dofs, fs.values)
    assert o.zero_pivot is not None
    return o.zero_pivot


CASES = {
    # (shape, targets(plan)) — levels counted from the top (-1 = root)
    "mid_level_k64": ((256, 256), lambda P: [pivot_at(P, P.n_levels - 5, 1, 40)]),
    "lookahead_level": ((256, 256), lambda P: [pivot_at(P, P.n_levels - 3, 2, 100)]),
    "root_last_pivot": ((256, 256), lambda P: [int(P.native.pivot_order[-1])]),
    "root_middle": ((256, 256), lambda P: [pivot_at(P, P.n_levels - 1, 0, 130)]),
    "two_fronts_one_level": ((256, 256), lambda P: [pivot_at(P, P.n_levels - 4, 3, 5),
                                                    pivot_at(P, P.n_levels - 4, 1, 60)]),
    "small_level_two_fronts": ((64, 64), lambda P: [pivot_at(P, 4, 9, 1), pivot_at(P, 4, 200, 0)]),
    "leaf_and_root": ((128, 128), lambda P: [int(P.native.pivot_order[-1]),
                                             pivot_at(P, 6, 17, 2)]),
    "3d_upper": ((16, 16, 16), lambda P: [pivot_at(P, P.n_levels - 3, 1, 100)]),
}


def run_case(case):
    shape, fn = CASES[case]
    mesh, fs, system, plan, targets = zeroed_problem(shape, fn)
    front, pivot = expected(mesh, fs)
    assert pivot in targets
    with pytest.raises(tf.ZeroPivotError) as ei:
        tf.run_sequential(plan, tf.init_state(system, plan))
    assert (ei.value.front, ei.value.pivot) == (front, pivot)


@pytest.fixture(params=["default", "large"])
def path(request, cuda_ok):
    old = device.set_small_front_limit(1 if request.param == "large" else 112)
    yield request.param
    device.set_small_front_limit(old)


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(CASES))
def test_zero_pivot_matches_reference(case, path):
    run_case(case)


_SUB = r"""
import sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import test_gpu_zero_pivot as T
for c in sorted(T.CASES):
    T.run_case(c)
print("ok")
"""


@pytest.mark.gpu
def test_zero_pivot_lookahead_paths(cuda_ok):
    """Narrow (64-column) lookahead super-blocks on every k > 64 level with
    <= 64 fronts, and the lookahead path for the root instead of the dataflow
    kernel (fresh process: the widths are read once from the environment)."""
    import os
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, TFB_LOOKAHEAD_COLS="64", TFB_LOOKAHEAD_ROOT_COLS="64",
               TFB_ROOT_DATAFLOW="0")
    out = subprocess.run([sys.executable, "-c", _SUB.format(root=str(root), tests=str(root / "tests"))],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-3000:]
    assert out.stdout.strip().endswith("ok")


def test_oracle_zero_pivot_cases_target_the_zeroed_dofs():
    """CPU: each case's zeroed DOF is where the reference arithmetic fails."""
    for case in ("two_fronts_one_level", "small_level_two_fronts", "leaf_and_root"):
        shape, fn = CASES[case]
        mesh, fs, system, plan, targets = zeroed_problem(shape, fn)
        front, pivot = expected(mesh, fs)
        pos = {int(g): i for i, g in enumerate(plan.native.pivot_order)}
        assert pivot == min(targets, key=lambda g: pos[g])
        assert plan.locate_pivot(pos[pivot]) == (front, pivot)
