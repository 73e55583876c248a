"""The CPU baseline's closed-form work model (oracle/workmodel.py) equals the
native plan's per-front shapes and the reference's task counts."""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden
from oracle import workmodel as W


@pytest.mark.parametrize("ns,p", [((8, 8), 1), ((64, 64), 2), ((256, 256), 1), ((16, 16, 16), 1),
                                  ((8, 8, 8), 2), ((1024,), 1), ((32, 32), 3)])
def test_shapes_equal_native_plan(ns, p):
    mesh = tf.TensorMesh(ns, p) if len(ns) > 1 else tf.Mesh(ns[0], p)
    fr = tf.sort_fronts(tf.generate_fronts(mesh))
    plan = tf.symbolic_eliminate(tf.build_elimination_tree(fr, n_dof=mesh.n_dof))
    shapes = W.level_shapes(ns, p)
    assert len(shapes) == plan.n_levels
    for lt, (m, k) in zip(plan.native.levels, shapes):
        assert np.array_equal(lt.front_m(), m) and np.array_equal(lt.front_k(), k)
    lu = sum(s["lu_flops"] for s in plan.level_stats())
    assert W.workload(ns, p)["lu_task_flops"] == lu


def test_task_count_equals_reference_2d():
    """2D: the dense-front LU count is the reference's Division+Multiplication+
    Subtraction count (golden from the reference's own task graph)."""
    g = golden("2d_8x8_p2")
    from collections import Counter
    w = W.workload((8, 8), 2)
    n_cells = int(g["n_cells"])
    assert w["lu_task_flops"] + n_cells == int(g["fnf_n_tasks"])
