"""Native atomic Foata normal form (tf_atomic_fnf) against the reference's own
task graph + compute_fnf (tasks.py:162-252, schedule.py:60-82).

Pinned two ways: the goldens' task/edge counts and class widths, written by
tests/golden/make_golden.py from the reference itself, and the Python
restatement of the graph (oracle/restate.py, itself pinned in test_oracle.py)
for the class kind sets and for meshes whose goldens carry no FNF.
"""
import time

import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden, golden_names
from oracle import restate
from paper_2306_08994_b200.tree import EliminationTree


def _plan(g):
    dims = [int(d) for d in g["dims"]]
    p = int(g["degree"])
    mesh = tf.Mesh(dims[0], p) if len(dims) == 1 else tf.TensorMesh(tuple(dims), p)
    system = tf.assemble_system(mesh, "one")
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)), n_dof=mesh.n_dof)
    return tf.symbolic_eliminate(tree, system)


def _restated(g):
    leaves = [tuple(int(x) for x in row) for row in g["elem_dofs"]]
    tree = restate.build_tree(leaves)
    lower = {(a, b) for dofs in leaves for a in dofs for b in dofs if a >= b}
    tasks, succs = restate.task_graph(restate.symbolic(tree, lower, int(g["n_dof"])))
    cls = restate.fnf_classes(tasks, succs)
    kinds = [set() for _ in range(max(cls))]
    for t, c in zip(tasks, cls):
        kinds[c - 1].add(t[0])
    return len(tasks), sum(len(s) for s in succs), np.bincount(cls)[1:], kinds


@pytest.mark.parametrize("name", [n for n in golden_names() if "fnf_widths" in golden(n)])
def test_atomic_fnf_matches_reference_goldens(name):
    g = golden(name)
    s = tf.compute_atomic_fnf(_plan(g))
    assert s.n_tasks == int(g["fnf_n_tasks"])
    assert s.n_edges == int(g["fnf_n_edges"])
    assert np.array_equal(np.array(s.widths), g["fnf_widths"])


@pytest.mark.parametrize("name", ["2d_5x3_p1", "3d_2x2x2_p1", "3d_3x2x2_p2", "3d_4x4x4_p1",
                                  "2d_7x6_p3", "1d_n64_p3"])
def test_atomic_fnf_matches_restated_graph(name):
    g = golden(name)
    n_tasks, n_edges, widths, kinds = _restated(g)
    s = tf.compute_atomic_fnf(_plan(g))
    assert (s.n_tasks, s.n_edges) == (n_tasks, n_edges)
    assert np.array_equal(np.array(s.widths), widths)
    assert [{int(k) for k in ks} for ks in s.class_kinds] == kinds
    assert s.n_cells == len(_plan(g).cells)


def test_atomic_fnf_cfg1_stats_and_csv():
    mesh = tf.Mesh(1024, 1)
    system = tf.assemble_system(mesh, "one")
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)), n_dof=mesh.n_dof)
    s = tf.compute_atomic_fnf(tf.symbolic_eliminate(tree, system))
    st = tf.schedule_stats(s)
    assert st.n_classes == 50 and st.max_width == max(s.widths)
    csv = tf.schedule_stats_csv(s).splitlines()
    assert csv[0] == "class_index,kind_set,size" and len(csv) == 51
    assert sum(int(r.split(",")[2]) for r in csv[1:]) == s.n_tasks == 15181


def test_atomic_fnf_cfg2_scale():
    """cfg2 (2D Q2 64x64): the reference's graph is ~57 GB; streamed here in seconds."""
    g = golden("2d_64x64_p2")
    plan = _plan(g)
    t0 = time.perf_counter()
    s = tf.compute_atomic_fnf(plan)
    dt = time.perf_counter() - t0
    assert s.n_tasks == s.n_cells + sum(
        len(st.active) + 2 * len(st.active) ** 2 for st in plan.steps)
    assert s.n_tasks > 7e7 and sum(s.widths) == s.n_tasks
    assert dt < 60


def test_atomic_fnf_needs_node_lists():
    mesh = tf.TensorMesh((8, 8), 1)
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = EliminationTree(fronts, n_dof=mesh.n_dof, keep_lists=False)
    plan = tf.symbolic_eliminate(tree, tf.assemble_system(mesh, "one"))
    with pytest.raises(RuntimeError):
        tf.compute_atomic_fnf(plan)
