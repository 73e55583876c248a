"""The level schedule is a valid linearization of the reference's Diekert graph.

The package executes one Foata class of the FRONT-granularity trace per
launch sequence: class L = tree level L (schedule.py docstring).  That is
valid for the reference's ATOMIC trace (tasks.py:162-252) iff every
dependency edge J1-J4 goes from a task of level <= the level of its target,
where a Division / Multiplication / Subtraction of pivot z runs at the level
of the node that eliminates z, and the Assertion of cell (x, y) runs when
that cell is final, i.e. at the level of whichever of x, y is eliminated
first.  Inside one level the kernels respect the remaining (same-level)
edges by construction: per front the pivots run in pivot order, and the
extend-add of a child happens before any pivot of the parent.

The atomic graph here is the restatement in oracle/restate.py, itself pinned
to the reference (task / edge counts and Foata widths, tests/test_oracle.py).
"""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden, golden_names, mesh_of
from oracle import restate

SMALL = [n for n in golden_names() if int(golden(n)["n_dof"]) <= 400]


def restated(g):
    leaves = [tuple(int(x) for x in row) for row in g["elem_dofs"]]
    tree = restate.build_tree(leaves)
    lower = {(ga, gb) for dofs in leaves for ga in dofs for gb in dofs if ga >= gb}
    plan = restate.symbolic(tree, lower, int(g["n_dof"]))
    return tree, plan


@pytest.mark.parametrize("name", SMALL)
def test_every_atomic_edge_is_level_nondecreasing(name):
    g = golden(name)
    tree, plan = restated(g)
    level_of_node = {nid: L for L, ids in enumerate(tree.levels) for nid in ids}
    pos = {z: i for i, z in enumerate(plan.pivot_order)}
    piv_level = {z: level_of_node[f] for (f, z, _) in plan.steps}
    tasks, succs = restate.task_graph(plan)

    def level(t):
        kind, f, z, x, y = t
        if kind == restate.ASSERT:
            return piv_level[x if pos[x] <= pos[y] else y]
        return level_of_node[f]

    lv = [level(t) for t in tasks]
    n_edges = 0
    for u, outs in enumerate(succs):
        for v in outs:
            assert lv[u] <= lv[v], (tasks[u], tasks[v], lv[u], lv[v])
            n_edges += 1
    assert n_edges == sum(len(s) for s in succs) > 0 or len(tasks) == 1

    # the package's front-granularity FNF: one class per tree level, same node ids
    mesh = mesh_of(g)
    ptree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    pplan = tf.symbolic_eliminate(ptree, tf.assemble_system(mesh, "one"))
    sched = tf.compute_fnf(pplan)
    assert [list(c) for c in sched.classes] == tree.levels
    # pivot order runs level by level (the launch order of the classes)
    lev = [piv_level[int(z)] for z in pplan.pivot_order]
    assert lev == sorted(lev)


@pytest.mark.parametrize("name", ["1d_n13_p2", "2d_5x3_p1", "3d_2x2x2_p1"])
def test_atomic_fnf_classes_fit_inside_level_windows(name):
    """Executing levels in order, and inside a level the atomic Foata classes in
    order, never runs a task before one of its predecessors (a topological
    order of the reference's graph).  In 1D the atomic classes straddle at most
    two adjacent levels; in 2D/3D they can span more, which
    the level schedule does not need."""
    g = golden(name)
    tree, plan = restated(g)
    level_of_node = {nid: L for L, ids in enumerate(tree.levels) for nid in ids}
    pos = {z: i for i, z in enumerate(plan.pivot_order)}
    piv_level = {z: level_of_node[f] for (f, z, _) in plan.steps}
    tasks, succs = restate.task_graph(plan)
    cls = restate.fnf_classes(tasks, succs)
    lv = []
    for kind, f, z, x, y in tasks:
        lv.append(piv_level[x if pos[x] <= pos[y] else y] if kind == restate.ASSERT
                  else level_of_node[f])
    if len(g["dims"]) == 1:
        by_class = {}
        for c, L in zip(cls, lv):
            by_class.setdefault(c, set()).add(L)
        for c, levels in by_class.items():
            assert max(levels) - min(levels) <= 1, (c, levels)
    # level-major order sorted by (level, FNF class) is a topological order
    order = sorted(range(len(tasks)), key=lambda t: (lv[t], cls[t]))
    where = np.empty(len(tasks), dtype=np.int64)
    where[order] = np.arange(len(tasks))
    for u, outs in enumerate(succs):
        for v in outs:
            assert where[u] < where[v]
