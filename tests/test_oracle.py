"""The CPU oracle is pinned to the reference's golden vectors before it is trusted."""
import numpy as np
import pytest

from conftest import golden, golden_names
from oracle import restate
from oracle.mesh_nd import element_matrix, tensor_mesh
from oracle.tfo import OracleFactors


@pytest.mark.parametrize("name", golden_names())
def test_c_oracle_bitwise_equals_reference(name):
    g = golden(name)
    o = OracleFactors(int(g["n_dof"]), g["elem_dofs"], g["elem_matrix"])
    a = o.arrays()
    assert np.array_equal(a["pivot_order"], g["pivot_order"])
    u, l = o.dicts()
    assert len(u) == int(g["u_count"]) and len(l) == int(g["l_count"])
    for keys, vals, d in ((g["u_keys"], g["u_vals"], u), (g["l_keys"], g["l_vals"], l)):
        got = np.array([d[(int(x), int(y))] for x, y in keys])
        assert np.array_equal(got, vals)  # bitwise
    assert np.array_equal(o.solve(g["rhs"]), g["x"])


@pytest.mark.parametrize("name", [n for n in golden_names() if n != "2d_64x64_p2"])
def test_python_restatement_matches_reference(name):
    g = golden(name)
    if int(g["n_dof"]) > 1200:
        pytest.skip("pure-Python restatement is for small sizes")
    leaves = [tuple(int(x) for x in row) for row in g["elem_dofs"]]
    tree = restate.build_tree(leaves)
    assert [len(l) for l in tree.levels] == list(g["level_sizes"])
    emat = g["elem_matrix"]
    entries = {}
    for dofs in leaves:
        for a, ga in enumerate(dofs):
            for b, gb in enumerate(dofs):
                if ga >= gb:
                    entries[(ga, gb)] = entries.get((ga, gb), 0.0) + emat[a, b]
    _, u, l, order = restate.nested_loops(tree, entries, int(g["n_dof"]))
    assert np.array_equal(np.array(order), g["pivot_order"])
    got = np.array([u[(int(x), int(y))] for x, y in g["u_keys"]])
    assert np.array_equal(got, g["u_vals"])
    assert np.array_equal(restate.solve(u, l, order, g["rhs"]), g["x"])


@pytest.mark.parametrize("name", golden_names())
def test_mesh_generator_restatement(name):
    g = golden(name)
    dims = tuple(int(x) for x in g["dims"])
    n_dof, elems, _ = tensor_mesh(dims, int(g["degree"]))
    assert n_dof == int(g["n_dof"])
    assert np.array_equal(np.array(elems, dtype=np.int32), g["elem_dofs"])
    assert np.array_equal(element_matrix(dims, int(g["degree"])), g["elem_matrix"])


@pytest.mark.parametrize("name", ["1d_n1_p1", "1d_n2_p1", "2d_2x2_p1", "1d_n5_p3", "2d_5x3_p1",
                                  "3d_2x2x2_p1", "2d_8x8_p1"])
def test_fnf_restatement_matches_reference(name):
    g = golden(name)
    leaves = [tuple(int(x) for x in row) for row in g["elem_dofs"]]
    tree = restate.build_tree(leaves)
    lower = set()
    for dofs in leaves:
        for ga in dofs:
            for gb in dofs:
                if ga >= gb:
                    lower.add((ga, gb))
    plan = restate.symbolic(tree, lower, int(g["n_dof"]))
    tasks, succs = restate.task_graph(plan)
    assert len(tasks) == int(g["fnf_n_tasks"])
    assert sum(len(s) for s in succs) == int(g["fnf_n_edges"])
    cls = restate.fnf_classes(tasks, succs)
    widths = np.bincount(cls)[1:]
    assert np.array_equal(widths, g["fnf_widths"])
