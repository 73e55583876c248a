"""Native symbolic layer (tree, pivot order, NodeReorder, active sets) vs the reference."""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden, golden_names, mesh_of


@pytest.mark.parametrize("name", golden_names())
def test_plan_matches_reference(name):
    g = golden(name)
    mesh = mesh_of(g)
    fronts = tf.generate_fronts(mesh)
    assert np.array_equal(fronts.dofs, g["elem_dofs"])
    assert np.array_equal(fronts.values, g["elem_matrix"])
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts))
    assert tuple(tree.level_sizes) == tuple(int(x) for x in g["level_sizes"])
    assert tree.root_id == int(g["root_id"])
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    assert np.array_equal(plan.pivot_order_array, g["pivot_order"])
    assert tf.init_state(system, plan).zero_threshold == float(g["threshold"])
    if int(g["n_dof"]) > 5000:
        return
    ro = plan.reorders
    assert [r.node_id for r in ro] == list(g["reorder_node"])
    cnt = np.array([(len(r.eliminable), len(r.shared), len(r.computed)) for r in ro])
    assert np.array_equal(cnt, g["reorder_counts"])
    assert np.array_equal(np.array([x for r in ro for x in r.eliminable]), g["reorder_elim"])
    assert np.array_equal(np.array([x for r in ro for x in r.shared], dtype=np.int64),
                          g["reorder_shared"].astype(np.int64))
    assert np.array_equal(np.array([len(s.active) for s in plan.steps]), g["active_sizes"])
    assert np.array_equal(np.array([s.node_id for s in plan.steps]), g["step_node"])
    assert len(plan.cells) == int(g["n_cells"])
    assert len(plan.fill_cells) == int(g["n_fill"])


def test_spec_tree_examples():
    """8 fronts -> levels 8,4,2,1; 5 fronts -> 5,3,2,1."""
    for n, sizes in ((8, (8, 4, 2, 1)), (5, (5, 3, 2, 1)), (1, (1,))):
        tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(tf.Mesh(n, 1))))
        assert tree.level_sizes == sizes


def test_spec_pivot_order_n2():
    """mesh(n=2, p=1) pivots (1, 3, 2)."""
    mesh = tf.Mesh(2, 1)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    plan = tf.symbolic_eliminate(tree, tf.assemble_system(mesh, "one"))
    assert plan.pivot_order == (1, 3, 2)


def test_membership_and_nodes_n2():
    """membership [(1,2),(2,1)] at the leaves."""
    mesh = tf.Mesh(2, 1)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    assert [tree.nodes[i].front.membership for i in tree.levels[0]] == [(1, 2), (2, 1)]
    assert tree.nodes[tree.root_id].front.indices == (1, 2, 3)


def test_generate_fronts_membership_kats():
    """SPEC.md:90-92 (fem.py:241-250): shared endpoints count 2, others 1."""
    fr = tf.generate_fronts(tf.Mesh(2, 1))
    assert [f.membership for f in fr] == [(1, 2), (2, 1)]
    assert [f.membership for f in tf.generate_fronts(tf.Mesh(1, 3))] == [(1, 1, 1, 1)]
    assert [f.membership for f in tf.generate_fronts(tf.Mesh(3, 2))] == \
        [(1, 1, 2), (2, 1, 2), (2, 1, 1)]
    # against the reference's own generate_fronts for every 1D golden mesh
    for name in golden_names():
        g = golden(name)
        if len(g["dims"]) != 1:
            continue
        n, p = int(g["dims"][0]), int(g["degree"])
        mem = [f.membership for f in tf.generate_fronts(tf.Mesh(n, p))]
        ref = [(1 if e == 0 else 2,) + (1,) * (p - 1) + (1 if e == n - 1 else 2,) for e in range(n)]
        assert mem == ref
    # sorting keeps it; 2D/3D: number of elements holding the DOF
    f2 = tf.sort_fronts(tf.generate_fronts(tf.TensorMesh((2, 2), 1)))
    assert sorted(f2[0].membership) == [1, 2, 2, 4]
    # caller-built fronts keep their own membership
    user = tf.Front(0, (1, 2), (3, 1), (False, False), np.eye(2))
    assert tf.build_elimination_tree([user]).fronts[0].membership == (3, 1)


def test_element_and_assembly_kats():
    """SPEC.md:63, 73, 81."""
    assert np.allclose(tf.element_mass_matrix(1.0, 1), np.array([[2, 1], [1, 2]]) / 6, atol=1e-16)
    from paper_2306_08994_b200.fem import element_load_vector
    assert np.allclose(element_load_vector(1.0, 1, lambda x: 1.0, 0.0), [0.5, 0.5])
    s = tf.assemble_system(tf.Mesh(2, 1), "one")
    assert s.entry(2, 2) == 0.33333333333333337


def test_empty_and_invalid_inputs():
    with pytest.raises(tf.EmptyInputError):
        tf.sort_fronts([])
    with pytest.raises(tf.EmptyInputError):
        tf.build_elimination_tree([])
    with pytest.raises(tf.UnsupportedDegreeError):
        tf.Mesh(4, 4)
    with pytest.raises(tf.InvalidGeometryError):
        tf.Mesh(0, 1)
    with pytest.raises(tf.InvalidGeometryError):
        tf.TensorMesh((4, 0), 1)


def test_large_tensor_plan_shapes():
    """2D 256^2 p=1: level table maxima follow the nested-dissection model."""
    mesh = tf.TensorMesh((256, 256), 1)
    tree = tf.build_elimination_tree(tf.generate_fronts(mesh))
    plan = tf.symbolic_eliminate(tree)
    assert plan.native.n_pivots == mesh.n_dof
    ms = [lt.max_m for lt in plan.native.levels]
    ks = [lt.max_k for lt in plan.native.levels]
    assert ms[:6] == [4, 6, 9, 13, 19, 27] and ks[-1] == ms[-1] == 257
    for lt in plan.native.levels:
        assert lt.n_patterns <= 40  # structured mesh: a handful of shape classes per level


def test_scatter_tables_match_maps():
    """TF_PAT_SOFF tables (shared-memory extend-add targets) agree with the
    forward maps: entry (a, b) of source c lands at the layout position of
    front cell (max(map[a], map[b]), min(...)) in [pivot rows packed | L21
    rows of stride kp+1 | Schur block packed]; the Schur part is the update
    slot's packed order; fronts above order 232 carry no table."""
    from paper_2306_08994_b200 import _lib
    mesh = tf.TensorMesh((24, 20), 2)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
    plan = tf.symbolic_eliminate(tree, tf.assemble_system(mesh, "one"))
    checked = 0
    for lt in plan.native.levels:
        for row in lt.pat:
            m, k, kp = int(row[_lib.PAT_M]), int(row[_lib.PAT_K]), int(row[_lib.PAT_KP])
            soff = int(row[_lib.PAT_SOFF])
            if m > 232:
                assert soff == -1
                continue
            ks, u, tk = kp + 1, m - k, k * (k + 1) // 2
            seen = set()
            pos = soff
            for c in range(int(row[_lib.PAT_NSRC])):
                ln = int(row[_lib.PAT_LEN0 + c])
                fwd = lt.maps[int(row[_lib.PAT_OFF0 + c]):][:ln]
                for a in range(ln):
                    for b in range(a + 1):
                        R, C = max(fwd[a], fwd[b]), min(fwd[a], fwd[b])
                        if R < k:
                            want = R * (R + 1) // 2 + C
                        elif C < k:
                            want = tk + (R - k) * ks + C
                        else:
                            want = tk + u * ks + (R - k) * (R - k + 1) // 2 + (C - k)
                        assert lt.maps[pos] == want
                        if c == 0:
                            assert want not in seen  # one source never hits a cell twice
                            seen.add(want)
                        pos += 1
                        checked += 1
    assert checked > 1000
