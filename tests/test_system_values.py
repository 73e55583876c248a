"""The factorization starts from the system passed to init_state (engine.py:67-75).

ADVICE r1: the GPU used to factor the leaf fronts' element matrices whatever
the system said.  Now `leaf_values` seeds the leaves from the system: the
element matrices when the system is the ElementSystem of the plan's own
fronts, else each stored entry on the first leaf front holding it; a system
the fronts cannot represent raises ContractViolationError.
"""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200.engine import leaf_values


def assembled(fronts, vals):
    ent = {}
    for e in range(len(fronts)):
        d = fronts.dofs_of(e)
        for a, ga in enumerate(d):
            for b, gb in enumerate(d):
                if ga >= gb:
                    k = (int(ga), int(gb))
                    ent[k] = ent.get(k, 0.0) + float(vals[e][a, b])
    return ent


@pytest.mark.parametrize("n,p", [(8, 2), (13, 3), (1024, 1)])
def test_dict_system_split_over_leaves_is_exact(n, p):
    mesh = tf.Mesh(n, p)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    system = tf.assemble_system(mesh, "one")
    v = leaf_values(tree.fronts, system)
    assert assembled(tree.fronts, v) == system.entries  # bitwise: one leaf per entry


def test_element_system_uses_element_matrices():
    mesh = tf.TensorMesh((8, 8), 1)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    system = tf.assemble_system(mesh, "one")
    assert np.shares_memory(leaf_values(tree.fronts, system), tree.fronts.values)
    system.add(5, 5, 0.25)  # edited: no longer the element sum
    v = leaf_values(tree.fronts, system)
    ent = assembled(tree.fronts, v)
    assert ent == system.entries


def test_unrepresentable_system_raises():
    mesh = tf.TensorMesh((4, 4), 1)
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    system = tf.GlobalSystem(mesh.n_dof, dict(tf.assemble_system(mesh, "one").entries))
    system.add(mesh.n_dof, 1, 1.0)  # couples opposite corners: in no element
    with pytest.raises(tf.ContractViolationError):
        leaf_values(tree.fronts, system)
    other = tf.assemble_system(tf.TensorMesh((4, 4), 2), "one")
    with pytest.raises(tf.ContractViolationError):
        leaf_values(tree.fronts, other)


@pytest.mark.gpu
def test_edited_system_is_what_gets_factorized(cuda_ok):
    from oracle.tfo import OracleFactors
    mesh = tf.TensorMesh((16, 16), 2)
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = tf.build_elimination_tree(fronts)
    system = tf.assemble_system(mesh, "one")
    for g in (3, 40, 200, 1000):
        system.add(g, g, 0.5 * system.entry(g, g))
    plan = tf.symbolic_eliminate(tree, system)
    f = tf.run_sequential(plan, tf.init_state(system, plan))
    b = np.random.default_rng(2).standard_normal(mesh.n_dof)
    x = tf.solve(f, b)
    r = system.matvec(x) - b
    assert np.abs(r).max() / np.abs(b).max() < 1e-12
    # the C port of the reference on the same entries (split the same way)
    vals = leaf_values(tree.fronts, system)
    o = OracleFactors(mesh.n_dof, tree.fronts.dofs, vals)
    xr = o.solve(b)
    assert np.abs(x - xr).max() / np.abs(xr).max() <= 1e-10
