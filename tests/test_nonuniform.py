"""Non-uniform element matrices: graded tensor meshes and
per-element densities.  Element matrices are the reference's 1D mass matrices
(fem.py:108-114) of each element's widths, kron'd, times the density; the GPU
factor/solve must match the C port of the reference arithmetic on the same
per-element values."""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200.fem import element_mass_matrix


def graded(n, power=1.7):
    x = np.linspace(0.0, 1.0, n + 1) ** power
    x[-1] = 1.0
    return x


def test_graded_element_values_are_kron_of_1d_matrices():
    nodes = (graded(6), graded(4, 1.3))
    mesh = tf.TensorMesh((6, 4), 2, nodes=nodes)
    vals = mesh.element_values()
    coords = mesh.element_coords()
    for e in (0, 5, 17, 23):
        cx, cy = coords[e]
        mx = element_mass_matrix(nodes[0][cx + 1] - nodes[0][cx], 2)
        my = element_mass_matrix(nodes[1][cy + 1] - nodes[1][cy], 2)
        assert np.allclose(vals[e], np.kron(my, mx), rtol=1e-14, atol=0)
    # total mass of the unit square = sum of all entries
    system = tf.assemble_system(mesh, "one")
    assert abs(system.total_entry_sum() - 1.0) < 1e-13
    rho = np.linspace(1.0, 3.0, mesh.n_elements)
    heavy = tf.TensorMesh((6, 4), 2, nodes=nodes, density=rho)
    assert np.allclose(heavy.element_values(), rho[:, None, None] * vals, rtol=1e-15, atol=0)
    with pytest.raises(tf.InvalidGeometryError):
        tf.TensorMesh((3,), 1, nodes=(np.array([0.0, 0.5, 0.4, 1.0]),))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,p,dens", [((96, 64), 1, False), ((48, 40), 2, True),
                                          ((12, 10, 8), 1, True), ((300,), 3, True)])
def test_nonuniform_factor_solve_matches_c_port(shape, p, dens, cuda_ok):
    from oracle.tfo import OracleFactors
    rng = np.random.default_rng(3)
    nodes = tuple(graded(n, 1.0 + 0.3 * a) for a, n in enumerate(shape))
    n_el = int(np.prod(shape))
    mesh = tf.TensorMesh(shape, p, nodes=nodes,
                         density=rng.uniform(0.5, 4.0, n_el) if dens else None)
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = tf.build_elimination_tree(fronts, n_dof=mesh.n_dof)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    f = tf.run_sequential(plan, tf.init_state(system, plan))
    b = rng.standard_normal((mesh.n_dof, 3))
    x = tf.solve(f, b)
    o = OracleFactors(mesh.n_dof, fronts.dofs, fronts.values)
    assert np.array_equal(o.arrays()["pivot_order"], plan.pivot_order_array)
    for j in range(3):
        xr = o.solve(b[:, j])
        assert np.abs(x[:, j] - xr).max() / np.abs(xr).max() <= 1e-10
    r = system.matvec(x) - b
    assert np.abs(r).max() / np.abs(b).max() < 1e-10
