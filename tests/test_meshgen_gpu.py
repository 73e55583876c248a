"""GPU mesh generation (csrc/mesh.cu) is bitwise the host generator."""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf

SHAPES = [((8,), 1), ((13,), 3), ((5, 3), 2), ((64, 64), 1), ((17, 9), 1), ((6, 5, 4), 2),
          ((16, 16, 16), 1), ((31, 2), 3), ((1024, 1024), 1)]


@pytest.mark.gpu
@pytest.mark.parametrize("shape,p", SHAPES)
def test_device_table_equals_host(shape, p, cuda_ok):
    from paper_2306_08994_b200.meshgen import element_table_device
    mesh = tf.TensorMesh(shape, p)
    dofs, order = element_table_device(mesh)
    assert np.array_equal(dofs.cpu().numpy(), mesh.element_table())
    coords = mesh.element_coords()
    lin = coords[:, 0].astype(np.int64)
    stride = 1
    for a in range(1, mesh.dim):
        stride *= shape[a - 1]
        lin += coords[:, a] * stride
    assert np.array_equal(order.cpu().numpy(), lin)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,p", [((12, 7), 2), ((9, 8, 5), 1), ((40,), 3)])
def test_device_values_equal_host_and_factor_identically(shape, p, cuda_ok):
    from paper_2306_08994_b200.meshgen import element_table_device, element_values_device
    from paper_2306_08994_b200.device import DevicePlan
    rng = np.random.default_rng(1)
    nodes = tuple(np.concatenate([[0.0], np.sort(rng.uniform(0, 1, n - 1)), [1.0]]) for n in shape)
    mesh = tf.TensorMesh(shape, p, nodes=nodes, density=rng.uniform(0.5, 2.0, int(np.prod(shape))))
    dofs, order = element_table_device(mesh)
    vals = element_values_device(mesh, order)
    assert np.array_equal(vals.cpu().numpy(), mesh.element_values())
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    plan = tf.symbolic_eliminate(tf.build_elimination_tree(fronts, n_dof=mesh.n_dof))
    thr = tf.init_state(tf.assemble_system(mesh, "one"), plan).zero_threshold
    a = DevicePlan(plan, plan.tree.fronts)
    b = DevicePlan(plan, plan.tree.fronts, values=vals)   # device-generated, no upload
    import torch
    rhs = torch.from_numpy(rng.standard_normal(mesh.n_dof)).cuda()
    xs = []
    for dp in (a, b):
        dp.factor(thr)
        x = torch.empty_like(rhs)
        dp.solve_into(rhs, x)
        xs.append(x.cpu().numpy())
    assert np.array_equal(xs[0], xs[1])  # same element values, same arithmetic
