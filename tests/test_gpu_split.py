"""Concurrent top slices (DevicePlan.split_top): the levels with few large
fronts are factored as independent subtree halves on separate streams, each
with its own lookahead streams.  Every front sees the same kernels in the
same order, so factors and solutions are bitwise those of the one-stream
schedule (which is itself checked against the C port elsewhere)."""
import numpy as np
import pytest
import torch

import paper_2306_08994_b200 as tf


@pytest.mark.gpu
@pytest.mark.parametrize("shape,p", [((512, 512), 1), ((20, 20, 20), 1), ((16, 16, 16), 1), ((256, 256), 2)])
def test_split_top_bitwise(shape, p, cuda_ok):
    mesh = tf.TensorMesh(shape, p)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    state = tf.init_state(system, plan)
    dp = tf.compile_execution(plan, None, state)
    b = torch.from_numpy(np.random.default_rng(2).standard_normal(mesh.n_dof)).to(dp.device)
    out = {}
    for H in (1, 2):
        dp.split_top = H
        if H == 2:
            assert dp._split_plan() is not None, "expected concurrent top slices on this tree"
        for t in dp.factors:
            t.zero_()
        dp.factor(state.zero_threshold)
        x = torch.empty_like(b)
        dp.solve_into(b, x)
        torch.cuda.synchronize()
        assert dp.zero_pivot_position() == -1
        out[H] = ([t.clone() for t in dp.factors], x.clone())
    for a, c in zip(out[1][0], out[2][0]):
        assert torch.equal(a, c)
    assert torch.equal(out[1][1], out[2][1])
    r = system.matvec(out[2][1].cpu().numpy()) - b.cpu().numpy()
    assert np.abs(r).max() / np.abs(b.cpu().numpy()).max() < 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,p", [(1024, 1), (1000, 2), (3000, 3)])
def test_tiny_tree_one_launch_bitwise(n, p, cuda_ok):
    """1D trees take the one-launch path (tf_tree_factor_solve); its per-front
    arithmetic is the level kernels' (G < 32 groups compute every entry in
    one thread), so factors and solutions are bitwise the per-level path's."""
    mesh = tf.Mesh(n, p)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    state = tf.init_state(system, plan)
    dp = tf.compile_execution(plan, None, state)
    assert dp._tiny(), "a 1D tree should qualify for the one-launch path"
    b = torch.from_numpy(np.random.default_rng(4).standard_normal(mesh.n_dof)).to(dp.device)
    out = {}
    for tiny in (False, True):
        dp._tiny_ok = tiny
        for t in dp.factors:
            t.zero_()
        dp.factor(state.zero_threshold)
        x = torch.empty_like(b)
        dp.solve_into(b, x)
        x2 = torch.empty_like(b)
        dp.factor_solve(state.zero_threshold, b, x2)
        torch.cuda.synchronize()
        assert dp.zero_pivot_position() == -1
        out[tiny] = ([t.clone() for t in dp.factors], x.clone(), x2.clone())
    for a, c in zip(out[False][0], out[True][0]):
        assert torch.equal(a, c)
    assert torch.equal(out[False][1], out[True][1])
    assert torch.equal(out[True][1], out[True][2])
    assert torch.equal(out[False][2], out[True][2])
