"""Subtree-sharded factor/solve, all ranks simulated on one GPU (LocalComm).

The sharded run uses the same kernels on slice views plus the rank-to-rank
transfers; its factors must be bitwise identical to the single-GPU run and
its solution must match the reference golden vectors.
"""
import numpy as np
import pytest
import torch

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200.distributed import LocalComm, ShardedFactorization
from conftest import golden, mesh_of


def setup(name):
    g = golden(name)
    mesh = mesh_of(g)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts))
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    state = tf.init_state(system, plan)
    return g, plan, state


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["2d_64x64_p2", "2d_5x3_p1", "1d_n1000_p1", "3d_4x4x4_p1"])
@pytest.mark.parametrize("world", [2, 3, 4, 8])
def test_sharded_equals_single_gpu(name, world, cuda_ok):
    g, plan, state = setup(name)
    single = tf.run_sequential(plan, state)
    dp = single.device_plan
    ref = [t.clone() for t in dp.factors]
    sh = ShardedFactorization(dp, world, LocalComm())
    assert sh.factor(state.zero_threshold) == -1
    got = sh.gather_factors()
    for L, dl in enumerate(dp.levels):
        n = dl.n_fronts * dl.fac_stride
        if n == 0:
            continue
        # compare the written (lower/diagonal) entries: gather masks unused slots with 0
        lt = dl.tables
        for f in range(dl.n_fronts):
            row = lt.pat[lt.pattern_of[f]]
            m, k, kp = int(row[0]), int(row[1]), int(row[9])
            if k == 0:
                continue
            a = ref[L][f * dl.fac_stride: f * dl.fac_stride + m * kp + kp].view(m * kp + kp)
            b = got[L][f * dl.fac_stride: f * dl.fac_stride + m * kp + kp].view(m * kp + kp)
            P_a, P_b = a[:m * kp].view(m, kp), b[:m * kp].view(m, kp)
            mask = torch.tril(torch.ones(m, kp, dtype=torch.bool, device=a.device))
            mask[:, k:] = False
            assert torch.equal(P_a[mask], P_b[mask]), (L, f)
            assert torch.equal(a[m * kp: m * kp + k], b[m * kp: m * kp + k])
    B = torch.from_numpy(np.stack([g["rhs"], np.random.default_rng(3).standard_normal(len(g["rhs"]))], 1)).cuda()
    X = torch.empty_like(B)
    sh.solve_into(B, X)
    x = X[:, 0].cpu().numpy()
    assert np.abs(x - g["x"]).max() / np.abs(g["x"]).max() <= 1e-10
    X1 = torch.empty_like(B)
    dp.solve_into(B, X1)
    assert torch.equal(X, X1) or torch.allclose(X, X1, rtol=0, atol=1e-13 * X1.abs().max().item())
