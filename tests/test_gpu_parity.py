"""GPU parity against the reference's own golden vectors (tests/golden/*.npz).

Contract: identical tree / pivot order; factors within
1e-10 normwise (max|dU| / max|U_ref|, same for L) on the reference's exact key
sets; solution within 1e-10 relative (inf-norm) per right-hand side.
"""
import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden, golden_names, mesh_of

FACTOR_TOL = 1e-10
SOLVE_TOL = 1e-10
SMALL = [n for n in golden_names() if n != "2d_64x64_p2"]


def pipeline(g):
    mesh = mesh_of(g)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts))
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    state = tf.init_state(system, plan)
    return mesh, system, plan, state


def normwise(keys, vals, d):
    got = np.array([d[(int(a), int(b))] for a, b in keys])
    return np.abs(got - vals).max() / np.abs(vals).max()


@pytest.fixture(params=["smem", "large", "fused"])
def front_path(request, cuda_ok):
    """Shared-memory fronts up to m=232; every non-leaf level forced through the
    blocked large-front (DMMA) kernels; or the bottom levels fused into
    subtree launches (tf_subtree_factor)."""
    from paper_2306_08994_b200 import device
    old = device.set_small_front_limit(1 if request.param == "large" else 232)
    device.FUSE_CAP_DEFAULT = 10 if request.param == "fused" else 0
    auto = device.FUSE_AUTO_MAX_LEAVES
    device.FUSE_AUTO_MAX_LEAVES = 0  # per-level kernels unless "fused"
    yield request.param
    device.FUSE_CAP_DEFAULT = 0
    device.FUSE_AUTO_MAX_LEAVES = auto
    device.set_small_front_limit(old)


@pytest.mark.gpu
@pytest.mark.parametrize("name", SMALL)
def test_factor_and_solve_match_reference(name, front_path):
    g = golden(name)
    mesh, system, plan, state = pipeline(g)
    factors = tf.run_sequential(plan, state)
    assert np.array_equal(np.array(factors.pivot_order), g["pivot_order"])
    u, l = factors.u_entries, factors.l_entries
    assert len(u) == int(g["u_count"]) and len(l) == int(g["l_count"])
    assert set(u) == {(int(a), int(b)) for a, b in g["u_keys"]}
    assert normwise(g["u_keys"], g["u_vals"], u) <= FACTOR_TOL
    assert normwise(g["l_keys"], g["l_vals"], l) <= FACTOR_TOL
    x = tf.solve(factors, g["rhs"])
    assert np.abs(x - g["x"]).max() / np.abs(g["x"]).max() <= SOLVE_TOL
    if "x_one" in g:
        x1 = tf.solve(factors, g["rhs_one"])
        assert np.abs(x1 - g["x_one"]).max() / np.abs(g["x_one"]).max() <= SOLVE_TOL


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["2d_16x16_p2", "3d_4x4x4_p1", "1d_n1000_p1"])
def test_multi_rhs_columnwise(name, front_path):
    g = golden(name)
    mesh, system, plan, state = pipeline(g)
    factors = tf.run_sequential(plan, state)
    rng = np.random.default_rng(1)
    B = rng.standard_normal((plan.n_dof, 7))
    B[:, 0] = g["rhs"]
    X = tf.solve(factors, B)
    assert np.abs(X[:, 0] - g["x"]).max() / np.abs(g["x"]).max() <= SOLVE_TOL
    for j in range(1, 7):
        xj = tf.solve(factors, B[:, j])
        assert np.abs(X[:, j] - xj).max() <= 1e-12 * np.abs(xj).max()


@pytest.mark.gpu
def test_cfg2_against_reference_nested_loops(front_path):
    g = golden("2d_64x64_p2")
    mesh, system, plan, state = pipeline(g)
    factors = tf.run_sequential(plan, state)
    assert np.array_equal(np.array(factors.pivot_order), g["pivot_order"])
    x = tf.solve(factors, g["rhs"])
    assert np.abs(x - g["x"]).max() / np.abs(g["x"]).max() <= SOLVE_TOL
    u, l = factors.u_entries, factors.l_entries
    assert len(u) == int(g["u_count"]) and len(l) == int(g["l_count"])
    # strided sample of the reference factor dictionaries, normalised by the full max
    for keys, vals, d, amax in ((g["u_keys"], g["u_vals"], u, g["u_absmax"]),
                                (g["l_keys"], g["l_vals"], l, g["l_absmax"])):
        got = np.array([d[(int(a), int(b))] for a, b in keys])
        assert np.abs(got - vals).max() / float(amax) <= FACTOR_TOL


@pytest.mark.gpu
def test_zero_pivot_singular_front(cuda_ok):
    """[[1,1],[1,1]] raises ZeroPivotError at pivot 2, front 0."""
    vals = np.array([[1.0, 1.0], [1.0, 1.0]])
    front = tf.Front(0, (1, 2), (1, 1), (False, False), vals)
    system = tf.GlobalSystem(2, {(1, 1): 1.0, (2, 1): 1.0, (2, 2): 1.0}, np.zeros(2))
    tree = tf.build_elimination_tree([front])
    plan = tf.symbolic_eliminate(tree, system)
    with pytest.raises(tf.ZeroPivotError) as ei:
        tf.run_sequential(plan, tf.init_state(system, plan))
    assert ei.value.pivot == 2 and ei.value.front == 0


@pytest.mark.gpu
def test_two_by_two_known_answer(cuda_ok):
    """[[2,1],[1,2]]: u={(1,1):2,(1,2):.5,(2,2):1.5}, l={(2,1):.5}, x=[1,1]."""
    vals = np.array([[2.0, 1.0], [1.0, 2.0]])
    front = tf.Front(0, (1, 2), (1, 1), (False, False), vals)
    system = tf.GlobalSystem(2, {(1, 1): 2.0, (2, 1): 1.0, (2, 2): 2.0}, np.array([3.0, 3.0]))
    tree = tf.build_elimination_tree([front])
    plan = tf.symbolic_eliminate(tree, system)
    f = tf.run_sequential(plan, tf.init_state(system, plan))
    assert f.u_entries == {(1, 2): 0.5, (1, 1): 2.0, (2, 2): 1.5}
    assert f.l_entries == {(2, 1): 0.5}
    assert np.allclose(tf.solve(f, np.array([3.0, 3.0])), [1.0, 1.0], rtol=0, atol=1e-15)
