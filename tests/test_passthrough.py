"""Pass-through tables (tf_level_view.leaf_direct, DevicePlan._setup_leaf_direct):
for every pivot-free leaf that level 1 reads from its element matrix, the
table lookup must equal the update the leaf would have written -- emulated
here from the leaf's forward extend-add map (fem.py:235-259 element
matrices in front order)."""
import numpy as np
import pytest
import torch

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200 import _lib, device


def _plan(shape, p, graded=False):
    if graded:  # graded nodes and per-element densities: every element matrix differs
        rng = np.random.default_rng(4)
        nodes = tuple(np.concatenate([[0.0], np.cumsum(w)]) / w.sum()
                      for w in (rng.uniform(0.5, 1.5, n) for n in shape))
        rho = rng.uniform(0.5, 2.0, int(np.prod(shape)))
        mesh = tf.TensorMesh(shape, p, nodes=nodes, density=rho)
    else:
        mesh = tf.TensorMesh(shape, p)
    fronts = tf.generate_fronts(mesh)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts), n_dof=mesh.n_dof)
    system = tf.assemble_system(mesh, "one")
    plan = tf.symbolic_eliminate(tree, system)
    return mesh, fronts, plan


def _tri(r):
    return r * (r + 1) // 2


def _leaf_update(lt0, f, E, ld):
    """Packed update (front order) of a pivot-free leaf: its element's lower
    entries scattered through the forward map."""
    p = lt0.pattern_of[f]
    m = int(lt0.pat[p, _lib.PAT_M])
    fwd = lt0.maps[lt0.pat[p, _lib.PAT_OFF0]:lt0.pat[p, _lib.PAT_OFF0] + m]
    U = np.zeros(_tri(m))
    for a in range(m):
        for b in range(a + 1):
            x, y = fwd[a], fwd[b]
            U[_tri(max(x, y)) + min(x, y)] += E[a * ld + b]
    return U


@pytest.mark.parametrize("shape,p,graded", [((16, 12), 1, False), ((6, 6), 2, False),
                                            ((4, 4, 4), 1, False), ((14, 10), 1, True)])
def test_leaf_index_tables_match_leaf_updates(shape, p, graded):
    """Level 1 reads a pivot-free leaf child through leaf_index (per leaf
    pattern: packed update entry -> element index); the result must be the
    leaf's packed update exactly (bitwise)."""
    mesh, fronts, plan = _plan(shape, p, graded)
    vals = np.ascontiguousarray(fronts.values, dtype=np.float64)
    dp = device.DevicePlan(plan, fronts, device=torch.device("cpu"), values=vals)
    l0, l1 = dp.levels[0], dp.levels[1]
    if not l1.view.leaf_direct:
        pytest.skip("pass-through not enabled for this tree")
    ld = l0.view.elem_ld
    E = vals.reshape(-1, ld * ld) if vals.ndim == 3 else np.tile(vals.ravel(), (l0.n_fronts, 1))
    lt0 = l0.tables
    tab = l1.leaf_index.numpy()
    kk = lt0.pat[lt0.pattern_of, _lib.PAT_K]
    free = np.nonzero(kk == 0)[0]
    if len(free) == 0:
        pytest.skip("no pivot-free leaves on this mesh (every leaf has pivots)")
    for ch in free[:300]:
        want = _leaf_update(lt0, ch, E[ch], ld)
        T = tab[tab[lt0.pattern_of[ch]]:][:len(want)]
        assert np.array_equal(E[ch][T], want), ch
