"""The native symbolic plan equals the REFERENCE's symbolic_eliminate beyond the
small goldens (tests/golden/symbolic_*.npz, made by make_symbolic_golden.py
with the reference itself: 66k DoF 2D Q1, 66k DoF 2D Q2, 3D 16^3, and where
present 263k DoF 2D Q2): pivot order, every NodeReorder's eliminable and
shared lists, per-step active-set sizes, stored and fill cell counts."""
import hashlib
import os

import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import GOLDEN
from paper_2306_08994_b200.tree import EliminationTree

NAMES = sorted(p.stem[len("symbolic_"):] for p in GOLDEN.glob("symbolic_*.npz"))


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest()


@pytest.mark.parametrize("name", NAMES)
def test_native_plan_equals_reference_symbolic(name):
    g = dict(np.load(GOLDEN / f"symbolic_{name}.npz"))
    mesh = tf.TensorMesh(tuple(int(x) for x in g["dims"]), int(g["degree"]))
    fronts = tf.sort_fronts(tf.generate_fronts(mesh))
    tree = EliminationTree(fronts, n_dof=mesh.n_dof, keep_lists=True)
    assert list(tree.level_sizes) == list(g["level_sizes"])
    plan = tf.symbolic_eliminate(tree, tf.assemble_system(mesh, "one"))
    assert sha(plan.pivot_order_array.astype("<i4")) == bytes(g["pivot_order_sha"])
    elim, shared, counts = [], [], []
    for L in range(plan.n_levels):
        ptr, k, idx = plan.native.node_lists(L)
        for i in range(len(k)):
            lst = idx[ptr[i]:ptr[i + 1]]
            elim.append(lst[:k[i]])
            shared.append(lst[k[i]:])
            counts.append((int(k[i]), len(lst) - int(k[i])))
    assert sha(np.concatenate(elim).astype("<i4")) == bytes(g["reorder_elim_sha"])
    assert sha(np.concatenate(shared).astype("<i4")) == bytes(g["reorder_shared_sha"])
    assert sha(np.array(counts, dtype="<i8")) == bytes(g["reorder_counts_sha"])
    if os.environ.get("TFB_SLOW_TESTS") == "1":
        # the Python boolean structure simulation behind plan.steps / plan.cells
        # takes minutes at these sizes (passes: 2D 256^2 p1 143 s, 2D 128^2 p2 137 s,
        # 3D 16^3 42 s on the build container)
        act = np.array([len(s.active) for s in plan.steps], dtype="<i4")
        assert sha(act) == bytes(g["active_sizes_sha"])
        assert len(plan.cells) == int(g["n_cells"]) and len(plan.fill_cells) == int(g["n_fill"])
