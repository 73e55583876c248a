"""Pin the native symbolic plan to the REFERENCE's symbolic_eliminate at scale.

Build container only (imports /root/reference):
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_symbolic_golden.py NAME...

For each mesh it runs the reference's sort_fronts + build_elimination_tree +
symbolic_eliminate (tree.py:44-160, tasks.py:88-159) on tensor-mesh fronts
(oracle/mesh_nd.py) and stores sha256 digests of the pivot order, of the
per-node reorders (eliminable / shared lists) and of the per-step active-set
sizes, plus level sizes and cell counts (tests/golden/symbolic_<name>.npz).
"""
import hashlib
import sys
import time
from pathlib import Path

import numpy as np

import tracefront as tf
from oracle.mesh_nd import element_matrix, tensor_mesh

OUT = Path(__file__).resolve().parent
INSTANCES = {"2d_256x256_p1": ((256, 256), 1), "2d_128x128_p2": ((128, 128), 2),
             "3d_16x16x16_p1": ((16, 16, 16), 1), "2d_256x256_p2": ((256, 256), 2)}


def sha(a):
    return np.frombuffer(hashlib.sha256(np.ascontiguousarray(a).tobytes()).digest(), np.uint8)


def run(name):
    dims, p = INSTANCES[name]
    t0 = time.time()
    n_dof, elems, _ = tensor_mesh(dims, p)
    emat = element_matrix(dims, p)
    fronts = [tf.Front(front_id=e, indices=tuple(d), membership=(1,) * len(d),
                       computed=(False,) * len(d), values=emat) for e, d in enumerate(elems)]
    lower = {}
    for d in elems:
        for a in d:
            for b in d:
                if a >= b:
                    lower[(a, b)] = 1.0
    system = tf.GlobalSystem(n_dof=n_dof, entries=lower, rhs=np.zeros(n_dof))
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts))
    plan = tf.symbolic_eliminate(tree, system)
    po = np.array(plan.pivot_order, dtype="<i4")
    elim = np.array([g for r in plan.reorders for g in r.eliminable], dtype="<i4")
    shared = np.array([g for r in plan.reorders for g in r.shared], dtype="<i4")
    counts = np.array([(len(r.eliminable), len(r.shared)) for r in plan.reorders], dtype="<i8")
    act = np.array([len(s.active) for s in plan.steps], dtype="<i4")
    np.savez_compressed(OUT / f"symbolic_{name}.npz", dims=np.array(dims), degree=np.int64(p),
                        n_dof=np.int64(n_dof), level_sizes=np.array([len(l) for l in tree.levels]),
                        pivot_order_sha=sha(po), reorder_elim_sha=sha(elim),
                        reorder_shared_sha=sha(shared), reorder_counts_sha=sha(counts),
                        active_sizes_sha=sha(act), n_cells=np.int64(len(plan.cells)),
                        n_fill=np.int64(len(plan.fill_cells)), t_s=np.float64(time.time() - t0))
    print(f"{name}: n_dof={n_dof} {time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    for nm in sys.argv[1:] or list(INSTANCES):
        run(nm)
