"""One small factor + solve that reaches the persistent / flag-synchronised
kernels, for compute-sanitizer (tools/sanitize.sh).

Every non-leaf level runs on the blocked large-front kernels (small-front
limit 1), so the root dataflow kernel (acquire/release flags between chain and
tile CTAs), the wavefront sweeps (solve_fwd_wave / solve_bwd_wave, per-block
flags) and, through the TFB_* environment knobs set by the caller, the split
and CTA-per-front sweeps and the lookahead streams all execute.
"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2306_08994_b200 as tf  # noqa: E402
from paper_2306_08994_b200 import device  # noqa: E402

shape = tuple(int(t) for t in (sys.argv[1] if len(sys.argv) > 1 else "48x48").split("x"))
nrhs = int(sys.argv[2]) if len(sys.argv) > 2 else 1
device.set_small_front_limit(1)
mesh = tf.TensorMesh(shape, 1)
tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)), n_dof=mesh.n_dof)
system = tf.assemble_system(mesh, "one")
plan = tf.symbolic_eliminate(tree, system)
f = tf.run_sequential(plan, tf.init_state(system, plan))
B = np.random.default_rng(0).standard_normal((mesh.n_dof, nrhs))
X = tf.solve(f, B if nrhs > 1 else B[:, 0])
X = X.reshape(mesh.n_dof, nrhs)
res = np.abs(system.matvec(X) - B).max() / np.abs(B).max()
print(f"sanitize case {shape} nrhs={nrhs}: levels={plan.n_levels} residual={res:.2e}")
assert res < 1e-12
