import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2306_08994_b200 as tf
mesh = tf.TensorMesh((4096, 4096), 1)
tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)), n_dof=mesh.n_dof)
system = tf.assemble_system(mesh, "one")
plan = tf.symbolic_eliminate(tree, system)
st = tf.init_state(system, plan)
dp = tf.compile_execution(plan, None, st)
for _ in range(2):
    dp.factor(st.zero_threshold)
torch.cuda.synchronize()
