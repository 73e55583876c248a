"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container only (needs /root/reference):
    PYTHONPATH=/root/reference/pkg/src:/root/repo python tests/golden/make_golden.py [names...]

For every instance it builds reference `Front`s and a reference
`GlobalSystem` (1D through fem.py's own Mesh/generate_fronts/assemble_system;
2D/3D through oracle/mesh_nd.py's tensor Q_p fronts assembled with
`GlobalSystem.add`), then calls the reference entry points:
  sort_fronts + build_elimination_tree   (tree.py:44, 106)
  symbolic_eliminate                     (tasks.py:88)
  factorize_nested_loops                 (engine.py:500)
  solve                                  (engine.py:468)
and, for small instances, build_task_graph + compute_fnf + run_sequential
(tasks.py:360, schedule.py:60, engine.py:177) to pin the FNF statistics and
to check run_sequential == nested loops bitwise.
Outputs tests/golden/<name>.npz (np.savez_compressed).
"""
import sys
import time
from pathlib import Path

import numpy as np

import tracefront as tf
from tracefront import engine as tf_engine
from oracle.mesh_nd import element_matrix, tensor_mesh

OUT = Path(__file__).resolve().parent

INSTANCES = {
    # name: (dims, degree, fnf?)
    "1d_n1_p1": ((1,), 1, True),
    "1d_n2_p1": ((2,), 1, True),
    "1d_n4_p1": ((4,), 1, True),
    "1d_n5_p3": ((5,), 3, True),
    "1d_n13_p2": ((13,), 2, True),
    "1d_n64_p3": ((64,), 3, True),
    "1d_n1000_p1": ((1000,), 1, True),
    "1d_n1024_p1": ((1024,), 1, True),  # cfg1
    "2d_2x2_p1": ((2, 2), 1, True),
    "2d_5x3_p1": ((5, 3), 1, True),
    "2d_8x8_p1": ((8, 8), 1, True),
    "2d_8x8_p2": ((8, 8), 2, True),
    "2d_7x6_p3": ((7, 6), 3, False),
    "2d_16x16_p2": ((16, 16), 2, False),
    "2d_32x32_p1": ((32, 32), 1, False),
    "3d_2x2x2_p1": ((2, 2, 2), 1, True),
    "3d_4x4x4_p1": ((4, 4, 4), 1, False),
    "3d_3x2x2_p2": ((3, 2, 2), 2, False),
    "2d_64x64_p2": ((64, 64), 2, False),  # cfg2 (~11 min nested loops)
}
SAMPLED = {"2d_64x64_p2"}  # factor dicts too large to commit: keep a strided sample


def build(dims, p):
    if len(dims) == 1:
        mesh = tf.Mesh(dims[0], p)
        fronts = tf.generate_fronts(mesh)
        system = tf.assemble_system(mesh, tf.fem.RHS_FUNCTIONS["one"])
        elems = [f.indices for f in fronts]
        emat = tf.fem.element_mass_matrix(mesh.element_width, p)
        n_dof = mesh.n_dof
        n2, elems2, _ = tensor_mesh(dims, p)
        assert n2 == n_dof and [tuple(e) for e in elems2] == [tuple(e) for e in elems]
        assert np.array_equal(element_matrix(dims, p), emat)
        rhs_one = system.rhs.copy()
    else:
        n_dof, elems, _ = tensor_mesh(dims, p)
        emat = element_matrix(dims, p)
        fronts = []
        system = tf.GlobalSystem(n_dof=n_dof, rhs=np.zeros(n_dof))
        for e, dofs in enumerate(elems):
            fronts.append(tf.Front(front_id=e, indices=tuple(dofs),
                                   membership=(1,) * len(dofs),
                                   computed=(False,) * len(dofs), values=emat.copy()))
            for a, ga in enumerate(dofs):
                for b, gb in enumerate(dofs):
                    if ga >= gb:
                        system.add(ga, gb, emat[a, b])
        rhs_one = None
    return n_dof, elems, emat, fronts, system, rhs_one


def keyvals(d):
    keys = sorted(d)
    k = np.array(keys, dtype=np.int32).reshape(-1, 2)
    v = np.array([d[c] for c in keys], dtype=np.float64)
    return k, v


def run(name):
    dims, p, do_fnf = INSTANCES[name]
    t0 = time.time()
    n_dof, elems, emat, fronts, system, rhs_one = build(dims, p)
    tree = tf.build_elimination_tree(tf.sort_fronts(fronts))
    plan = tf.symbolic_eliminate(tree, system)
    out = {
        "dims": np.array(dims, dtype=np.int64), "degree": np.int64(p), "n_dof": np.int64(n_dof),
        "elem_dofs": np.array(elems, dtype=np.int32), "elem_matrix": emat,
        "level_sizes": np.array([len(l) for l in tree.levels], dtype=np.int64),
        "root_id": np.int64(tree.root_id),
        "pivot_order": np.array(plan.pivot_order, dtype=np.int32),
        "reorder_node": np.array([r.node_id for r in plan.reorders], dtype=np.int64),
        "reorder_counts": np.array([(len(r.eliminable), len(r.shared), len(r.computed))
                                    for r in plan.reorders], dtype=np.int64),
        "reorder_elim": np.array([g for r in plan.reorders for g in r.eliminable], dtype=np.int32),
        "reorder_shared": np.array([g for r in plan.reorders for g in r.shared], dtype=np.int32),
        "n_cells": np.int64(len(plan.cells)), "n_fill": np.int64(len(plan.fill_cells)),
        "active_sizes": np.array([len(s.active) for s in plan.steps], dtype=np.int32),
        "step_node": np.array([s.node_id for s in plan.steps], dtype=np.int64),
    }
    state = tf.init_state(system, plan)
    out["threshold"] = np.float64(state.zero_threshold)
    t1 = time.time()
    values, factors = tf.factorize_nested_loops(tree, system)
    t_nested = time.time() - t1
    assert factors.pivot_order == plan.pivot_order
    rng = np.random.default_rng(0)
    rhs = rng.standard_normal(n_dof)
    out["rhs"] = rhs
    t1 = time.time()
    out["x"] = tf.solve(factors, rhs)
    t_solve = time.time() - t1
    if rhs_one is not None:
        out["rhs_one"] = rhs_one
        out["x_one"] = tf.solve(factors, rhs_one)
    uk, uv = keyvals(factors.u_entries)
    lk, lv = keyvals(factors.l_entries)
    out["u_count"], out["l_count"] = np.int64(len(uv)), np.int64(len(lv))
    out["u_absmax"], out["l_absmax"] = np.float64(np.abs(uv).max()), np.float64(np.abs(lv).max())
    if name in SAMPLED:
        stride = 61
        uk, uv, lk, lv = uk[::stride], uv[::stride], lk[::stride], lv[::stride]
        out["sample_stride"] = np.int64(stride)
    out["u_keys"], out["u_vals"], out["l_keys"], out["l_vals"] = uk, uv, lk, lv
    if do_fnf:
        graph = tf.build_task_graph(tree, system)
        sched = tf.compute_fnf(graph)
        stats = tf.schedule_stats(sched)
        out["fnf_n_tasks"] = np.int64(graph.n_tasks)
        out["fnf_n_edges"] = np.int64(graph.n_edges)
        out["fnf_widths"] = np.array(stats.widths, dtype=np.int64)
        st = tf.init_state(system, graph.plan)
        seq = tf.run_sequential(graph, st)
        assert seq.u_entries == factors.u_entries and seq.l_entries == factors.l_entries, \
            "run_sequential != nested loops (bitwise)"
    out["t_nested_s"] = np.float64(t_nested)
    out["t_solve_s"] = np.float64(t_solve)
    np.savez_compressed(OUT / f"{name}.npz", **out)
    print(f"{name}: n_dof={n_dof} levels={len(tree.levels)} nested={t_nested:.2f}s "
          f"total={time.time() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or [n for n in INSTANCES if n != "2d_64x64_p2"]
    from multiprocessing import Pool
    with Pool(min(8, len(names))) as pool:
        pool.map(run, names)
