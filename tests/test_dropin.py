"""The reference's own pipeline runs against the package (cli.py:142-161, 184-195).

CPU part: the reference's task-graph API (tasks.py:162-360, schedule.py:60-82)
is served by `paper_2306_08994_b200.tasks` / `.schedule` with the reference's
counts; and, where /root/reference exists (the build container), the
reference's UNMODIFIED cli.py is loaded as a submodule of this package so its
`_build_pipeline` / `cmd_plan` resolve `engine`, `tasks`, `schedule`, `tree`,
`fem`, `errors`, `fileio` to ours, and its `plan` report must equal the
reference's own.
GPU part: the `_build_pipeline` -> `_timed_factorize` -> `solve` call sequence
of cli.py:142-161, 217-222, written out with the reference's module aliases.
"""
import importlib.util
import io
import os
import subprocess
import sys
from contextlib import redirect_stdout
from pathlib import Path

import numpy as np
import pytest

import paper_2306_08994_b200 as tf
from conftest import golden, golden_names, mesh_of

REF_SRC = Path("/root/reference/pkg/src")
FNF = [n for n in golden_names() if "fnf_n_tasks" in golden(n)]


def plan_of(g):
    mesh = mesh_of(g)
    system = tf.assemble_system(mesh, "one")
    tree = tf.build_elimination_tree(tf.sort_fronts(tf.generate_fronts(mesh)))
    return system, tree, tf.symbolic_eliminate(tree, system)


@pytest.mark.parametrize("name", FNF)
def test_task_graph_api_counts(name):
    g = golden(name)
    system, tree, plan = plan_of(g)
    tasks = tf.enumerate_tasks(plan)
    graph = tf.build_dependency_edges(tasks, plan)
    assert graph.plan is plan
    assert len(tasks) == graph.n_tasks == int(g["fnf_n_tasks"])
    assert graph.n_edges == int(g["fnf_n_edges"])
    report = tf.validate_dag(graph)
    assert report.ok and report.longest_path == len(g["fnf_widths"])
    assert sum(report.kind_counts.values()) == graph.n_tasks
    foata = tf.compute_fnf(graph)
    stats = tf.schedule_stats(foata)
    assert list(stats.widths) == list(g["fnf_widths"])
    assert stats.n_classes == len(g["fnf_widths"])
    g2 = tf.build_task_graph(tree, system)
    assert g2.n_tasks == graph.n_tasks and g2.n_edges == graph.n_edges


@pytest.mark.parametrize("name", ["1d_n5_p3", "2d_5x3_p1", "3d_2x2x2_p1"])
def test_materialised_graph_equals_restated_reference(name):
    """tasks / preds / succs, materialised, equal the restatement (pinned to the reference)."""
    from oracle import restate
    g = golden(name)
    _, _, plan = plan_of(g)
    graph = tf.build_task_graph(plan.tree, plan.system)
    leaves = [tuple(int(x) for x in row) for row in g["elem_dofs"]]
    rtree = restate.build_tree(leaves)
    lower = {(a, b) for d in leaves for a in d for b in d if a >= b}
    rtasks, rsuccs = restate.task_graph(restate.symbolic(rtree, lower, int(g["n_dof"])))
    assert [(int(t.kind), t.front, t.pivot, t.row, t.col) for t in graph.tasks] == \
        [tuple(t) for t in rtasks]
    assert [sorted(s) for s in graph.succs] == [sorted(s) for s in rsuccs]
    assert sum(len(p) for p in graph.preds) == graph.n_edges


def test_run_concurrent_workers_without_group_is_an_error():
    g = golden("1d_n4_p1")
    system, tree, plan = plan_of(g)
    with pytest.raises(ValueError):
        tf.run_concurrent(None, plan, tf.init_state(system, plan), workers=0)
    with pytest.raises(ValueError):
        tf.run_concurrent(None, plan, tf.init_state(system, plan), workers=2)


def _load_reference_cli():
    spec = importlib.util.spec_from_file_location("paper_2306_08994_b200._reference_cli",
                                                  REF_SRC / "tracefront" / "cli.py")
    mod = importlib.util.module_from_spec(spec)
    sys.modules[spec.name] = mod
    spec.loader.exec_module(mod)
    return mod


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference sources only in the build container")
@pytest.mark.parametrize("argv", [["plan", "--elements", "64", "--degree", "3"],
                                  ["plan", "--elements", "1000", "--degree", "1"],
                                  ["plan", "--elements", "13", "--degree", "2"]])
def test_reference_cli_plan_runs_against_package(argv):
    refcli = _load_reference_cli()
    buf = io.StringIO()
    with redirect_stdout(buf):
        rc = refcli.main(argv)
    assert rc == 0
    env = dict(os.environ, PYTHONPATH=str(REF_SRC))
    ref = subprocess.run([sys.executable, "-m", "tracefront.cli"] + argv, env=env,
                         capture_output=True, text=True, timeout=600)
    assert ref.returncode == 0, ref.stderr
    assert buf.getvalue() == ref.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["1d_n1024_p1", "1d_n64_p3", "2d_8x8_p2", "3d_2x2x2_p1"])
@pytest.mark.parametrize("workers", [1])
def test_reference_pipeline_sequence_on_gpu(name, workers, cuda_ok):
    """cli.py:142-161 + 217-222, with the reference's module aliases."""
    from paper_2306_08994_b200 import engine, schedule as schedule_mod, tasks as tasks_mod, \
        tree as tree_mod
    from paper_2306_08994_b200.fem import assemble_system, generate_fronts
    g = golden(name)
    mesh = mesh_of(g)
    # _build_pipeline
    system = assemble_system(mesh, "one")
    elim_tree = tree_mod.build_elimination_tree(tree_mod.sort_fronts(generate_fronts(mesh)))
    plan = tasks_mod.symbolic_eliminate(elim_tree, system)
    graph = tasks_mod.build_dependency_edges(tasks_mod.enumerate_tasks(plan), plan)
    foata = schedule_mod.compute_fnf(graph)
    # _timed_factorize
    state = engine.init_state(system, graph.plan)
    if workers == 1:
        factors = engine.run_sequential(graph, state)
    else:
        factors = engine.run_concurrent(foata, graph, state, workers)
    assert factors.pivot_order == tuple(int(z) for z in g["pivot_order"])
    x = engine.solve(factors, g["rhs"])
    assert np.abs(x - g["x"]).max() / np.abs(g["x"]).max() <= 1e-10
    # run_concurrent(debug=True) checks the atomic schedule against the plan
    f2 = engine.run_concurrent(foata, graph, engine.init_state(system, graph.plan), 1, debug=True)
    assert np.array_equal(engine.solve(f2, g["rhs"]), x)
