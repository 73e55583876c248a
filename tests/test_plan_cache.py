"""On-disk plan cache: a cached plan equals a fresh one."""
import time

import numpy as np

import paper_2306_08994_b200 as tf
from paper_2306_08994_b200.plan import NativePlan, plan_cache_path
from paper_2306_08994_b200.tree import EliminationTree


def test_plan_cache_roundtrip(tmp_path):
    mesh = tf.TensorMesh((256, 256), 1)
    fr = tf.sort_fronts(tf.generate_fronts(mesh))
    fresh = NativePlan(fr, mesh.n_dof)
    t0 = time.perf_counter()
    a = NativePlan(fr, mesh.n_dof, cache_dir=tmp_path)       # builds + stores
    t_build = time.perf_counter() - t0
    assert not a.cache_hit and plan_cache_path(fr, mesh.n_dof, tmp_path).exists()
    t0 = time.perf_counter()
    b = NativePlan(fr, mesh.n_dof, cache_dir=tmp_path)       # loads
    t_load = time.perf_counter() - t0
    assert b.cache_hit
    for k in ("n_dof", "n_leaves", "n_nodes", "n_pivots", "n_levels", "max_m", "max_k"):
        assert getattr(b, k) == getattr(fresh, k)
    assert np.array_equal(b.pivot_order, fresh.pivot_order)
    for x, y in zip(b.levels, fresh.levels):
        for k in ("level", "n_fronts", "node_base", "piv_base", "n_pivots", "max_m", "max_k",
                  "max_upd"):
            assert getattr(x, k) == getattr(y, k)
        for k in ("pattern_of", "piv_off", "pat", "maps"):
            assert np.array_equal(getattr(x, k), getattr(y, k))
    assert b.level_stats() == fresh.level_stats()
    assert t_load < t_build


def test_plan_cache_keys_on_the_fronts(tmp_path):
    m1, m2 = tf.TensorMesh((16, 16), 1), tf.TensorMesh((16, 16), 2)
    f1, f2 = tf.generate_fronts(m1), tf.generate_fronts(m2)
    assert plan_cache_path(f1, m1.n_dof, tmp_path) != plan_cache_path(f2, m2.n_dof, tmp_path)
    t = EliminationTree(f1, n_dof=m1.n_dof, keep_lists=False, cache_dir=tmp_path)
    t2 = EliminationTree(f1, n_dof=m1.n_dof, keep_lists=False, cache_dir=tmp_path)
    assert t2.plan.cache_hit and t2.level_sizes == t.level_sizes
    # plans with node lists are never cached (they carry the native handle)
    t3 = EliminationTree(f2, n_dof=m2.n_dof, keep_lists=True, cache_dir=tmp_path)
    assert not t3.plan.cache_hit and not plan_cache_path(f2, m2.n_dof, tmp_path).exists()
