"""Host wrapper of the native symbolic plan (libtfb200.so `tf_plan`).

One `NativePlan` is the C++ result of sort-order leaf fronts ->
elimination tree -> symbolic elimination (tree.py:106-160,
tasks.py:88-159): pivot order, per-level front patterns and extend-add maps.
"""

from __future__ import annotations

import ctypes as C
import hashlib
import os
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _lib
from .errors import EmptyInputError
from .fem import FrontSet


@dataclass
class LevelTables:
    """Numpy copies of one level's tf_level_host tables."""

    level: int
    n_fronts: int
    node_base: int
    piv_base: int
    n_pivots: int
    max_m: int
    max_k: int
    max_upd: int
    pattern_of: np.ndarray  # int32 [n_fronts]
    piv_off: np.ndarray     # int64 [n_fronts]
    pat: np.ndarray         # int32 [n_patterns, 8]
    maps: np.ndarray        # int32

    @property
    def n_patterns(self) -> int:
        return len(self.pat)

    def front_m(self) -> np.ndarray:
        return self.pat[self.pattern_of, _lib.PAT_M]

    def front_k(self) -> np.ndarray:
        return self.pat[self.pattern_of, _lib.PAT_K]

    def pattern_counts(self) -> np.ndarray:
        return np.bincount(self.pattern_of, minlength=self.n_patterns)


PLAN_CACHE_VERSION = 2
_SCALARS = ("n_dof", "n_leaves", "n_nodes", "n_pivots", "n_levels", "max_m", "max_k")
_LEVEL_FIELDS = ("level", "n_fronts", "node_base", "piv_base", "n_pivots", "max_m", "max_k",
                 "max_upd")
_LEVEL_ARRAYS = ("pattern_of", "piv_off", "pat", "maps")


def plan_cache_path(fronts: FrontSet, n_dof: int, cache_dir) -> Path:
    """Cache file of the plan of these leaf fronts: keyed by a digest of n_dof, the
    front index lists (in order) and the cache format version."""
    h = hashlib.sha256()
    kp_align = os.environ.get("TFB_KP_ALIGN", "2")  # panel layout knob of the native planner
    h.update(f"tfb-plan-v{PLAN_CACHE_VERSION}:{kp_align}:{int(n_dof)}:{len(fronts)}".encode())
    h.update(np.ascontiguousarray(fronts.dofs, dtype=np.int32).tobytes())
    if fronts.ptr is not None:
        h.update(np.ascontiguousarray(fronts.ptr, dtype=np.int64).tobytes())
    return Path(cache_dir) / f"plan_{h.hexdigest()[:32]}.npz"


class NativePlan:
    """The symbolic plan (tree, pivot order, level tables) of a set of leaf fronts.

    With `cache_dir` (or TFB_PLAN_CACHE) and without per-node lists, the plan is
    stored on disk after it is built and loaded from there the next time the
    same fronts are planned (cfg5: ~20 s of symbolic work -> one file read);
    a cached plan carries no native handle (node lists / atomic FNF need
    keep_lists, which is never cached)."""

    def __init__(self, fronts: FrontSet, n_dof: int, keep_lists: bool = False, cache_dir=None):
        if len(fronts) == 0:
            raise EmptyInputError("cannot build a tree from zero fronts")
        lib = _lib.load()
        self._lib = lib
        self._h = C.c_void_p()
        cache_dir = cache_dir if cache_dir is not None else os.environ.get("TFB_PLAN_CACHE")
        path = plan_cache_path(fronts, n_dof, cache_dir) if cache_dir and not keep_lists else None
        self.cache_hit = False
        if path is not None and path.exists():
            try:
                self._load(path)
                self.cache_hit = True
                return
            except Exception:
                pass  # unreadable / stale: rebuild below and overwrite
        self._build(fronts, n_dof, keep_lists)
        if path is not None:
            self._save(path)

    def _save(self, path: Path) -> None:
        d = {k: np.int64(getattr(self, k)) for k in _SCALARS}
        d["pivot_order"] = self.pivot_order
        d["n_level_tables"] = np.int64(len(self.levels))
        for L, lt in enumerate(self.levels):
            for k in _LEVEL_FIELDS:
                d[f"L{L}_{k}"] = np.int64(getattr(lt, k))
            for k in _LEVEL_ARRAYS:
                d[f"L{L}_{k}"] = getattr(lt, k)
        path.parent.mkdir(parents=True, exist_ok=True)
        tmp = path.with_name(path.name + f".{os.getpid()}.tmp")
        with open(tmp, "wb") as fh:
            np.savez(fh, **d)
        os.replace(tmp, path)

    def _load(self, path: Path) -> None:
        with np.load(path) as z:
            for k in _SCALARS:
                setattr(self, k, int(z[k]))
            self.keep_lists = False
            self.pivot_order = z["pivot_order"].astype(np.int32)
            levels = []
            for L in range(int(z["n_level_tables"])):
                kw = {k: int(z[f"L{L}_{k}"]) for k in _LEVEL_FIELDS}
                kw.update({k: z[f"L{L}_{k}"] for k in _LEVEL_ARRAYS})
                levels.append(LevelTables(**kw))
            self.levels = levels

    def _build(self, fronts: FrontSet, n_dof: int, keep_lists: bool) -> None:
        lib = self._lib
        h = C.c_void_p()
        dofs = np.ascontiguousarray(fronts.dofs, dtype=np.int32)
        if fronts.ptr is None:
            ptr = None
            nloc = dofs.shape[1]
        else:
            ptr = np.ascontiguousarray(fronts.ptr, dtype=np.int64)
            nloc = 0
        rc = lib.tf_plan_create(int(n_dof), len(fronts), None if ptr is None else _lib.i64p(ptr),
                                int(nloc), _lib.i32p(dofs), 1 if keep_lists else 0, C.byref(h))
        if rc != _lib.TF_OK:
            raise ValueError("tf_plan_create rejected the fronts (DOF out of range or a "
                             "front index map that is not injective)")
        self._h = h
        s = _lib.PlanSummary()
        _lib.check(lib.tf_plan_summary_get(h, C.byref(s)), "tf_plan_summary_get")
        self.n_dof = int(s.n_dof)
        self.n_leaves = int(s.n_leaves)
        self.n_nodes = int(s.n_nodes)
        self.n_pivots = int(s.n_pivots)
        self.n_levels = int(s.n_levels)
        self.max_m = int(s.max_m)
        self.max_k = int(s.max_k)
        self.keep_lists = bool(s.keep_lists)
        self.levels = [self._level(L) for L in range(self.n_levels)]
        po = np.empty(self.n_pivots, dtype=np.int32)
        _lib.check(lib.tf_plan_pivot_order(h, _lib.i32p(po)), "tf_plan_pivot_order")
        self.pivot_order = po

    def atomic_fnf(self):
        """(FnfStats, widths[int64], kinds[int32]) of the atomic Foata normal form."""
        if not self.keep_lists or not self._h.value:
            raise RuntimeError("atomic FNF needs a plan built with keep_lists")
        st = _lib.FnfStats()
        rc = self._lib.tf_atomic_fnf(self._h, C.byref(st), None, None, 0)
        if rc == _lib.TF_ERR_STRAY:
            from .errors import SymbolicSingularityError
            raise SymbolicSingularityError(int(st.singular))
        _lib.check(rc, "tf_atomic_fnf")
        n = max(int(st.n_classes), 1)
        widths = np.zeros(n, dtype=np.int64)
        kinds = np.zeros(n, dtype=np.int32)
        _lib.check(self._lib.tf_atomic_fnf(self._h, C.byref(st), _lib.i64p(widths),
                                           _lib.i32p(kinds), n), "tf_atomic_fnf")
        return st, widths[:st.n_classes], kinds[:st.n_classes]

    def _level(self, L: int) -> LevelTables:
        lh = _lib.LevelHost()
        _lib.check(self._lib.tf_plan_level(self._h, L, C.byref(lh)), "tf_plan_level")
        nf, npat = lh.n_fronts, lh.n_patterns

        def arr(ptr, n, dt):
            if n == 0:
                return np.zeros(0, dtype=dt)
            return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dt, copy=True)

        return LevelTables(
            level=L, n_fronts=nf, node_base=int(lh.node_base), piv_base=int(lh.piv_base),
            n_pivots=int(lh.n_pivots), max_m=lh.max_m, max_k=lh.max_k, max_upd=lh.max_upd,
            pattern_of=arr(lh.pattern_of, nf, np.int32), piv_off=arr(lh.piv_off, nf, np.int64),
            pat=arr(lh.pat, npat * _lib.PAT_WIDTH, np.int32).reshape(npat, _lib.PAT_WIDTH),
            maps=arr(lh.maps, int(lh.maps_len), np.int32),
        )

    def node_lists(self, L: int):
        """(ptr, k, idx): per-front [eliminable | shared] global indices of level L."""
        if not self.keep_lists:
            raise RuntimeError("plan was built without keep_lists")
        n = self.levels[L].n_fronts
        total = int(self._lib.tf_plan_node_lists_len(self._h, L))
        ptr = np.empty(n + 1, dtype=np.int64)
        k = np.empty(n, dtype=np.int32)
        idx = np.empty(max(total, 1), dtype=np.int32)
        _lib.check(self._lib.tf_plan_node_lists(self._h, L, _lib.i64p(ptr), _lib.i32p(k),
                                                _lib.i32p(idx)), "tf_plan_node_lists")
        return ptr, k, idx[:total]

    def close(self) -> None:
        if getattr(self, "_h", None) is not None and self._h.value:
            self._lib.tf_plan_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- per-level work model -------------------------------

    def level_stats(self) -> list[dict]:
        """Per level: fronts, max m/k, reference LU flops and LDL^T flops, bytes."""
        out = []
        for lt in self.levels:
            m = lt.front_m().astype(np.float64)
            k = lt.front_k().astype(np.float64)
            # sum_{i=1..k} (m-i) + 2 (m-i)^2   (reference task count)
            s1 = k * m - k * (k + 1) / 2
            s2 = k * m * m - m * k * (k + 1) + k * (k + 1) * (2 * k + 1) / 6
            lu_flops = float(np.sum(s1 + 2 * s2))
            # LDL^T on the lower triangle: per pivot (m-i) divisions + (m-i)(m-i+1) FMA-flops
            ldl_flops = float(np.sum(s1 + (s2 + s1)))
            fac_entries = float(np.sum(k * m - k * (k - 1) / 2))
            upd_entries = float(np.sum((m - k) * (m - k + 1) / 2))
            out.append(dict(level=lt.level, fronts=lt.n_fronts, max_m=lt.max_m, max_k=lt.max_k,
                            pivots=lt.n_pivots, lu_flops=lu_flops, ldl_flops=ldl_flops,
                            fac_entries=fac_entries, upd_entries=upd_entries))
        for L, st in enumerate(out):
            child_read = out[L - 1]["upd_entries"] if L > 0 else 0.0
            st["bytes"] = 8.0 * (child_read + st["fac_entries"] + st["upd_entries"])
        return out
