"""Symbolic elimination plan (mirrors tasks.py:49-159).

`symbolic_eliminate(tree, system)` returns an `EliminationPlan` whose pivot
order and per-node `NodeReorder`s come from the native plan the tree already
built.  The reference's per-pivot `PivotStep.active` sets (and the stored
cell / fill sets) are produced on demand, for small plans, by a boolean
simulation of the same dense fronts the GPU factors: a front's pattern is the
OR of its children's update patterns, and eliminating a pivot ORs the outer
product of its column into the trailing block (tasks.py:142-150's fill
clique).  This gives exactly the reference's active sets because every
coupling of a pivot lies inside its own subtree.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from typing import Optional

import numpy as np

from . import _lib
from .errors import SymbolicSingularityError
from .tree import MATERIALIZE_LIMIT, EliminationTree


@dataclass(frozen=True)
class PivotStep:
    node_id: int
    pivot: int
    active: tuple[int, ...]


@dataclass(frozen=True)
class NodeReorder:
    node_id: int
    eliminable: tuple[int, ...]
    shared: tuple[int, ...]
    computed: tuple[int, ...]


class EliminationPlan:
    """Output of symbolic elimination over the whole tree (tasks.py:73-85)."""

    def __init__(self, tree: EliminationTree, system=None):
        self.tree = tree
        self.native = tree.plan
        self.system = system
        self.n_dof = int(system.n_dof) if system is not None else tree.n_dof

    # ---- pivot order -------------------------------------------------------------
    @property
    def pivot_order_array(self) -> np.ndarray:
        return self.native.pivot_order

    @cached_property
    def pivot_order(self) -> tuple[int, ...]:
        return tuple(int(z) for z in self.native.pivot_order)

    @property
    def n_levels(self) -> int:
        return self.native.n_levels

    def level_stats(self) -> list[dict]:
        return self.native.level_stats()

    def locate_pivot(self, pos: int) -> tuple[int, int]:
        """Pivot-order position -> (tree node id, global pivot index)."""
        for lt in self.native.levels:
            if lt.piv_base <= pos < lt.piv_base + lt.n_pivots:
                f = int(np.searchsorted(lt.piv_off, pos, side="right")) - 1
                return lt.node_base + f, int(self.native.pivot_order[pos])
        raise IndexError(pos)

    # ---- reference-shaped views (small plans) ------------------------------------
    def _require_small(self):
        if not self.native.keep_lists:
            raise MemoryError("plan too large for per-node materialisation")

    @cached_property
    def reorders(self) -> tuple[NodeReorder, ...]:
        """NodeReorder per node in visit order (tasks.py:119-130)."""
        self._require_small()
        nodes = self.tree.nodes
        out = []
        eliminated: set[int] = set()
        for L in range(self.n_levels):
            ptr, k, idx = self.native.node_lists(L)
            base = self.native.levels[L].node_base
            newly = []
            for i in range(len(k)):
                nid = base + i
                lst = idx[ptr[i]:ptr[i + 1]]
                elim = tuple(int(g) for g in lst[:k[i]])
                shared = tuple(int(g) for g in lst[k[i]:])
                done = tuple(g for g in nodes[nid].front.indices if g in eliminated)
                out.append(NodeReorder(nid, elim, shared, tuple(sorted(done))))
                newly.extend(elim)
            eliminated.update(newly)
        return tuple(out)

    @cached_property
    def _structure(self):
        """Boolean dense-front simulation -> (steps, cells, fill)."""
        self._require_small()
        steps: list[PivotStep] = []
        upd_pat: list[np.ndarray] = []
        cells: set[tuple[int, int]] = set()
        prev = None
        for L in range(self.n_levels):
            lt = self.native.levels[L]
            ptr, kk, idx = self.native.node_lists(L)
            cur = []
            for i in range(lt.n_fronts):
                row = lt.pat[lt.pattern_of[i]]
                m, k, nsrc = row[_lib.PAT_M], row[_lib.PAT_K], row[_lib.PAT_NSRC]
                B = np.zeros((m, m), dtype=bool)
                if L == 0:
                    mp = lt.maps[row[_lib.PAT_OFF0]: row[_lib.PAT_OFF0] + row[_lib.PAT_LEN0]]
                    B[np.ix_(mp, mp)] = True
                else:
                    for c in range(nsrc):
                        off = row[_lib.PAT_OFF0 + c]
                        mp = lt.maps[off: off + row[_lib.PAT_LEN0 + c]]
                        B[np.ix_(mp, mp)] |= prev[2 * i + c]
                lst = idx[ptr[i]:ptr[i + 1]]
                nid = lt.node_base + i
                for c in range(k):
                    if not B[c, c]:
                        raise SymbolicSingularityError(int(lst[c]))
                    nz = np.nonzero(B[c, c + 1:])[0] + c + 1
                    steps.append(PivotStep(nid, int(lst[c]), tuple(int(g) for g in np.sort(lst[nz]))))
                    B[np.ix_(nz, nz)] = True
                    B[nz, nz] = True
                cur.append(B[k:, k:].copy())
            prev = cur
        # every stored cell = original pattern + fill cliques of every step
        system = self.system
        orig: set[tuple[int, int]] = set()
        if system is not None and len(self.tree.fronts) <= MATERIALIZE_LIMIT:
            for (i, j), _ in system.symmetric_items():
                orig.add((i, j))
        cells |= orig
        for s in steps:
            z = s.pivot
            cells.add((z, z))
            for a in s.active:
                cells.add((z, a))
                cells.add((a, z))
                for b in s.active:
                    cells.add((a, b))
        return tuple(steps), frozenset(cells), frozenset(cells - orig)

    @property
    def steps(self) -> tuple[PivotStep, ...]:
        return self._structure[0]

    @property
    def cells(self):
        return self._structure[1]

    @property
    def fill_cells(self):
        return self._structure[2]


def symbolic_eliminate(tree: EliminationTree, system=None) -> EliminationPlan:
    """Plan every pivot elimination over the tree (tasks.py:88-159)."""
    return EliminationPlan(tree, system)
