"""Balanced binary elimination tree by pairwise joining (mirrors tree.py:1-186).

`build_elimination_tree` hands the sorted leaf fronts to the native symbolic
layer (libtfb200 `tf_plan_create`), which uses the identity "leaf j's
ancestor at level L is node j >> L" of the reference's pairing rule
(tree.py:131-149) instead of materialising merged index unions.  Reference
node ids (leaves 0..n-1, then level by level, tree.py:133,153) are kept, and
`EliminationTree.nodes` materialises reference-identical `TreeNode`s on
demand for small trees.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import cached_property
from typing import Optional, Sequence, Union

import numpy as np

from .errors import EmptyInputError
from .fem import Front, FrontSet
from .plan import NativePlan

MATERIALIZE_LIMIT = 200_000  # leaves up to which reference-style node objects are built


@dataclass(frozen=True)
class TreeNode:
    node_id: int
    level: int
    front: Front
    children: tuple[int, ...]


def _n_dof_of(fronts: FrontSet) -> int:
    return int(fronts.dofs.max()) if fronts.dofs.size else 0


def sort_fronts(fronts: Union[Sequence[Front], FrontSet]):
    """Stable ascending sort by minimum global index (tree.py:44-48)."""
    if len(fronts) == 0:
        raise EmptyInputError("no fronts to sort")
    if isinstance(fronts, FrontSet):
        mins = fronts.min_indices()
        if np.all(mins[1:] >= mins[:-1]):
            return fronts
        return fronts.take(np.argsort(mins, kind="stable"))
    return sorted(fronts, key=lambda f: f.min_index)


def join_fronts(left: Front, right: Front, new_id: int = -1,
                with_values: Optional[bool] = None) -> Front:
    """Merge two same-level fronts over the union of their indices (tree.py:51-85)."""
    union = sorted(left.index_set | right.index_set)
    pos = {g: k for k, g in enumerate(union)}
    computed = np.zeros(len(union), dtype=bool)
    for src in (left, right):
        idx = [pos[g] for g in src.indices]
        computed[idx] |= np.asarray(src.computed, dtype=bool)
    if with_values is None:
        with_values = left.values is not None and right.values is not None
    values = None
    if with_values:
        values = np.zeros((len(union), len(union)))
        for src in (left, right):
            idx = [pos[g] for g in src.indices]
            values[np.ix_(idx, idx)] += src.values
    return Front(front_id=new_id, indices=tuple(union), membership=(1,) * len(union),
                 computed=tuple(bool(c) for c in computed), values=values)


class EliminationTree:
    """Elimination tree over leaf fronts (tree.py:28-41), backed by a NativePlan."""

    def __init__(self, fronts: FrontSet, n_dof: Optional[int] = None, keep_lists: bool = None,
                 cache_dir=None):
        self.fronts = fronts
        self.n_dof = _n_dof_of(fronts) if n_dof is None else int(n_dof)
        if keep_lists is None:
            keep_lists = len(fronts) <= MATERIALIZE_LIMIT
        self.plan = NativePlan(fronts, self.n_dof, keep_lists=keep_lists, cache_dir=cache_dir)
        sizes = [lt.n_fronts for lt in self.plan.levels]
        bases = np.concatenate([[0], np.cumsum(sizes)])
        self.level_sizes = tuple(sizes)
        self.levels = tuple(range(int(bases[L]), int(bases[L + 1])) for L in range(len(sizes)))
        self.root_id = int(bases[-1]) - 1

    @property
    def n_levels(self) -> int:
        return len(self.levels)

    @property
    def n_leaves(self) -> int:
        return len(self.levels[0])

    def level_of(self, node_id: int) -> int:
        for L, r in enumerate(self.levels):
            if node_id in r:
                return L
        raise KeyError(node_id)

    @cached_property
    def nodes(self) -> tuple[TreeNode, ...]:
        """Reference-identical TreeNodes (tree.py:106-160 output), small trees only."""
        if self.n_leaves > MATERIALIZE_LIMIT:
            raise MemoryError("tree too large to materialise per-node Front objects")
        idx_sets: list[tuple[int, ...]] = []
        children: list[tuple[int, ...]] = []
        for i in range(self.n_leaves):
            idx_sets.append(tuple(int(g) for g in self.fronts.dofs_of(i)))
            children.append(())
        prev = list(self.levels[0])
        for L in range(1, self.n_levels):
            cur = list(self.levels[L])
            for i, nid in enumerate(cur):
                kids = tuple(prev[2 * i: 2 * i + 2])
                if len(kids) == 2:
                    idx_sets.append(tuple(sorted(set(idx_sets[kids[0]]) | set(idx_sets[kids[1]]))))
                else:
                    idx_sets.append(idx_sets[kids[0]])
                children.append(kids)
            prev = cur
        # per-level membership (tree.py:88-103); `computed` is never set True by the
        # reference (generate_fronts starts it False and join_fronts only ORs it)
        out = []
        for L, ids in enumerate(self.levels):
            count: dict[int, int] = {}
            for nid in ids:
                for g in idx_sets[nid]:
                    count[g] = count.get(g, 0) + 1
            for nid in ids:
                ind = idx_sets[nid]
                vals = None
                if L == 0:
                    vals = np.array(self.fronts.values_of(nid), copy=True)
                front = Front(front_id=nid, indices=ind, membership=tuple(count[g] for g in ind),
                              computed=(False,) * len(ind),
                              values=vals)
                out.append(TreeNode(node_id=nid, level=L, front=front, children=children[nid]))
        return tuple(out)


def build_elimination_tree(fronts: Union[Sequence[Front], FrontSet],
                           n_dof: Optional[int] = None) -> EliminationTree:
    """Pair consecutive fronts level by level until one root remains (tree.py:106-160).

    Input fronts must already be sorted (as in the reference).
    """
    if len(fronts) == 0:
        raise EmptyInputError("cannot build a tree from zero fronts")
    fs = fronts if isinstance(fronts, FrontSet) else FrontSet.from_fronts(list(fronts))
    return EliminationTree(fs, n_dof=n_dof)


def tree_level_listing(tree: EliminationTree) -> str:
    """Per-level node listing with index spans (tree.py:163-186 analogue)."""
    lines = []
    for L, ids in enumerate(tree.levels):
        parts = []
        for nid in ids:
            ind = tree.nodes[nid].front.indices
            parts.append(f"{nid}[{min(ind)}..{max(ind)}]")
        lines.append(f"level {L}: " + " ".join(parts))
    return "\n".join(lines) + "\n"
