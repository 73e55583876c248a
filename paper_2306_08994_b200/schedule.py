"""Foata Normal Form schedule at front granularity (mirrors schedule.py:1-128).

The reference builds the FNF of its atomic trace (Division / Multiplication /
Subtraction / Assertion tasks, schedule.py:60-82).  This package schedules
the coarser trace whose letters are whole front factorizations
(extend-add + partial factorization of one tree node) and whose dependency
relation is child -> parent.  Its canonical FNF is exactly the tree levels:
class(L) = 1 + max class(children) = L + 1.  Every atomic J-edge of the
reference goes from a level to the same or a later level, so executing the
level classes in order (one GPU launch sequence per class, stream order as
the barrier) is a valid linearization of the reference's Diekert graph
(every J1-J4 edge of the restated atomic graph is level-nondecreasing:
tests/test_schedule.py).
"""

from __future__ import annotations

from dataclasses import dataclass
from enum import IntEnum

import numpy as np


class TaskKind(IntEnum):
    DIVISION = 1
    MULTIPLICATION = 2
    SUBTRACTION = 3
    ASSERTION = 4


@dataclass(frozen=True)
class FoataSchedule:
    """Ordered Foata classes of front tasks; class c holds the node ids of level c-1."""

    classes: tuple  # tuple of node-id ranges, leaves first
    class_kinds: tuple[frozenset, ...]
    level_sizes: tuple[int, ...]

    @property
    def n_classes(self) -> int:
        return len(self.classes)

    def class_of(self, node_id: int) -> int:
        for c, r in enumerate(self.classes):
            if node_id in r:
                return c + 1
        raise KeyError(node_id)


@dataclass(frozen=True)
class ScheduleStats:
    n_classes: int
    widths: tuple[int, ...]
    kinds: tuple[frozenset, ...]
    max_width: int
    mixed_classes: tuple[int, ...]


def compute_fnf(plan_or_graph):
    """Canonical FNF (schedule.py:60-82).

    Given a `DependencyGraph` (the reference's call, cli.py:149) this is the
    FNF of the atomic trace, as statistics (`AtomicFoataSchedule`: class
    widths and kind sets equal the reference's).  Given an `EliminationPlan`
    it is the FNF of the front-granularity trace the GPU executes: one class
    per tree level.
    """
    from .tasks import DependencyGraph
    if isinstance(plan_or_graph, DependencyGraph):
        return compute_atomic_fnf(plan_or_graph.plan)
    plan = plan_or_graph
    native = plan.native
    kinds = []
    for lt in native.levels:
        m, k = lt.front_m(), lt.front_k()
        ks = {TaskKind.ASSERTION}
        if np.any(k > 0):
            ks.add(TaskKind.DIVISION)
            if np.any((m - 1) > 0):
                ks |= {TaskKind.MULTIPLICATION, TaskKind.SUBTRACTION}
        kinds.append(frozenset(ks))
    return FoataSchedule(classes=tuple(plan.tree.levels), class_kinds=tuple(kinds),
                         level_sizes=tuple(plan.tree.level_sizes))


@dataclass(frozen=True)
class AtomicFoataSchedule:
    """Canonical FNF of the reference's atomic trace (schedule.py:60-82), as statistics.

    Computed natively (`tf_atomic_fnf`, csrc/symbolic.cpp) by streaming the
    Diekert graph of tasks.py:162-252 in elimination order; per-task class
    lists are not materialised.  `widths[c]` and `class_kinds[c]` equal
    `len(compute_fnf(graph).classes[c])` and `class_kinds[c]` of the reference.
    """

    n_tasks: int
    n_edges: int
    n_cells: int
    kind_counts: dict
    widths: tuple[int, ...]
    class_kinds: tuple[frozenset, ...]

    @property
    def n_classes(self) -> int:
        return len(self.widths)

    @property
    def level_sizes(self) -> tuple[int, ...]:
        return self.widths


def compute_atomic_fnf(plan) -> AtomicFoataSchedule:
    """Atomic-granularity FNF statistics of `plan` (needs a plan small enough to keep node lists)."""
    st, widths, kinds = plan.native.atomic_fnf()
    ks = tuple(frozenset(k for k in TaskKind if int(m) >> (int(k) - 1) & 1) for m in kinds)
    return AtomicFoataSchedule(n_tasks=int(st.n_tasks), n_edges=int(st.n_edges),
                               n_cells=int(st.n_cells),
                               kind_counts={TaskKind.DIVISION: int(st.n_divisions),
                                            TaskKind.MULTIPLICATION: int(st.n_multiplications),
                                            TaskKind.SUBTRACTION: int(st.n_multiplications),
                                            TaskKind.ASSERTION: int(st.n_cells)},
                               widths=tuple(int(w) for w in widths), class_kinds=ks)


def schedule_stats(schedule) -> ScheduleStats:
    widths = tuple(schedule.level_sizes)
    mixed = tuple(i + 1 for i, ks in enumerate(schedule.class_kinds)
                  if TaskKind.DIVISION in ks and TaskKind.SUBTRACTION in ks)
    return ScheduleStats(n_classes=schedule.n_classes, widths=widths,
                         kinds=schedule.class_kinds, max_width=max(widths) if widths else 0,
                         mixed_classes=mixed)


def schedule_stats_csv(schedule) -> str:
    lines = ["class_index,kind_set,size"]
    for i, (w, ks) in enumerate(zip(schedule.level_sizes, schedule.class_kinds)):
        lines.append(f"{i + 1},{'|'.join(sorted(k.name.lower() for k in ks))},{w}")
    return "\n".join(lines) + "\n"
