"""The reference's atomic task graph at the Python boundary (tasks.py:32-360).

The GPU path never executes this graph: it runs the front-granularity level
schedule, which tests/test_schedule.py proves is a linearization of it.  The
graph is still part of the reference's API -- `cli._build_pipeline` calls
`build_dependency_edges(enumerate_tasks(plan), plan)` and hands the result to
`compute_fnf`, `validate_dag`, `run_sequential` and `run_concurrent`
(cli.py:142-161, 184-195) -- so the same calls work here:

* `enumerate_tasks(plan)` returns a `TaskAlphabet`: a lazy sequence in the
  reference's canonical order (assertions of the sorted cells, then per
  pivot step its divisions, multiplications, subtractions; tasks.py:162-182).
  Its length and kind counts come from the native streamed graph
  (`tf_atomic_fnf`); tasks are materialised only when indexed / iterated.
* `build_dependency_edges(tasks, plan)` returns a `DependencyGraph` whose
  `plan`, `n_tasks`, `n_edges` and Foata statistics are native; `preds` and
  `succs` (the J1-J4 wiring of tasks.py:207-252) are built on first access,
  for plans small enough to keep per-node lists.
* `validate_dag(graph)` reports kind counts and the longest path (= number of
  atomic Foata classes, computed by the streamed FNF).  A plan's graph is
  acyclic by construction: every J1-J4 edge is level-nondecreasing and, inside
  a level, advances the atomic Foata class (tests/test_schedule.py), so `ok`
  is always True here; a symbolically singular plan raises
  SymbolicSingularityError from the native FNF instead.
"""

from __future__ import annotations

from collections.abc import Sequence
from dataclasses import dataclass
from functools import cached_property
from typing import NamedTuple, Optional

from .schedule import TaskKind
from .symbolic import EliminationPlan, symbolic_eliminate


class Task(NamedTuple):
    """One atomic operation (tasks.py:38-46); front and pivot are -1 for assertions."""

    kind: TaskKind
    front: int
    pivot: int
    row: int
    col: int


def _stats(plan: EliminationPlan):
    cached = getattr(plan, "_atomic_stats", None)
    if cached is None:
        cached = plan.native.atomic_fnf()
        plan._atomic_stats = cached
    return cached


class TaskAlphabet(Sequence):
    """Lazy canonical task list of a plan (tasks.py:162-182)."""

    def __init__(self, plan: EliminationPlan):
        self.plan = plan

    def __len__(self) -> int:
        return int(_stats(self.plan)[0].n_tasks)

    @cached_property
    def _list(self) -> list[Task]:
        plan = self.plan
        out = [Task(TaskKind.ASSERTION, -1, -1, x, y) for (x, y) in sorted(plan.cells)]
        for st in plan.steps:
            f, z, act = st.node_id, st.pivot, st.active
            out.extend(Task(TaskKind.DIVISION, f, z, z, y) for y in act)
            out.extend(Task(TaskKind.MULTIPLICATION, f, z, x, y) for x in act for y in act)
            out.extend(Task(TaskKind.SUBTRACTION, f, z, x, y) for x in act for y in act)
        return out

    def __getitem__(self, i):
        return self._list[i]

    def __iter__(self):
        return iter(self._list)

    def kind_counts(self) -> dict:
        st = _stats(self.plan)[0]
        return {TaskKind.DIVISION: int(st.n_divisions),
                TaskKind.MULTIPLICATION: int(st.n_multiplications),
                TaskKind.SUBTRACTION: int(st.n_multiplications),
                TaskKind.ASSERTION: int(st.n_cells)}


def enumerate_tasks(plan: EliminationPlan) -> TaskAlphabet:
    """The task alphabet in canonical order (tasks.py:162-182)."""
    return TaskAlphabet(plan)


class DependencyGraph:
    """Dependency DAG over the task alphabet (tasks.py:185-204)."""

    def __init__(self, tasks: TaskAlphabet, plan: EliminationPlan):
        self.tasks = tasks
        self.plan = plan

    @property
    def n_tasks(self) -> int:
        return len(self.tasks)

    @property
    def n_edges(self) -> int:
        return int(_stats(self.plan)[0].n_edges)

    @cached_property
    def _adjacency(self):
        """J1-J4 (tasks.py:207-252), replayed over the canonical layout."""
        plan = self.plan
        n = self.n_tasks
        preds: list[list[int]] = [[] for _ in range(n)]
        succs: list[list[int]] = [[] for _ in range(n)]

        def edge(a: int, b: int) -> None:
            succs[a].append(b)
            preds[b].append(a)

        cells = sorted(plan.cells)
        aid = {c: i for i, c in enumerate(cells)}
        chain_end: dict[tuple[int, int], int] = {}
        t = len(cells)
        for st in plan.steps:
            z, act = st.pivot, st.active
            a = len(act)
            div0, mul0, sub0 = t, t + a, t + a + a * a
            for j, y in enumerate(act):          # J1
                edge(aid[(z, y)], div0 + j)
                edge(aid[(z, z)], div0 + j)
            for i, x in enumerate(act):          # J2
                for j in range(a):
                    edge(div0 + j, mul0 + i * a + j)
                    edge(aid[(x, z)], mul0 + i * a + j)
            for i, x in enumerate(act):          # J3
                for j, y in enumerate(act):
                    s = sub0 + i * a + j
                    edge(mul0 + i * a + j, s)
                    if (x, y) in chain_end:
                        edge(chain_end[(x, y)], s)
                    chain_end[(x, y)] = s
            t = sub0 + a * a
        for cell, s in chain_end.items():      # J4
            edge(s, aid[cell])
        return preds, succs

    @property
    def preds(self) -> list[list[int]]:
        return self._adjacency[0]

    @property
    def succs(self) -> list[list[int]]:
        return self._adjacency[1]


def build_dependency_edges(tasks, plan: EliminationPlan) -> DependencyGraph:
    """Wire J1-J4 into one DAG (tasks.py:207-252)."""
    if not isinstance(tasks, TaskAlphabet):
        tasks = TaskAlphabet(plan)
    return DependencyGraph(tasks, plan)


def build_task_graph(tree, system) -> DependencyGraph:
    """symbolic_eliminate + enumerate_tasks + build_dependency_edges (tasks.py:360-363)."""
    plan = symbolic_eliminate(tree, system)
    return build_dependency_edges(enumerate_tasks(plan), plan)


@dataclass(frozen=True)
class DagReport:
    """tasks.py:255-260."""

    ok: bool
    kind_counts: dict
    longest_path: int
    cycle: Optional[tuple] = None


def validate_dag(graph: DependencyGraph) -> DagReport:
    """Kind counts and longest path (tasks.py:309-330), from the native streamed graph."""
    st, widths, _ = _stats(graph.plan)
    return DagReport(ok=True, kind_counts=graph.tasks.kind_counts(),
                     longest_path=int(st.n_classes) if st.n_tasks else 0)


__all__ = ["Task", "TaskKind", "TaskAlphabet", "DependencyGraph", "DagReport", "EliminationPlan",
           "build_dependency_edges", "build_task_graph", "enumerate_tasks", "symbolic_eliminate",
           "validate_dag"]
