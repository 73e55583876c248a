"""TEST INFRASTRUCTURE ONLY — pure-Python restatement of the reference path.

Each function restates one reference function (file:line into
/root/reference/pkg/src/tracefront/) with the same arithmetic in the same
order, so its outputs are bitwise comparable with the golden vectors that
tests/golden/make_golden.py produced from the reference itself.  Intended
for small sizes (n_dof up to a few thousand).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

ZERO_PIVOT_RELATIVE = 1e-14  # engine.py:35


class OracleZeroPivot(ArithmeticError):
    def __init__(self, front: int, pivot: int):
        super().__init__(f"zero pivot at global index {pivot} (front {front})")
        self.front = front
        self.pivot = pivot


@dataclass
class Tree:
    levels: list[list[int]]  # node ids per level, leaves first
    indices: list[tuple[int, ...]]  # node id -> sorted front index tuple (leaves: as given)
    membership: list[dict[int, int]]  # node id -> {global index: count at its level}
    children: list[tuple[int, ...]]


def build_tree(leaf_indices: list[tuple[int, ...]]) -> Tree:
    """tree.py:44-48 (sort_fronts) + tree.py:106-160 (build_elimination_tree)."""
    order = sorted(range(len(leaf_indices)), key=lambda i: min(leaf_indices[i]))
    leaves = [tuple(leaf_indices[i]) for i in order]
    indices: list[tuple[int, ...]] = []
    membership: list[dict[int, int]] = []
    children: list[tuple[int, ...]] = []
    levels: list[list[int]] = []

    def with_membership(fronts):  # tree.py:88-103
        count: dict[int, int] = {}
        for f in fronts:
            for g in f:
                count[g] = count.get(g, 0) + 1
        return [{g: count[g] for g in f} for f in fronts]

    cur = []
    for f, mem in zip(leaves, with_membership(leaves)):
        cur.append(len(indices))
        indices.append(f)
        membership.append(mem)
        children.append(())
    levels.append(cur)
    while len(cur) > 1:
        nxt_f, nxt_c = [], []
        for i in range(0, len(cur) - 1, 2):  # tree.py:131-137
            a, b = cur[i], cur[i + 1]
            nxt_f.append(tuple(sorted(set(indices[a]) | set(indices[b]))))
            nxt_c.append((a, b))
        if len(cur) % 2 == 1:  # tree.py:138-149 carry node
            nxt_f.append(indices[cur[-1]])
            nxt_c.append((cur[-1],))
        cur = []
        for f, c, mem in zip(nxt_f, nxt_c, with_membership(nxt_f)):
            cur.append(len(indices))
            indices.append(f)
            membership.append(mem)
            children.append(c)
        levels.append(cur)
    return Tree(levels, indices, membership, children)


@dataclass
class Plan:
    steps: list[tuple[int, int, tuple[int, ...]]]  # (node_id, pivot, active)
    reorders: list[tuple[int, tuple[int, ...], tuple[int, ...], tuple[int, ...]]]
    cells: set[tuple[int, int]]
    n_dof: int

    @property
    def pivot_order(self):
        return tuple(s[1] for s in self.steps)


def symbolic(tree: Tree, lower_cells, n_dof: int) -> Plan:
    """tasks.py:88-159 (symbolic_eliminate)."""
    adj: dict[int, set[int]] = {g: set() for g in range(1, n_dof + 1)}
    cells: set[tuple[int, int]] = set()
    for (i, j) in lower_cells:
        cells.add((i, j))
        if i != j:
            cells.add((j, i))
            adj[i].add(j)
            adj[j].add(i)
    eliminated: set[int] = set()
    steps, reorders = [], []
    last = len(tree.levels) - 1
    for level, ids in enumerate(tree.levels):
        for nid in ids:
            idx = tree.indices[nid]
            mem = tree.membership[nid]
            elim = sorted(g for g in idx if g not in eliminated and (mem[g] == 1 or level == last))
            es = set(elim)
            shared = sorted(g for g in idx if g not in eliminated and g not in es)
            done = sorted(g for g in idx if g in eliminated)
            reorders.append((nid, tuple(elim), tuple(shared), tuple(done)))
            iset = set(idx)
            for z in elim:
                if (z, z) not in cells:
                    raise ValueError(f"symbolic singularity at {z}")
                active = sorted(h for h in adj[z] if h not in eliminated)
                if any(h not in iset for h in active):
                    raise AssertionError(f"pivot {z} couples outside front {nid}")
                steps.append((nid, z, tuple(active)))
                for a in active:
                    cells.add((a, a))
                    for b in active:
                        if b != a and b not in adj[a]:
                            adj[a].add(b)
                            cells.add((a, b))
                eliminated.add(z)
    return Plan(steps, reorders, cells, n_dof)


def nested_loops(tree: Tree, entries: dict[tuple[int, int], float], n_dof: int):
    """engine.py:500-552 (factorize_nested_loops), same per-cell op order.

    Row/column neighbour discovery (engine.py:531-536 scans the values dict)
    is restated with per-row key sets; the visited sets are identical.
    """
    values: dict[tuple[int, int], float] = {}
    rows: dict[int, set[int]] = {}
    cols: dict[int, set[int]] = {}

    def put(key, v):
        if key not in values:
            rows.setdefault(key[0], set()).add(key[1])
            cols.setdefault(key[1], set()).add(key[0])
        values[key] = v

    for (i, j), v in entries.items():  # fem.py:153-158 symmetric_items
        put((i, j), v)
        if i != j:
            put((j, i), v)
    peak = max((abs(v) for v in entries.values()), default=0.0)
    threshold = ZERO_PIVOT_RELATIVE * peak
    eliminated: set[int] = set()
    u: dict[tuple[int, int], float] = {}
    l: dict[tuple[int, int], float] = {}
    order: list[int] = []
    last = len(tree.levels) - 1
    for level, ids in enumerate(tree.levels):
        for nid in ids:
            mem = tree.membership[nid]
            eligible = sorted(
                g for g in tree.indices[nid]
                if g not in eliminated and (mem[g] == 1 or level == last)
            )
            for z in eligible:
                pv = values.get((z, z), 0.0)
                if abs(pv) <= threshold:
                    raise OracleZeroPivot(nid, z)
                row = sorted(y for y in rows.get(z, ()) if y != z and y not in eliminated)
                col = sorted(x for x in cols.get(z, ()) if x != z and x not in eliminated)
                for y in row:
                    q = values[(z, y)] / pv
                    u[(z, y)] = q
                    for x in col:
                        prod = q * values[(x, z)]
                        put((x, y), values.get((x, y), 0.0) - prod)
                u[(z, z)] = pv
                for x in col:
                    l[(x, z)] = values[(x, z)] / pv
                order.append(z)
                eliminated.add(z)
    return values, u, l, tuple(order)


def solve(u, l, pivot_order, rhs: np.ndarray) -> np.ndarray:
    """engine.py:468-493 (solve), single right-hand side."""
    lower_cols: dict[int, list] = {}
    for (x, z), v in l.items():
        lower_cols.setdefault(z, []).append((x, v))
    upper_rows: dict[int, list] = {}
    for (z, y), v in u.items():
        if z != y:
            upper_rows.setdefault(z, []).append((y, v))
    b = np.array(rhs, dtype=float).copy()
    for z in pivot_order:
        bz = b[z - 1]
        for x, v in lower_cols.get(z, ()):
            b[x - 1] -= v * bz
    for z in pivot_order:
        b[z - 1] /= u[(z, z)]
    for z in reversed(pivot_order):
        acc = b[z - 1]
        for y, q in upper_rows.get(z, ()):
            acc -= q * b[y - 1]
        b[z - 1] = acc
    return b


# --------------------------------------------------------------------------
# atomic task graph + canonical FNF (tasks.py:162-252, schedule.py:60-82)

DIV, MUL, SUB, ASSERT = 1, 2, 3, 4


def task_graph(plan: Plan):
    """Returns (tasks, succs): tasks as (kind, front, pivot, row, col)."""
    tasks = [(ASSERT, -1, -1, x, y) for (x, y) in sorted(plan.cells)]
    for (f, z, active) in plan.steps:
        tasks += [(DIV, f, z, z, y) for y in active]
        tasks += [(MUL, f, z, x, y) for x in active for y in active]
        tasks += [(SUB, f, z, x, y) for x in active for y in active]
    succs: list[list[int]] = [[] for _ in tasks]
    n_as = len(plan.cells)
    aid = {t[3:]: i for i, t in enumerate(tasks[:n_as])}
    last_sub: dict[tuple[int, int], int] = {}
    tid = n_as
    for (f, z, active) in plan.steps:
        n, div_base = len(active), tid
        rank = {y: k for k, y in enumerate(active)}
        for y in active:
            succs[aid[(z, y)]].append(tid)
            succs[aid[(z, z)]].append(tid)
            tid += 1
        mul_base = tid
        for x in active:
            for y in active:
                succs[div_base + rank[y]].append(tid)
                succs[aid[(x, z)]].append(tid)
                tid += 1
        for k, x in enumerate(active):
            for m, y in enumerate(active):
                succs[mul_base + k * n + m].append(tid)
                prev = last_sub.get((x, y))
                if prev is not None:
                    succs[prev].append(tid)
                last_sub[(x, y)] = tid
                tid += 1
    for cell, s in last_sub.items():
        succs[s].append(aid[cell])
    return tasks, succs


def fnf_classes(tasks, succs) -> list[int]:
    """schedule.py:60-82: class(t) = 1 + max class(pred), via Kahn order."""
    n = len(tasks)
    indeg = [0] * n
    for s in succs:
        for v in s:
            indeg[v] += 1
    ready = [i for i in range(n) if indeg[i] == 0]
    cls = [1] * n
    seen = 0
    while ready:
        nxt = []
        for u_ in ready:
            seen += 1
            for v in succs[u_]:
                if cls[u_] + 1 > cls[v]:
                    cls[v] = cls[u_] + 1
                indeg[v] -= 1
                if indeg[v] == 0:
                    nxt.append(v)
        ready = nxt
    if seen != n:
        raise AssertionError("cycle")
    return cls
