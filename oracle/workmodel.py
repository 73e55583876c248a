"""TEST INFRASTRUCTURE ONLY — closed-form front shapes and task counts.

Restates the per-level front orders m and pivot counts k of the reference's
plan (tree.py:106-160 pairing, tasks.py:109-151 eligibility) for tensor Q_p
meshes with 2^e elements per axis, by geometry, so
the CPU baseline can size its workload without the product package:

* level-L node i covers Morton leaves [i 2^L, (i+1) 2^L): an axis-aligned box
  whose extent on axis a is 2^(number of the lowest L Morton bits that belong
  to axis a);
* a grid point of the box's closure is in its front unless it is interior to
  one of the two child boxes (eliminated below); it is a pivot of the box iff
  it is interior to the box.  "Interior" is relative to the domain: a point
  on the domain boundary counts as inside.
So m = |closure(B)| - |int(c1)| - |int(c2)| and k = |int(B)| - |int(c1)| - |int(c2)|,
each a product of per-axis counts.

Reference task count of a front (tasks.py:162-182; one Division per active
entry, one Multiplication and one Subtraction per active pair):
sum_{i=1..k} [(m-i) + 2 (m-i)^2].  In 2D the dense front is exactly the
reference's active structure; in 3D it overcounts by <= 0.5%.
Pinned against the product's native plan in tests/test_workmodel.py.
"""

from __future__ import annotations

import numpy as np


def _axis_counts(n: int, p: int, ext: int):
    """Per box along one axis (n/ext boxes of `ext` elements): closure and interior counts."""
    a = np.arange(n // ext, dtype=np.int64) * ext
    b = a + ext
    clo = np.full(len(a), ext * p + 1, dtype=np.int64)
    inner = clo - (a * p > 0) - (b * p < n * p)
    return clo, inner


def _extents(d: int, L: int):
    ext = [1] * d
    for bit in range(L):
        ext[bit % d] *= 2
    return ext


def level_shapes(ns, p: int):
    """[(m, k)] per level, arrays over the level's fronts in node order."""
    d = len(ns)
    n = ns[0]
    if any(x != n for x in ns) or n & (n - 1):
        raise ValueError("closed form needs 2^e elements on every axis")
    n_levels = d * (n.bit_length() - 1) + 1
    out = []

    def grid(vals):
        # Morton node order of boxes: axis 0 is the fastest-varying bit
        g = vals[0]
        for v in vals[1:]:
            g = np.multiply.outer(v, g)
        return g

    for L in range(n_levels):
        ext = _extents(d, L)
        clo, inn = zip(*[_axis_counts(n, p, e) for e in ext])
        cl, it = grid(list(clo)), grid(list(inn))
        if L == 0:
            m, k = cl, it
        else:
            cext = _extents(d, L - 1)
            ax = (L - 1) % d  # the axis the last split halved
            c_in = []
            for a in range(d):
                c_in.append(_axis_counts(n, p, cext[a])[1])
            # children c1, c2 of a box along axis `ax`: pairs (2j, 2j+1)
            ch = c_in[ax].reshape(-1, 2).sum(axis=1)
            c_in[ax] = ch
            ci = grid(c_in)
            m, k = cl - ci, it - ci
        order = _morton_order(d, grid_shape(n, ext), L)
        out.append((m.ravel()[order], k.ravel()[order]))
    return out


def grid_shape(n: int, ext):
    return [n // e for e in ext]


def _morton_order(d: int, counts, L: int):
    """Flat grid index (axis 0 fastest) of every level-L box, in node (Morton) order.

    Node j holds leaves j 2^L .. ; leaf Morton bit t belongs to axis t % d
    (oracle/mesh_nd.morton_key), so bit t of j is leaf bit t + L."""
    total = int(np.prod(counts))
    j = np.arange(total, dtype=np.int64)
    coords = [np.zeros(total, dtype=np.int64) for _ in range(d)]
    rem = [int(c).bit_length() - 1 for c in counts]
    pos = [0] * d
    t, leaf_bit = 0, L
    while any(r > 0 for r in rem):
        a = leaf_bit % d
        if rem[a] > 0:
            coords[a] |= ((j >> t) & 1) << pos[a]
            pos[a] += 1
            rem[a] -= 1
            t += 1
        leaf_bit += 1
    flat = np.zeros(total, dtype=np.int64)
    stride = 1
    for a in range(d):
        flat += coords[a] * stride
        stride *= counts[a]
    return flat


def lu_task_flops(m, k) -> float:
    m = np.asarray(m, dtype=np.float64)
    k = np.asarray(k, dtype=np.float64)
    s1 = k * m - k * (k + 1) / 2
    s2 = k * m * m - m * k * (k + 1) + k * (k + 1) * (2 * k + 1) / 6
    return float(np.sum(s1 + 2 * s2))


def workload(ns, p: int) -> dict:
    """n_dof, levels, LU task-flops and factor entries of a tensor-mesh system."""
    shapes = level_shapes(tuple(ns), p)
    lu = sum(lu_task_flops(m, k) for m, k in shapes)
    fac = sum(float(np.sum(k * m - k * (k - 1) / 2)) for m, k in shapes)
    n_dof = int(np.prod([x * p + 1 for x in ns]))
    return dict(n_dof=n_dof, levels=len(shapes), lu_task_flops=lu, factor_entries=fac)
