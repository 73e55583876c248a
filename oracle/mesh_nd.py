"""TEST INFRASTRUCTURE ONLY — tensor-product FEM problem generator (oracle side).

Restates the reference's 1D element machinery and extends it to 2D/3D the
way SURVEY.md fact 2 prescribes:

* `element_mass_matrix_1d` follows fem.py:83-114 (equispaced Lagrange basis,
  (p+2)-point Gauss-Legendre on [0,1], M_e = h (B^T w) B).
* A d-dimensional Q_p element matrix is the Kronecker product of 1D matrices
  with the x-local node index fastest: kron(Mz, kron(My, Mx)).
* DOFs are numbered by the Morton (Z-order) index of their *owning* element;
  grid point i on an axis with n elements is owned by element min(i//p, n-1).
  Within one element, owned points are numbered lexicographically (z, y, x),
  x fastest.  Because Morton order is monotone in every coordinate, the
  minimum global index of element e is its first owned DOF, so the
  reference's `sort_fronts` (tree.py:44-48) reproduces Morton element order
  and pairwise joining (tree.py:131-137) is geometric nested dissection.
* For d = 1 this is exactly the reference numbering (fem.py:59-80): element
  e holds DOFs e*p+1 .. e*p+p+1.

Outputs are plain Python/numpy so the same description can be fed to the
reference (golden generation) and to the product package (tests).
"""

from __future__ import annotations

import numpy as np


def reference_basis(degree: int, xi: float) -> np.ndarray:
    """fem.py:83-96: equispaced Lagrange basis values at xi."""
    nodes = [k / degree for k in range(degree + 1)]
    out = np.empty(degree + 1)
    for k, xk in enumerate(nodes):
        v = 1.0
        for m, xm in enumerate(nodes):
            if m != k:
                v *= (xi - xm) / (xk - xm)
        out[k] = v
    return out


def element_mass_matrix_1d(width: float, degree: int) -> np.ndarray:
    """fem.py:97-114 (gauss_rule fem.py:97-105 inlined)."""
    pts, wts = np.polynomial.legendre.leggauss(degree + 2)
    xi, w = (pts + 1.0) / 2.0, wts / 2.0
    basis = np.array([reference_basis(degree, x) for x in xi])
    return width * (basis.T * w) @ basis


def element_matrix(ns: tuple[int, ...], degree: int) -> np.ndarray:
    """Q_p element mass matrix on the unit box, x-local index fastest."""
    mats = [element_mass_matrix_1d(1.0 / n, degree) for n in ns]
    out = mats[0]
    for m in mats[1:]:
        out = np.kron(m, out)
    return out


def morton_key(coords: tuple[int, ...]) -> int:
    """Interleave coordinate bits: bit b of axis a lands at position d*b + a."""
    d = len(coords)
    key = 0
    for b in range(max(1, max(c.bit_length() for c in coords))):
        for a, c in enumerate(coords):
            key |= ((c >> b) & 1) << (d * b + a)
    return key


def _lex_points(lo: tuple[int, ...], hi: tuple[int, ...]):
    """All integer points lo <= x < hi, lexicographic with axis 0 fastest."""
    d = len(lo)
    if d == 1:
        return [(i,) for i in range(lo[0], hi[0])]
    pts = []
    for rest in _lex_points(lo[1:], hi[1:]):
        for i in range(lo[0], hi[0]):
            pts.append((i,) + rest)
    return pts


def tensor_mesh(ns: tuple[int, ...], degree: int):
    """Elements in Morton order with their global DOFs (1-based, local order).

    Returns (n_dof, element_dofs, element_coords) where element_dofs[e] is the
    tuple of global DOFs of the e-th element (Morton order) in element-local
    order (x-local fastest), and element_coords[e] its (ex, ey, ...) tuple.
    """
    d = len(ns)
    p = degree
    coords = _lex_points((0,) * d, tuple(ns))
    coords.sort(key=morton_key)
    gid: dict[tuple[int, ...], int] = {}
    nxt = 1
    for ec in coords:
        lo = tuple(ec[a] * p for a in range(d))
        hi = tuple(ec[a] * p + p + (1 if ec[a] == ns[a] - 1 else 0) for a in range(d))
        for pt in _lex_points(lo, hi):
            gid[pt] = nxt
            nxt += 1
    n_dof = nxt - 1
    assert n_dof == int(np.prod([n * p + 1 for n in ns]))
    elems = []
    for ec in coords:
        lo = tuple(ec[a] * p for a in range(d))
        hi = tuple(ec[a] * p + p + 1 for a in range(d))
        elems.append(tuple(gid[pt] for pt in _lex_points(lo, hi)))
    return n_dof, elems, coords
