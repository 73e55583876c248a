"""FEM problem generation: meshes, Lagrange bases, element mass matrices, fronts.

Mirrors the reference module fem.py (1D `Mesh`, `Front`, `GlobalSystem`,
`assemble_system`, `generate_fronts`; fem.py:39-259) and extends it to
tensor-product Q_p meshes in 2D/3D (`TensorMesh`), whose DOFs are numbered by
the Morton index of their owning element so that the
reference's own `sort_fronts` + pairwise joining yields nested dissection.

Large meshes never materialise per-front Python objects: `generate_fronts`
returns a `FrontSet`, an array-backed sequence of `Front`s (element DOF table
plus element matrices), and `assemble_system` on a `TensorMesh` returns an
`ElementSystem` whose dictionary entries are built only on demand.
Global DOF indices are 1-based everywhere (fem.py:8-9).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np

from .errors import InvalidGeometryError, UnsupportedDegreeError

SUPPORTED_DEGREES = (1, 2, 3)

RHS_FUNCTIONS: dict[str, Callable[[float], float]] = {
    "one": lambda x: 1.0,
    "sin_pi": lambda x: math.sin(math.pi * x),
    "x_squared": lambda x: x * x,
}


def _check_degree(degree: int) -> None:
    if degree not in SUPPORTED_DEGREES:
        raise UnsupportedDegreeError(f"degree must be one of {SUPPORTED_DEGREES}, got {degree}")


# ---------------------------------------------------------------------------
# 1D element machinery (fem.py:83-130)


def reference_basis(degree: int, xi) -> np.ndarray:
    """Equispaced Lagrange basis values at xi (scalar or array) on [0, 1].

    Same product order as fem.py:83-96, vectorised over xi.
    """
    _check_degree(degree)
    x = np.asarray(xi, dtype=float)
    nodes = [k / degree for k in range(degree + 1)]
    vals = []
    for k, xk in enumerate(nodes):
        v = np.ones_like(x)
        for j, xj in enumerate(nodes):
            if j != k:
                v = v * ((x - xj) / (xk - xj))
        vals.append(v)
    return np.stack(vals, axis=-1)


def gauss_rule(degree: int) -> tuple[np.ndarray, np.ndarray]:
    """(p+2)-point Gauss-Legendre rule mapped to [0, 1] (fem.py:97-105)."""
    pts, wts = np.polynomial.legendre.leggauss(degree + 2)
    return (pts + 1.0) / 2.0, wts / 2.0


def element_mass_matrix(width: float, degree: int) -> np.ndarray:
    """(p+1)x(p+1) Gram matrix of the basis over one element (fem.py:107-114)."""
    _check_degree(degree)
    if width <= 0:
        raise InvalidGeometryError(f"element width must be positive, got {width}")
    xi, w = gauss_rule(degree)
    basis = reference_basis(degree, xi)  # n_q x (p+1)
    return width * (basis.T * w) @ basis


def element_load_vector(width: float, degree: int, f: Callable[[float], float],
                        element_offset: float) -> np.ndarray:
    """Moments of f against the element basis (fem.py:117-130)."""
    _check_degree(degree)
    if width <= 0:
        raise InvalidGeometryError(f"element width must be positive, got {width}")
    xi, w = gauss_rule(degree)
    basis = reference_basis(degree, xi)
    fvals = np.array([f(element_offset + x * width) for x in xi])
    return width * basis.T @ (w * fvals)


# ---------------------------------------------------------------------------
# meshes


@dataclass(frozen=True)
class Mesh:
    """Uniform 1D mesh; element e owns DOFs e*p+1 .. e*p+p+1 (fem.py:39-80)."""

    n_elements: int
    degree: int
    domain_start: float = 0.0
    domain_end: float = 1.0

    def __post_init__(self) -> None:
        if self.n_elements < 1:
            raise InvalidGeometryError(f"n_elements must be >= 1, got {self.n_elements}")
        _check_degree(self.degree)
        if not self.domain_start < self.domain_end:
            raise InvalidGeometryError(f"empty domain [{self.domain_start}, {self.domain_end}]")

    dim = 1

    @property
    def n_dof(self) -> int:
        return self.degree * self.n_elements + 1

    @property
    def element_width(self) -> float:
        return (self.domain_end - self.domain_start) / self.n_elements

    def element_dofs(self, element: int) -> tuple[int, ...]:
        base = element * self.degree
        return tuple(range(base + 1, base + self.degree + 2))

    def element_offset(self, element: int) -> float:
        return self.domain_start + element * self.element_width

    def dof_coordinate(self, dof: int) -> float:
        return self.domain_start + (dof - 1) / self.degree * self.element_width

    def element_table(self) -> np.ndarray:
        """(n_elements, p+1) int32 table of 1-based DOFs."""
        e = np.arange(self.n_elements, dtype=np.int64)[:, None] * self.degree
        return (e + np.arange(1, self.degree + 2)).astype(np.int32)

    def element_matrix(self) -> np.ndarray:
        return element_mass_matrix(self.element_width, self.degree)


@dataclass(frozen=True, eq=False)
class TensorMesh:
    """Tensor-product Q_p mesh of the unit box in 1, 2 or 3 dimensions (uniform, or
    graded through per-axis `nodes` and weighted by a per-element `density`).

    DOFs are numbered by the Morton index of their owning element (grid point
    i on an axis with n elements belongs to element min(i//p, n-1)); elements
    are listed in Morton order, which is exactly what the reference's
    `sort_fronts` (tree.py:44-48) produces from their minimum indices, so the
    pairwise elimination tree is geometric nested dissection.  In 1D this is
    the reference numbering of fem.py:59-80.  Element-local DOF order is
    x-fastest and element matrices are kron(Mz, kron(My, Mx)).
    """

    shape: tuple[int, ...]
    degree: int
    # Optional non-uniform data: per-axis element
    # boundaries (n_a + 1 increasing values from 0 to 1: a graded mesh) and a
    # per-element density (Morton element order) scaling each element matrix.
    nodes: Optional[tuple] = None
    density: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        if not 1 <= len(self.shape) <= 3 or any(n < 1 for n in self.shape):
            raise InvalidGeometryError(f"invalid mesh shape {self.shape}")
        _check_degree(self.degree)
        if self.nodes is not None:
            nodes = tuple(np.asarray(x, dtype=np.float64) for x in self.nodes)
            if len(nodes) != len(self.shape) or any(
                    len(x) != n + 1 or x[0] != 0.0 or x[-1] != 1.0 or np.any(np.diff(x) <= 0)
                    for x, n in zip(nodes, self.shape)):
                raise InvalidGeometryError("nodes: per axis n+1 increasing values from 0 to 1")
            object.__setattr__(self, "nodes", nodes)
        if self.density is not None:
            rho = np.asarray(self.density, dtype=np.float64).ravel()
            if len(rho) != self.n_elements or np.any(rho <= 0):
                raise InvalidGeometryError("density: one positive value per element")
            object.__setattr__(self, "density", rho)

    @property
    def uniform(self) -> bool:
        return self.nodes is None and self.density is None

    def _widths(self, a: int) -> np.ndarray:
        n = self.shape[a]
        return np.full(n, 1.0 / n) if self.nodes is None else np.diff(self.nodes[a])

    def _offsets(self, a: int) -> np.ndarray:
        n = self.shape[a]
        return np.arange(n) / n if self.nodes is None else self.nodes[a][:-1]

    @property
    def dim(self) -> int:
        return len(self.shape)

    @property
    def n_elements(self) -> int:
        return int(np.prod(self.shape))

    @property
    def n_dof(self) -> int:
        return int(np.prod([n * self.degree + 1 for n in self.shape]))

    @property
    def nloc(self) -> int:
        return (self.degree + 1) ** self.dim

    def element_table(self) -> np.ndarray:
        """(n_elements, (p+1)^d) int32 DOF table in Morton element order (native)."""
        from . import _lib
        import ctypes as C

        lib = _lib.load()
        ns = np.array(self.shape, dtype=np.int64)
        n_dof = C.c_int64()
        n_el = C.c_int64()
        out = np.empty((self.n_elements, self.nloc), dtype=np.int32)
        rc = lib.tf_mesh_tensor(self.dim, _lib.i64p(ns), self.degree, C.byref(n_dof),
                                C.byref(n_el), _lib.i32p(out))
        _lib.check(rc, "tf_mesh_tensor")
        return out

    def element_matrix(self) -> np.ndarray:
        """The uniform element matrix (or, for a non-uniform mesh, the stack of
        per-element matrices in Morton order: `element_values`)."""
        if not self.uniform:
            return self.element_values()
        mats = [element_mass_matrix(1.0 / n, self.degree) for n in self.shape]
        out = mats[0]
        for m in mats[1:]:
            out = np.kron(m, out)
        return out

    def element_values(self) -> np.ndarray:
        """Per-element matrices (n_elements, nloc, nloc): kron of the 1D mass
        matrices of each element's widths (fem.py:108-114 per axis), times its
        density.  M_e(h) = h M_e(1), so each is a scaled reference matrix."""
        ref = [element_mass_matrix(1.0, self.degree) for _ in self.shape]
        out = ref[0]
        for m in ref[1:]:
            out = np.kron(m, out)
        coords = self.element_coords()
        scale = np.ones(len(coords))
        for a in range(self.dim):
            scale *= self._widths(a)[coords[:, a]]
        if self.density is not None:
            scale *= self.density
        return scale[:, None, None] * out[None, :, :]

    def element_coords(self) -> np.ndarray:
        """(n_elements, d) integer element coordinates in Morton order."""
        d = self.dim
        grids = np.meshgrid(*[np.arange(n) for n in self.shape], indexing="ij")
        coords = np.stack([g.ravel(order="F") for g in grids], axis=1)  # x fastest
        key = np.zeros(len(coords), dtype=np.uint64)
        for b in range(21):
            for a in range(d):
                key |= ((coords[:, a].astype(np.uint64) >> np.uint64(b)) & np.uint64(1)) << \
                    np.uint64(d * b + a)
        return coords[np.argsort(key, kind="stable")]

    def load_vector(self, rhs_name: str = "one") -> np.ndarray:
        """Assembled load vector b_i = (f, phi_i) for a separable f = prod f1(x_a)."""
        f1 = RHS_FUNCTIONS[rhs_name]
        p = self.degree
        per_axis = []
        for a, n in enumerate(self.shape):
            hs, xs = self._widths(a), self._offsets(a)
            per_axis.append(np.array([element_load_vector(hs[e], p, f1, xs[e]) for e in range(n)]))
        coords = self.element_coords()
        loads = per_axis[0][coords[:, 0]]
        for a in range(1, self.dim):
            la = per_axis[a][coords[:, a]]
            loads = (la[:, :, None] * loads[:, None, :]).reshape(len(coords), -1)
        table = self.element_table()
        return np.bincount(table.ravel() - 1, weights=loads.ravel(), minlength=self.n_dof)


# ---------------------------------------------------------------------------
# fronts


@dataclass(frozen=True, eq=False)
class Front:
    """Dense (elemental or merged) submatrix plus its global index map (fem.py:177-215)."""

    front_id: int
    indices: tuple[int, ...]
    membership: tuple[int, ...]
    computed: tuple[bool, ...]
    values: Optional[np.ndarray] = None

    def __post_init__(self) -> None:
        if len(set(self.indices)) != len(self.indices):
            raise ValueError(f"front {self.front_id}: index map is not injective")
        if any(m < 1 for m in self.membership):
            raise ValueError(f"front {self.front_id}: membership counts must be >= 1")
        if not (len(self.indices) == len(self.membership) == len(self.computed)):
            raise ValueError(f"front {self.front_id}: field lengths disagree")
        if self.values is not None and self.values.shape != (self.size, self.size):
            raise ValueError(f"front {self.front_id}: values shape mismatch")

    @property
    def size(self) -> int:
        return len(self.indices)

    @property
    def min_index(self) -> int:
        return min(self.indices)

    @property
    def index_set(self) -> frozenset[int]:
        return frozenset(self.indices)


class FrontSet(Sequence):
    """Array-backed sequence of leaf `Front`s.

    `dofs` is an (n, nloc) int32 table (1-based, element-local order) or a
    CSR pair (ptr, flat); `values` is one shared (nloc, nloc) matrix or an
    (n, nloc, nloc) stack.  Indexing materialises a reference-style `Front`
    (membership computed like generate_fronts, fem.py:241-255).
    """

    def __init__(self, dofs, values, front_ids=None, ptr=None, membership=None):
        self.ptr = None if ptr is None else np.ascontiguousarray(ptr, dtype=np.int64)
        self.dofs = np.ascontiguousarray(dofs, dtype=np.int32)
        self.values = np.ascontiguousarray(values, dtype=np.float64)
        n = len(self.ptr) - 1 if self.ptr is not None else self.dofs.shape[0]
        self.front_ids = (np.arange(n, dtype=np.int64) if front_ids is None
                          else np.ascontiguousarray(front_ids, dtype=np.int64))
        # explicit per-entry membership (from user Fronts), else derived from the set
        self.membership = (None if membership is None
                           else np.ascontiguousarray(membership, dtype=np.int32).reshape(self.dofs.shape))
        self._n = n
        self._counts = None

    def membership_of(self, i: int) -> np.ndarray:
        """Per-index membership of front i.

        generate_fronts (fem.py:241-250) marks an index with the number of
        leaf fronts that hold it (2 at shared 1D endpoints, 1 elsewhere); the
        same count is used for 2D/3D element sets.  Fronts built by the caller
        keep the membership they were given.
        """
        if self.membership is not None:
            return self.membership[i] if self.ptr is None else \
                self.membership[self.ptr[i]:self.ptr[i + 1]]
        if self._counts is None:
            self._counts = np.bincount(self.dofs.ravel().astype(np.int64)).astype(np.int32)
        return self._counts[self.dofs_of(i)]

    @property
    def uniform_values(self) -> bool:
        return self.values.ndim == 2

    @property
    def uniform_size(self) -> bool:
        return self.ptr is None

    def __len__(self) -> int:
        return self._n

    def dofs_of(self, i: int) -> np.ndarray:
        if self.ptr is None:
            return self.dofs[i]
        return self.dofs[self.ptr[i]:self.ptr[i + 1]]

    def values_of(self, i: int) -> np.ndarray:
        return self.values if self.uniform_values else self.values[i]

    def min_indices(self) -> np.ndarray:
        if self.ptr is None:
            return self.dofs.min(axis=1)
        return np.minimum.reduceat(self.dofs, self.ptr[:-1])

    def __getitem__(self, i):
        if isinstance(i, slice):
            return [self[j] for j in range(*i.indices(len(self)))]
        if i < 0:
            i += len(self)
        if not 0 <= i < len(self):
            raise IndexError(i)
        idx = tuple(int(g) for g in self.dofs_of(i))
        n = len(idx)
        vals = self.values_of(i)
        if getattr(self, "padded_values", False):
            vals = vals[:n, :n]
        return Front(front_id=int(self.front_ids[i]), indices=idx,
                     membership=tuple(int(c) for c in self.membership_of(i)),
                     computed=(False,) * n, values=np.array(vals, copy=True))

    def take(self, order: np.ndarray) -> "FrontSet":
        order = np.asarray(order, dtype=np.int64)
        vals = self.values if self.uniform_values else self.values[order]
        if self.ptr is None:
            mem = None if self.membership is None else self.membership[order]
            out = FrontSet(self.dofs[order], vals, self.front_ids[order], membership=mem)
            out._counts = self._counts
            return out
        sizes = np.diff(self.ptr)[order]
        ptr = np.concatenate([[0], np.cumsum(sizes)])
        flat = np.concatenate([self.dofs_of(int(i)) for i in order]) if len(order) else \
            np.zeros(0, np.int32)
        mem = None
        if self.membership is not None:
            mem = np.concatenate([self.membership_of(int(i)) for i in order]) if len(order) else \
                np.zeros(0, np.int32)
        out = FrontSet(flat, vals, self.front_ids[order], ptr=ptr, membership=mem)
        out.padded_values = getattr(self, "padded_values", False)
        return out

    @classmethod
    def from_fronts(cls, fronts: Sequence[Front]) -> "FrontSet":
        if isinstance(fronts, FrontSet):
            return fronts
        sizes = [f.size for f in fronts]
        ids = [f.front_id for f in fronts]
        if any(f.values is None for f in fronts):
            raise ValueError("leaf fronts must carry element values")
        if len(set(sizes)) == 1:
            dofs = np.array([f.indices for f in fronts], dtype=np.int32)
            v0 = fronts[0].values
            same = all(np.array_equal(f.values, v0) for f in fronts)
            vals = v0 if same else np.stack([f.values for f in fronts])
            mem = np.array([f.membership for f in fronts], dtype=np.int32)
            return cls(dofs, vals, ids, membership=mem)
        ptr = np.concatenate([[0], np.cumsum(sizes)])
        flat = np.array([g for f in fronts for g in f.indices], dtype=np.int32)
        raise_if = max(sizes)
        vals = np.zeros((len(fronts), raise_if, raise_if))
        for i, f in enumerate(fronts):
            vals[i, :f.size, :f.size] = f.values
        mem = np.array([c for f in fronts for c in f.membership], dtype=np.int32)
        fs = cls(flat, vals, ids, ptr=ptr, membership=mem)
        fs.padded_values = True
        return fs


def generate_fronts(mesh) -> FrontSet:
    """One leaf front per element, values = element mass matrix (fem.py:235-259)."""
    return FrontSet(mesh.element_table(), mesh.element_matrix())


# ---------------------------------------------------------------------------
# global systems


@dataclass
class GlobalSystem:
    """Assembled sparse system with lower-triangle dict storage (fem.py:133-174)."""

    n_dof: int
    entries: dict[tuple[int, int], float] = field(default_factory=dict)
    rhs: np.ndarray = field(default_factory=lambda: np.zeros(0))

    def add(self, i: int, j: int, value: float) -> None:
        key = (i, j) if i >= j else (j, i)
        self.entries[key] = self.entries.get(key, 0.0) + value

    def entry(self, i: int, j: int) -> float:
        key = (i, j) if i >= j else (j, i)
        return self.entries.get(key, 0.0)

    def symmetric_items(self):
        for (i, j), v in self.entries.items():
            yield (i, j), v
            if i != j:
                yield (j, i), v

    def total_entry_sum(self) -> float:
        return sum(v if i == j else 2.0 * v for (i, j), v in self.entries.items())

    @property
    def peak(self) -> float:
        """max |A_ij| (the zero-pivot scale of engine.py:74)."""
        return max((abs(v) for v in self.entries.values()), default=0.0)

    def to_dense(self) -> np.ndarray:
        m = np.zeros((self.n_dof, self.n_dof))
        for (i, j), v in self.symmetric_items():
            m[i - 1, j - 1] = v
        return m

    def matvec(self, u: np.ndarray) -> np.ndarray:
        u = np.asarray(u, dtype=float)
        out = np.zeros((self.n_dof,) + u.shape[1:])
        for (i, j), v in self.symmetric_items():
            out[i - 1] += v * u[j - 1]
        return out


class ElementSystem(GlobalSystem):
    """Global system defined by element matrices over a FrontSet (lazy entries).

    `entries` (the reference's lower-triangle dict) is assembled only on first
    access, in leaf order; `matvec` is element-by-element and vectorised;
    `peak` equals max|A_ij| of the assembled matrix.
    """

    def __init__(self, n_dof: int, fronts: FrontSet, rhs: np.ndarray, peak: Optional[float] = None):
        self.n_dof = n_dof
        self.rhs = rhs
        self.fronts = fronts
        self._entries = None
        self._peak = peak

    @property
    def entries(self):  # type: ignore[override]
        if self._entries is None:
            ent: dict[tuple[int, int], float] = {}
            for i in range(len(self.fronts)):
                dofs = self.fronts.dofs_of(i)
                vals = self.fronts.values_of(i)
                for a, ga in enumerate(dofs):
                    for b, gb in enumerate(dofs):
                        if ga >= gb:
                            key = (int(ga), int(gb))
                            ent[key] = ent.get(key, 0.0) + float(vals[a, b])
            self._entries = ent
        return self._entries

    @entries.setter
    def entries(self, value):
        self._entries = value
        self.modified = True

    modified = False  # True once entries were edited: they no longer equal the element sum

    def add(self, i: int, j: int, value: float) -> None:
        super().add(i, j, value)
        self.modified = True
        self._peak = None

    @property
    def peak(self) -> float:
        if self._peak is None:
            self._peak = max((abs(v) for v in self.entries.values()), default=0.0)
        return self._peak

    def matvec(self, u: np.ndarray) -> np.ndarray:
        u = np.asarray(u, dtype=float)
        fs = self.fronts
        if not fs.uniform_size or self.modified:
            return super().matvec(u)
        idx = fs.dofs.astype(np.int64) - 1  # (n_el, nloc)
        ue = u[idx]  # (n_el, nloc, ...)
        if fs.uniform_values:
            ye = np.einsum("ab,eb...->ea...", fs.values, ue)
        else:
            ye = np.einsum("eab,eb...->ea...", fs.values, ue)
        out = np.zeros((self.n_dof,) + u.shape[1:])
        if u.ndim == 1:
            return np.bincount(idx.ravel(), weights=ye.ravel(), minlength=self.n_dof)
        for j in range(u.shape[1]):
            out[:, j] = np.bincount(idx.ravel(), weights=ye[:, :, j].ravel(), minlength=self.n_dof)
        return out


def _tensor_peak(mesh: TensorMesh) -> float:
    """max|A_ij| of a uniform tensor mesh from a min(n,3)^d patch (same entry classes)."""
    patch = TensorMesh(tuple(min(n, 3) for n in mesh.shape), mesh.degree)
    emat = mesh.element_matrix()  # widths of the full mesh
    fs = FrontSet(patch.element_table(), emat)
    return ElementSystem(patch.n_dof, fs, np.zeros(patch.n_dof)).peak


def _element_peak(fs: FrontSet, n_dof: int) -> float:
    """max|A_ij| of the element assembly, vectorised (non-uniform element values)."""
    d = fs.dofs.astype(np.int64)
    nloc = d.shape[1]
    vals = np.broadcast_to(fs.values, (len(d), nloc, nloc)) if fs.uniform_values else fs.values
    ia = np.repeat(d, nloc, axis=1).ravel()
    ib = np.tile(d, (1, nloc)).ravel()
    keep = ia >= ib
    key = ia[keep] * (n_dof + 1) + ib[keep]
    uniq, inv = np.unique(key, return_inverse=True)
    sums = np.bincount(inv, weights=vals.reshape(len(d), -1).ravel()[keep], minlength=len(uniq))
    return float(np.abs(sums).max()) if len(sums) else 0.0


def assemble_system(mesh, f: Callable[[float], float] | str = "one") -> GlobalSystem:
    """Global system M u = b (fem.py:218-232).

    1D `Mesh`: the reference's dict assembly, element by element.
    `TensorMesh`: an `ElementSystem` (lazy entries, exact peak, load vector
    of the separable f = prod f1(x_a)).
    """
    if isinstance(mesh, TensorMesh):
        name = f if isinstance(f, str) else next(k for k, v in RHS_FUNCTIONS.items() if v is f)
        fs = generate_fronts(mesh)
        peak = _tensor_peak(mesh) if mesh.uniform else _element_peak(fs, mesh.n_dof)
        return ElementSystem(mesh.n_dof, fs, mesh.load_vector(name), peak=peak)
    func = RHS_FUNCTIONS[f] if isinstance(f, str) else f
    system = GlobalSystem(n_dof=mesh.n_dof, rhs=np.zeros(mesh.n_dof))
    h = mesh.element_width
    local = element_mass_matrix(h, mesh.degree)
    p = mesh.degree
    for e in range(mesh.n_elements):
        dofs = mesh.element_dofs(e)
        for a in range(p + 1):
            for b in range(a + 1):  # ga >= gb  <=>  a >= b on a 1D element
                system.add(dofs[a], dofs[b], local[a, b])
        load = element_load_vector(h, p, func, mesh.element_offset(e))
        system.rhs[e * p: e * p + p + 1] += load
    return system
