"""Numeric execution: factorize on the GPU, LDU-form factors, solve (engine.py:1-493).

Entry points keep the reference's names and meaning:
  init_state(system, plan)                 engine.py:67-75  (zero-pivot threshold)
  run_sequential(plan, state)              engine.py:177-184
  run_concurrent(schedule, plan, state, workers, debug, compiled)
                                           engine.py:354-419
  compile_execution(plan, schedule, state) engine.py:335-344
  solve(factors, rhs)                      engine.py:468-493
Every path runs the hand-written sm_100a kernels of libtfb200.so, one launch
sequence per Foata class (tree level); there is no CPU execution path.  The
factorization is the reference's no-pivoting elimination in its pivot order,
computed as LDL^T on dense fronts (the mass matrix is symmetric, so the
reference's division quotient u(z,y) equals its multiplier l(y,z) up to
rounding; both dictionaries are served from the one stored factor).
"""

from __future__ import annotations

from dataclasses import dataclass, field
from functools import cached_property
from typing import Optional

import numpy as np
import torch

from . import _lib
from .device import DevicePlan, require_cuda
from .errors import ZeroPivotError

ZERO_PIVOT_RELATIVE = 1e-14  # engine.py:35
FUSE_BOTTOM = True  # run the lowest tree levels as one subtree launch when they fit


@dataclass
class ExecState:
    """Execution state: zero-pivot threshold and the compiled device plan."""

    zero_threshold: float = 0.0
    debug: bool = False
    compiled: Optional[DevicePlan] = None
    factors: Optional["FactorResult"] = None
    system: object = None


def init_state(system, plan, debug: bool = False) -> ExecState:
    """Zero-pivot threshold = 1e-14 * max|A_ij| (engine.py:67-75); the system seeds the values."""
    return ExecState(zero_threshold=ZERO_PIVOT_RELATIVE * float(system.peak), debug=debug,
                     system=system)


def leaf_values(fronts, system) -> np.ndarray:
    """Numeric leaf-front values that make the factorization start from `system`.

    The reference seeds its state with the assembled entries
    (init_state, engine.py:67-75).  An `ElementSystem` over the plan's own
    leaf fronts IS the sum of their element matrices, so those are uploaded
    as they are.  Any other `GlobalSystem` (a dict of lower-triangle entries,
    e.g. the reference's 1D assembly or one edited with `add`) is split over
    the leaves: each stored entry goes, whole, to the first leaf front that
    holds both of its indices, so the extend-add sums reproduce every entry
    exactly.  An entry no leaf front covers, or an ElementSystem over other
    fronts, raises ContractViolationError instead of factorizing a different
    matrix.
    """
    from .errors import ContractViolationError
    from .fem import ElementSystem
    from .tree import sort_fronts
    if system is None:
        return fronts.values
    if isinstance(system, ElementSystem) and not system.modified:
        fs = system.fronts
        if fs is not fronts:
            fs = sort_fronts(fs)
        if fs is fronts or (fs.dofs.shape == fronts.dofs.shape and
                            np.array_equal(fs.dofs, fronts.dofs) and
                            fs.values.shape == fronts.values.shape and
                            np.array_equal(fs.values, fronts.values)):
            return fronts.values
        raise ContractViolationError("the system's element matrices are not the plan's leaf fronts")
    entries = system.entries
    n = len(fronts)
    width = fronts.values.shape[-1]
    vals = np.zeros((n, width, width))
    assigned = set()
    for e in range(n):
        d = [int(g) for g in fronts.dofs_of(e)]
        for a, ga in enumerate(d):
            for b, gb in enumerate(d):
                if ga >= gb and (ga, gb) not in assigned:
                    v = entries.get((ga, gb))
                    if v is None:
                        continue
                    vals[e, a, b] = v
                    vals[e, b, a] = v
                    assigned.add((ga, gb))
    if len(assigned) != len(entries):
        missing = next(k for k in entries if k not in assigned)
        raise ContractViolationError(f"system entry {missing} lies outside every leaf front")
    return vals


def compile_execution(plan, schedule=None, state: Optional[ExecState] = None) -> DevicePlan:
    """Upload the level tables and leaf values once; reusable across factorizations
    (engine.py:335-344).  The leaf values come from the state's system (leaf_values)."""
    plan = _plan_of(plan)
    system = state.system if state is not None and state.system is not None else plan.system
    dp = DevicePlan(plan, plan.tree.fronts, values=leaf_values(plan.tree.fronts, system))
    dp.fuse_bottom = FUSE_BOTTOM
    if state is not None:
        state.compiled = dp
    return dp


class FactorResult:
    """LDU-form factors in global coordinates (engine.py:110-144).

    Device-resident: `device_plan.factors[L]` holds every front's m x k panel.
    `u_entries` / `l_entries` are materialised on first access with the
    reference's key sets (small plans only).
    """

    def __init__(self, plan, device_plan: DevicePlan):
        self.plan = plan
        self.device_plan = device_plan
        self.n_dof = plan.n_dof

    @property
    def pivot_order(self) -> tuple[int, ...]:
        return self.plan.pivot_order

    def permutation(self) -> np.ndarray:
        return self.plan.pivot_order_array.astype(np.int64) - 1

    @cached_property
    def _dicts(self):
        plan = self.plan
        steps = plan.steps
        u: dict[tuple[int, int], float] = {}
        l: dict[tuple[int, int], float] = {}
        s = 0
        for L, dl in enumerate(self.device_plan.levels):
            lt = dl.tables
            ptr, kk, idx = plan.native.node_lists(L)
            fac = self.device_plan.factors[L].cpu().numpy()
            for i in range(lt.n_fronts):
                row = lt.pat[lt.pattern_of[i]]
                m, k, kp = int(row[_lib.PAT_M]), int(row[_lib.PAT_K]), int(row[_lib.PAT_KP])
                if k == 0:
                    continue
                P = fac[i * dl.fac_stride: i * dl.fac_stride + m * kp].reshape(m, kp)
                lst = idx[ptr[i]:ptr[i + 1]]
                pos = {int(g): r for r, g in enumerate(lst)}
                for c in range(k):
                    z = int(lst[c])
                    st = steps[s]
                    s += 1
                    assert st.pivot == z
                    for y in st.active:
                        v = float(P[pos[y], c])
                        u[(z, y)] = v
                        l[(y, z)] = v
                    u[(z, z)] = float(P[c, c])
        return u, l

    def _lookup(self, piv: np.ndarray, row: np.ndarray) -> np.ndarray:
        """Stored factor entry (row `row`, pivot column `piv`), global 1-based indices.

        Vectorised over key arrays; needs a plan built with node lists.  The
        entry is l(row, piv) = u(piv, row) (LDL^T), or the pivot d when row == piv.
        """
        plan, dp = self.plan, self.device_plan
        native = plan.native
        piv = np.asarray(piv, dtype=np.int64).ravel()
        row = np.asarray(row, dtype=np.int64).ravel()
        inv = np.full(self.n_dof + 1, -1, dtype=np.int64)
        inv[native.pivot_order.astype(np.int64)] = np.arange(native.n_pivots, dtype=np.int64)
        pos = inv[piv]
        if np.any(pos < 0):
            raise KeyError("key column is not a pivot")
        bases = np.array([lt.piv_base for lt in native.levels], dtype=np.int64)
        lev = np.searchsorted(bases, pos, side="right") - 1
        out = np.empty(len(piv), dtype=np.float64)
        for L in np.unique(lev):
            sel = np.nonzero(lev == L)[0]
            lt, dl = native.levels[int(L)], dp.levels[int(L)]
            ptr, _, idx = native.node_lists(int(L))
            f = np.searchsorted(lt.piv_off, pos[sel], side="right") - 1
            col = pos[sel] - lt.piv_off[f]
            kp = lt.pat[lt.pattern_of[f], _lib.PAT_KP].astype(np.int64)
            r = np.empty(len(sel), dtype=np.int64)
            for t, (ff, g) in enumerate(zip(f, row[sel])):
                hit = np.nonzero(idx[ptr[ff]:ptr[ff + 1]] == g)[0]
                if len(hit) != 1:
                    raise KeyError((int(g), int(piv[sel[t]])))
                r[t] = hit[0]
            if np.any(r < col):
                raise KeyError("key is above the diagonal of its front")
            flat = torch.from_numpy(f * dl.fac_stride + r * kp + col).to(dp.device)
            out[sel] = dp.factors[int(L)][flat].cpu().numpy()
        return out

    def u_values(self, keys) -> np.ndarray:
        """u(z, y) for an (n, 2) array of keys, without building the dictionaries."""
        k = np.asarray(keys, dtype=np.int64).reshape(-1, 2)
        return self._lookup(k[:, 0], k[:, 1])

    def l_values(self, keys) -> np.ndarray:
        """l(x, z) for an (n, 2) array of keys, without building the dictionaries."""
        k = np.asarray(keys, dtype=np.int64).reshape(-1, 2)
        return self._lookup(k[:, 1], k[:, 0])

    def pivot_values(self, positions) -> np.ndarray:
        """d at the given pivot-order positions."""
        po = self.plan.native.pivot_order.astype(np.int64)[np.asarray(positions, dtype=np.int64)]
        return self._lookup(po, po)

    @property
    def u_entries(self) -> dict[tuple[int, int], float]:
        return self._dicts[0]

    @property
    def l_entries(self) -> dict[tuple[int, int], float]:
        return self._dicts[1]

    def permuted_dense_factors(self) -> tuple[np.ndarray, np.ndarray]:
        """Unit-lower L and standard U with L @ U == P M P^T (engine.py:126-140)."""
        pos = {z: k for k, z in enumerate(self.pivot_order)}
        n = self.n_dof
        lower = np.eye(n)
        upper = np.zeros((n, n))
        u = self.u_entries
        for (x, z), v in self.l_entries.items():
            lower[pos[x], pos[z]] = v
        for (z, y), v in u.items():
            upper[pos[z], pos[y]] = v if z == y else v * u[(z, z)]
        return lower, upper

    def solve(self, rhs):
        return solve(self, rhs)


def _factorize(plan, state: ExecState, compiled: Optional[DevicePlan] = None) -> FactorResult:
    dp = compiled or state.compiled or compile_execution(plan, None, state)
    dp.factor_graphed(state.zero_threshold)
    pos = dp.zero_pivot_position()
    if pos >= 0:
        front, pivot = plan.locate_pivot(pos)
        raise ZeroPivotError(front, pivot)
    res = FactorResult(plan, dp)
    state.factors = res
    return res


def _plan_of(x):
    """EliminationPlan of a plan or of a DependencyGraph (graph.plan, tasks.py:185-204)."""
    return getattr(x, "plan", x) if not hasattr(x, "native") else x


def run_sequential(plan, state: ExecState) -> FactorResult:
    """Execute the level classes in order on the current CUDA stream (engine.py:177-184).

    Accepts the reference's DependencyGraph (cli.py:157) or an EliminationPlan."""
    return _factorize(_plan_of(plan), state)


def run_concurrent(schedule, plan, state: ExecState, workers: int = 1, debug: bool = False,
                   compiled: Optional[DevicePlan] = None) -> FactorResult:
    """Execute classes in order with a barrier between classes (engine.py:354-419).

    Within a class the GPU runs every front concurrently and the stream order
    between level launches is the class barrier.  The reference's `workers`
    are CPU processes sharing one matrix; here the unit of concurrency is a
    GPU.  workers == 1 runs on the current device.  workers > 1 requires an
    initialised torch.distributed group of exactly `workers` ranks (one per
    GPU; NCCL on a GPU box): the tree is sharded by subtrees
    (distributed.ShardedFactorization) and every rank
    returns the same FactorResult (factors gathered, bitwise equal to the
    one-GPU run).  Without such a group, workers > 1 raises ValueError rather
    than silently running on one GPU.
    """
    if workers < 1:
        raise ValueError(f"workers must be >= 1, got {workers}")
    plan = _plan_of(plan)
    if debug:
        from .verify import check_level_schedule
        check_level_schedule(plan, schedule)
    if workers == 1:
        return _factorize(plan, state, compiled)
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() != workers:
        raise ValueError(f"workers={workers} needs an initialised torch.distributed group of "
                         f"{workers} ranks (one per GPU)")
    from .distributed import HostStagedComm, ShardedFactorization, TorchComm
    dp = compiled or state.compiled or compile_execution(plan, None, state)
    # NCCL moves device buffers directly; a CPU backend (gloo) stages them through the host
    comm = HostStagedComm() if dist.get_backend() == "gloo" else TorchComm()
    sf = ShardedFactorization(dp, workers, comm, ranks=[dist.get_rank()])
    pos = sf.factor(state.zero_threshold)
    if pos >= 0:
        front, pivot = plan.locate_pivot(pos)
        raise ZeroPivotError(front, pivot)
    sf.gather_all()
    res = FactorResult(plan, dp)
    state.factors = res
    return res


def factor_and_solve(plan, state: ExecState, rhs, compiled: Optional[DevicePlan] = None):
    """run_sequential(plan, state) + solve(factors, rhs) in one call, with the
    forward sweep of each level overlapped with the factorization of the levels
    above it (DevicePlan.factor_solve; same results).  Returns (factors, x);
    x has rhs's kind and shape.  Raises ZeroPivotError like run_sequential."""
    plan = _plan_of(plan)
    dp = compiled or state.compiled or compile_execution(plan, None, state)
    n = plan.n_dof
    if not isinstance(rhs, torch.Tensor):
        arr = np.asarray(rhs, dtype=float)
        if arr.shape[:1] != (n,) or arr.ndim > 2:
            raise ValueError(f"rhs must have length {n}, got {arr.shape}")
    b = _as_device(rhs, dp.device, n)
    x = torch.empty_like(b)
    dp.factor_solve_graphed(state.zero_threshold, b, x)
    pos = dp.zero_pivot_position()
    if pos >= 0:
        front, pivot = plan.locate_pivot(pos)
        raise ZeroPivotError(front, pivot)
    res = FactorResult(plan, dp)
    state.factors = res
    return res, (x if isinstance(rhs, torch.Tensor) else x.cpu().numpy())


def factorize(plan, system) -> FactorResult:
    """Convenience: init_state + run_sequential."""
    return run_sequential(plan, init_state(system, plan))


def _as_device(rhs, device, n):
    if isinstance(rhs, torch.Tensor):
        t = rhs.to(device=device, dtype=torch.float64)
    else:
        t = torch.from_numpy(np.ascontiguousarray(rhs, dtype=np.float64)).to(device)
    if t.shape[0] != n or t.dim() > 2:
        raise ValueError(f"rhs must have length {n}, got {tuple(t.shape)}")
    return t.contiguous()


def solve(factors: FactorResult, rhs):
    """Forward (unit L), diagonal scaling, backward (U) substitution (engine.py:468-493).

    rhs: (n,) or (n, nrhs), numpy or torch.  Returns the same kind/shape
    (numpy in, numpy out; a CUDA tensor in, a CUDA tensor out).
    """
    dp = factors.device_plan
    n = factors.n_dof
    if not isinstance(rhs, torch.Tensor):
        arr = np.asarray(rhs, dtype=float)
        if arr.shape[:1] != (n,) or arr.ndim > 2:
            raise ValueError(f"rhs must have length {n}, got {arr.shape}")
    b = _as_device(rhs, dp.device, n)
    x = torch.empty_like(b)
    dp.solve_graphed(b, x)
    if isinstance(rhs, torch.Tensor):
        return x
    return x.cpu().numpy()
