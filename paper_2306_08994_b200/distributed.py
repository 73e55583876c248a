"""Subtree sharding of the factorization and solve across GPUs.

The elimination tree is cut at the split level L_s, the highest level with at
least `world` nodes.  Node i of L_s (and its whole subtree) belongs to rank
floor(i * world / n_{L_s}); a node above the split belongs to the owner of its
leftmost descendant at L_s.  Every rank's fronts form one contiguous range per
level, so each rank runs the same per-level kernels (`tf_level_factor`,
`tf_level_solve_*`) on a slice view of the level tables -- no kernel knows it
is distributed, and each front is computed by the same kernel variant as on
one GPU (the slice keeps the full level's maxima), so the factors are
bitwise identical for any rank count.

Data crosses ranks only where the tree does:
  factor / forward solve: a child's update block goes to its parent's owner;
  backward solve: a parent's solution block goes to the child's owner;
  end of solve: every rank's own solution rows are all-gathered.
These are point-to-point transfers issued per level through a `Comm`:
`TorchComm` (torch.distributed P2P, NCCL over NVLink on a GPU box; gloo on
CPU) or `LocalComm` (all ranks simulated in one process on one device: the
same slices and transfers, executed rank by rank, which the tests use to pin
the sharded path against the single-GPU one).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib


# --------------------------------------------------------------- ownership
@dataclass
class LevelShard:
    level: int
    owner: np.ndarray          # [n_fronts] rank of every front
    ranges: list               # rank -> (f0, f1) owned fronts (f0 == f1: none)
    slots: list                # rank -> (lo, hi) update/solve-block slots held


class ShardPlan:
    """Front ownership and transfer lists for `world` ranks."""

    def __init__(self, level_sizes, world: int):
        if world < 1:
            raise ValueError("world must be >= 1")
        self.world = world
        sizes = list(level_sizes)
        self.n_levels = len(sizes)
        cand = [L for L, n in enumerate(sizes) if n >= world]
        self.split = max(cand) if cand else 0
        Ls = self.split
        ns = sizes[Ls]
        base_owner = (np.arange(ns, dtype=np.int64) * world) // max(ns, 1)
        base_owner = np.minimum(base_owner, world - 1)
        self.levels: list[LevelShard] = []
        for L, n in enumerate(sizes):
            i = np.arange(n, dtype=np.int64)
            if L <= Ls:
                anc = i >> (Ls - L)
            else:
                anc = np.minimum(i << (L - Ls), ns - 1)
            owner = base_owner[anc]
            ranges = []
            for r in range(world):
                idx = np.nonzero(owner == r)[0]
                if len(idx):
                    assert idx[-1] - idx[0] + 1 == len(idx), "ownership not contiguous"
                    ranges.append((int(idx[0]), int(idx[-1]) + 1))
                else:
                    ranges.append((0, 0))
            self.levels.append(LevelShard(L, owner, ranges, [None] * world))
        # slots: own fronts plus the children of owned parents (received updates)
        for L, ls in enumerate(self.levels):
            for r in range(world):
                lo, hi = ls.ranges[r]
                if L + 1 < self.n_levels:
                    p0, p1 = self.levels[L + 1].ranges[r]
                    if p1 > p0:
                        c0, c1 = 2 * p0, min(2 * p1, len(ls.owner))
                        lo, hi = (c0, c1) if lo == hi else (min(lo, c0), max(hi, c1))
                ls.slots[r] = (lo, hi)

    def upward(self, L: int):
        """Transfers before level L (L >= 1): (child front, src rank, dst rank)."""
        out = []
        child, parent = self.levels[L - 1], self.levels[L]
        for c in range(len(child.owner)):
            q, p = int(child.owner[c]), int(parent.owner[c >> 1])
            if q != p:
                out.append((c, q, p))
        return out

    def downward(self, L: int):
        """Transfers before backward level L (L < top): (parent front, src, dst)."""
        out = []
        child, parent = self.levels[L], self.levels[L + 1]
        seen = set()
        for c in range(len(child.owner)):
            q, p = int(child.owner[c]), int(parent.owner[c >> 1])
            if q != p and ((c >> 1), q) not in seen:
                seen.add(((c >> 1), q))
                out.append((c >> 1, p, q))
        return out


# ------------------------------------------------------------------- comms
class LocalComm:
    """All ranks in one process: a transfer is a device-to-device copy."""

    def exchange(self, moves):
        """moves: list of (src_tensor_view, dst_tensor_view)."""
        for src, dst in moves:
            dst.copy_(src)

    def allreduce_sum(self, tensors):
        tot = tensors[0].clone()
        for t in tensors[1:]:
            tot += t
        for t in tensors:
            t.copy_(tot)

    def allreduce_min(self, tensors):
        m = tensors[0].clone()
        for t in tensors[1:]:
            m = torch_min(m, t)
        for t in tensors:
            t.copy_(m)


def torch_min(a, b):
    import torch
    return torch.minimum(a, b)


class TorchComm:
    """One rank of a torch.distributed group (NCCL on GPUs, gloo on CPU)."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.rank = dist.get_rank(group)

    def p2p(self, sends, recvs):
        """sends: [(tensor, dst)], recvs: [(tensor, src)]; one batched group."""
        dist = self.dist
        ops = [dist.P2POp(dist.isend, t, d, group=self.group) for t, d in sends]
        ops += [dist.P2POp(dist.irecv, t, s, group=self.group) for t, s in recvs]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    def allreduce_sum(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)

    def allreduce_min(self, t):
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)

    def broadcast(self, t, src: int):
        self.dist.broadcast(t, src, group=self.group)

    def allgather(self, out_list, t):
        self.dist.all_gather(out_list, t, group=self.group)


class HostStagedComm(TorchComm):
    """TorchComm over a CPU backend (gloo) for device tensors: every transfer
    is staged through host memory.  Lets several processes share ONE GPU in
    tests of the multi-process path (the ranks never wait on each other's
    kernels: all waiting happens in gloo on the host)."""

    def p2p(self, sends, recvs):
        hs = [(t.detach().cpu(), d) for t, d in sends]
        hr = [(torch_empty_like_cpu(t), s) for t, s in recvs]
        super().p2p(hs, hr)
        for (t, _), (h, _) in zip(recvs, hr):
            t.copy_(h)

    def allreduce_sum(self, t):
        h = t.detach().cpu()
        super().allreduce_sum(h)
        t.copy_(h)

    def allreduce_min(self, t):
        h = t.detach().cpu()
        super().allreduce_min(h)
        t.copy_(h)

    def broadcast(self, t, src: int):
        h = t.detach().cpu()
        super().broadcast(h, src)
        t.copy_(h)

    def allgather(self, out_list, t):
        hs = [torch_empty_like_cpu(o) for o in out_list]
        super().allgather(hs, t.detach().cpu())
        for o, h in zip(out_list, hs):
            o.copy_(h)


def torch_empty_like_cpu(t):
    import torch
    return torch.empty(t.shape, dtype=t.dtype, device="cpu")


# ------------------------------------------------------ per-rank GPU state
def _slice_view(full, f0: int, n: int, child_base: int = 0):
    """View of fronts [f0, f0+n) of a level; tree relations stay absolute."""
    v = _lib.LevelView()
    C.memmove(C.byref(v), C.byref(full), C.sizeof(_lib.LevelView))
    v.leaf_direct = 0  # every rank's leaf updates are written (slices read them as usual)
    v.n_fronts = n
    v.pattern_of = (full.pattern_of or 0) + 4 * f0
    v.piv_off = (full.piv_off or 0) + 8 * f0
    v.front_base = f0
    v.child_base = child_base
    if full.zero_upd:
        v.zero_upd = full.zero_upd + f0
    # implicit forward updates read the child's factors, which a rank only
    # holds for its own fronts: the sharded sweeps keep every update explicit
    v.implicit_upd = None
    v.factors = None
    return v


class RankState:
    """Device buffers and slice views of one rank (GPU executor)."""

    def __init__(self, dp, shard: ShardPlan, rank: int):
        import torch
        self.dp, self.shard, self.rank = dp, shard, rank
        dev = dp.device
        self.views, self.fac, self.aux, self.ws = [], [], [], []
        upd_max = 1
        for L, dl in enumerate(dp.levels):
            f0, f1 = shard.levels[L].ranges[rank]
            lo, hi = shard.levels[L].slots[rank]
            n = f1 - f0
            clo = shard.levels[L - 1].slots[rank][0] if L > 0 else 0
            v = _slice_view(dl.view, f0, n, child_base=clo)
            fac = torch.empty(max(1, n * dl.fac_stride), dtype=torch.float64, device=dev)
            aux = None
            if dl.aux_stride > 0:
                aux = torch.empty(max(1, n * dl.aux_stride), dtype=torch.float64, device=dev)
                v.aux = aux.data_ptr()
            wsb = int(dp.lib.tf_level_factor_workspace(C.byref(v))) if n > 0 else 0
            self.ws.append((torch.empty(wsb, dtype=torch.uint8, device=dev) if wsb else None, wsb))
            self.views.append(v)
            self.fac.append(fac)
            self.aux.append(aux)
            upd_max = max(upd_max, (hi - lo) * dl.upd_stride)
        self.upd = [torch.empty(upd_max, dtype=torch.float64, device=dev) for _ in range(2)]
        self.err = torch.full((1,), -1, dtype=torch.int64, device=dev)

    def upd_slot(self, L: int, f: int):
        dl = self.dp.levels[L]
        lo = self.shard.levels[L].slots[self.rank][0]
        buf = self.upd[L & 1]
        return buf[(f - lo) * dl.upd_stride:(f - lo + 1) * dl.upd_stride]

    def factor_level(self, L: int, threshold: float, sp) -> None:
        f0, f1 = self.shard.levels[L].ranges[self.rank]
        if f1 <= f0:
            return
        dp, dl = self.dp, self.dp.levels[L]
        lo = self.shard.levels[L].slots[self.rank][0]
        out = self.upd[L & 1].data_ptr() + 8 * (f0 - lo) * dl.upd_stride
        child = self.upd[(L - 1) & 1].data_ptr() if L > 0 else None
        rc = dp.lib.tf_level_factor(C.byref(self.views[L]),
                                    None if child is None else C.c_void_p(child),
                                    C.c_void_p(dp.elem.data_ptr() + 8 * f0 * dl.view.elem_stride),
                                    C.c_void_p(self.fac[L].data_ptr()), C.c_void_p(out),
                                    C.c_double(threshold), C.c_void_p(self.err.data_ptr()),
                                    None if self.ws[L][0] is None else
                                    C.c_void_p(self.ws[L][0].data_ptr()), self.ws[L][1], sp)
        _lib.check(rc, f"tf_level_factor(rank {self.rank}, level {L})")


class ShardedFactorization:
    """Factor (and solve) with the tree sharded over `world` ranks.

    `ranks` lists the ranks this process executes: all of them with
    LocalComm (one-device simulation), or just its own with TorchComm.
    """

    def __init__(self, dp, world: int, comm, ranks=None):
        self.dp = dp
        self.world = world
        self.comm = comm
        self.shard = ShardPlan([dl.n_fronts for dl in dp.levels], world)
        self.ranks = list(range(world)) if ranks is None else list(ranks)
        self.state = {r: RankState(dp, self.shard, r) for r in self.ranks}

    def _transfer_upward(self, L: int) -> None:
        moves = self.shard.upward(L)
        if isinstance(self.comm, LocalComm):
            self.comm.exchange([(self.state[q].upd_slot(L - 1, c), self.state[p].upd_slot(L - 1, c))
                                for c, q, p in moves])
            return
        me = self.ranks[0]
        sends = [(self.state[me].upd_slot(L - 1, c), p) for c, q, p in moves if q == me]
        recvs = [(self.state[me].upd_slot(L - 1, c), q) for c, q, p in moves if p == me]
        self.comm.p2p(sends, recvs)

    def factor(self, threshold: float, stream=None, level_hook=None) -> int:
        """Numeric factorization; returns the earliest zero-pivot position or -1.

        level_hook(L), if given, is called after level L's launches (event timing)."""
        import torch
        st = stream or torch.cuda.current_stream(self.dp.device)
        sp = C.c_void_p(st.cuda_stream)
        for r in self.ranks:
            self.state[r].err.fill_(-1)
        for L in range(len(self.dp.levels)):
            if L > 0:
                self._transfer_upward(L)
            for r in self.ranks:
                self.state[r].factor_level(L, threshold, sp)
            if level_hook is not None:
                level_hook(L)
        big = np.iinfo(np.int64).max
        if isinstance(self.comm, LocalComm):
            vals = [int(self.state[r].err.item()) for r in self.ranks]
            vals = [v for v in vals if v >= 0]
            return min(vals) if vals else -1
        e = self.state[self.ranks[0]].err.clone()
        e[e < 0] = big
        self.comm.allreduce_min(e)
        v = int(e.item())
        return -1 if v == big else v

    def gather_factors(self):
        """Per-level factor tensors in the single-GPU layout (for comparison)."""
        import torch
        out = []
        for L, dl in enumerate(self.dp.levels):
            full = torch.zeros(max(1, dl.n_fronts * dl.fac_stride), dtype=torch.float64,
                               device=self.dp.device)
            for r in self.ranks:
                f0, f1 = self.shard.levels[L].ranges[r]
                if f1 > f0:
                    full[f0 * dl.fac_stride:f1 * dl.fac_stride] = \
                        self.state[r].fac[L][:(f1 - f0) * dl.fac_stride]
            out.append(full)
        return out

    def gather_all(self) -> None:
        """Give every process the complete factorization in `dp`'s one-GPU layout.

        Each level's owned front ranges (factor panels and, on large levels,
        the diagonal-block inverses the solve reads) are broadcast from their
        owner, so `dp.solve_into` and the factor dictionaries then work on any
        rank without further communication.  Collective over the group.
        """
        dp = self.dp
        me = None if isinstance(self.comm, LocalComm) else self.ranks[0]
        for L, dl in enumerate(dp.levels):
            parts = [(dp.factors[L], dl.fac_stride, "fac")]
            if dl.aux is not None:
                parts.append((dl.aux, dl.aux_stride, "aux"))
            for full, stride, kind in parts:
                for r in range(self.world):
                    f0, f1 = self.shard.levels[L].ranges[r]
                    if f1 <= f0:
                        continue
                    dst = full[f0 * stride:f1 * stride]
                    if r in self.state:
                        src = self.state[r].fac[L] if kind == "fac" else self.state[r].aux[L]
                        dst.copy_(src[:(f1 - f0) * stride])
                    if me is not None:
                        self.comm.broadcast(dst, r)

    # ---------------------------------------------------------------- solve
    def _solve_slots(self, r: int, L: int):
        sh = self.shard
        n = len(sh.levels[L].owner)
        cand = []
        f0, f1 = sh.levels[L].ranges[r]
        if f1 > f0:
            cand.append((f0, f1))
        if L + 1 < sh.n_levels:
            p0, p1 = sh.levels[L + 1].ranges[r]
            if p1 > p0:
                cand.append((2 * p0, min(2 * p1, n)))
        if L > 0:
            c0, c1 = sh.levels[L - 1].ranges[r]
            if c1 > c0:
                cand.append((c0 >> 1, ((c1 - 1) >> 1) + 1))
        if not cand:
            return (0, 0)
        return (min(a for a, _ in cand), max(b for _, b in cand))

    def _prepare_solve(self, nrhs: int) -> None:
        import torch
        if getattr(self, "_nrhs", None) == nrhs:
            return
        dp = self.dp
        self._slots = {r: [self._solve_slots(r, L) for L in range(len(dp.levels))]
                       for r in self.ranks}
        self._own = None
        self._blk, self._y, self._ws = {}, {}, {}
        for r in self.ranks:
            n = max((hi - lo) * dp.levels[L].max_m for L, (lo, hi) in enumerate(self._slots[r]))
            self._blk[r] = [torch.empty(max(1, n * nrhs), dtype=torch.float64, device=dp.device)
                            for _ in range(2)]
            self._y[r] = torch.empty(max(1, dp.n_pivots * nrhs), dtype=torch.float64,
                                     device=dp.device)
            ws = max(int(dp.lib.tf_level_solve_workspace(C.byref(self.state[r].views[L]), nrhs))
                     for L in range(len(dp.levels)))
            self._ws[r] = (torch.empty(max(1, ws // 8), dtype=torch.float64, device=dp.device), ws)
        self._nrhs = nrhs

    def _owned_rows(self):
        """Pivot-order rows each rank owns (one contiguous range per level)."""
        import torch
        if self._own is not None:
            return self._own
        dp = self.dp
        self._own = []
        for r in range(self.world):
            parts = []
            for L, dl in enumerate(dp.levels):
                f0, f1 = self.shard.levels[L].ranges[r]
                if f1 > f0:
                    lt = dl.tables
                    a = int(lt.piv_off[f0])
                    z = int(lt.piv_off[f1]) if f1 < lt.n_fronts else lt.piv_base + lt.n_pivots
                    parts.append(np.arange(a, z, dtype=np.int64))
            idx = np.concatenate(parts) if parts else np.zeros(0, np.int64)
            self._own.append(torch.from_numpy(idx).to(dp.device))
        self._own_max = max(1, max(len(o) for o in self._own))
        return self._own

    def _blk_slot(self, r: int, L: int, f: int, nrhs: int):
        lo = self._slots[r][L][0]
        rows = self.dp.levels[L].max_m * nrhs
        buf = self._blk[r][L & 1]
        return buf[(f - lo) * rows:(f - lo + 1) * rows]

    def _move(self, moves, L: int, nrhs: int) -> None:
        if isinstance(self.comm, LocalComm):
            self.comm.exchange([(self._blk_slot(s, L, f, nrhs), self._blk_slot(d, L, f, nrhs))
                                for f, s, d in moves])
            return
        me = self.ranks[0]
        sends = [(self._blk_slot(me, L, f, nrhs), d) for f, s, d in moves if s == me]
        recvs = [(self._blk_slot(me, L, f, nrhs), s) for f, s, d in moves if d == me]
        self.comm.p2p(sends, recvs)

    def solve_into(self, b, x, stream=None) -> None:
        """x = A^-1 b (row-major (n, nrhs) device tensors, replicated on every rank)."""
        import torch
        dp = self.dp
        nrhs = 1 if b.dim() == 1 else b.shape[1]
        self._prepare_solve(nrhs)
        st = stream or torch.cuda.current_stream(dp.device)
        sp = C.c_void_p(st.cuda_stream)
        lib = dp.lib
        nl = len(dp.levels)
        po = C.c_void_p(dp.pivot_order.data_ptr())
        for r in self.ranks:
            _lib.check(lib.tf_permute_rows(po, dp.n_pivots, C.c_void_p(b.data_ptr()),
                                           C.c_void_p(self._y[r].data_ptr()), nrhs, 0, sp),
                       "tf_permute_rows")

        def sview(r, L):
            lo, hi = self._slots[r][L]
            return _slice_view(dp.levels[L].view, lo, hi - lo)

        for L in range(nl):
            if L > 0:
                self._move([(c, q, p) for c, q, p in self.shard.upward(L)], L - 1, nrhs)
            for r in self.ranks:
                f0, f1 = self.shard.levels[L].ranges[r]
                if f1 <= f0:
                    continue
                st_r = self.state[r]
                lo = self._slots[r][L][0]
                rows = dp.levels[L].max_m * nrhs
                cv = sview(r, L - 1) if L > 0 else None
                rc = lib.tf_level_solve_fwd(
                    C.byref(st_r.views[L]), C.byref(cv) if cv is not None else None,
                    C.c_void_p(st_r.fac[L].data_ptr()),
                    C.c_void_p(self._blk[r][(L - 1) & 1].data_ptr()) if L > 0 else None,
                    dp.levels[L - 1].max_m if L > 0 else 0,
                    C.c_void_p(self._blk[r][L & 1].data_ptr() + 8 * (f0 - lo) * rows),
                    dp.levels[L].max_m, C.c_void_p(self._y[r].data_ptr()), nrhs,
                    C.c_void_p(self._ws[r][0].data_ptr()), self._ws[r][1], sp)
                _lib.check(rc, f"tf_level_solve_fwd(rank {r}, level {L})")
        for L in range(nl - 1, -1, -1):
            if L + 1 < nl:
                self._move(self.shard.downward(L), L + 1, nrhs)
            for r in self.ranks:
                f0, f1 = self.shard.levels[L].ranges[r]
                if f1 <= f0:
                    continue
                st_r = self.state[r]
                lo = self._slots[r][L][0]
                rows = dp.levels[L].max_m * nrhs
                pv = sview(r, L + 1) if L + 1 < nl else None
                ws, wsb = self._ws[r]
                rc = lib.tf_level_solve_bwd(
                    C.byref(st_r.views[L]), C.byref(pv) if pv is not None else None,
                    C.c_void_p(st_r.fac[L].data_ptr()),
                    C.c_void_p(self._blk[r][(L + 1) & 1].data_ptr()) if pv is not None else None,
                    dp.levels[L + 1].max_m if pv is not None else 0,
                    C.c_void_p(self._blk[r][L & 1].data_ptr() + 8 * (f0 - lo) * rows),
                    dp.levels[L].max_m, C.c_void_p(self._y[r].data_ptr()), nrhs,
                    C.c_void_p(ws.data_ptr()), wsb, sp)
                _lib.check(rc, f"tf_level_solve_bwd(rank {r}, level {L})")
        # every rank's own pivot rows -> every rank (all-gather of owned rows,
        # n x nrhs doubles received per rank), then scatter to natural order
        npiv = dp.n_pivots
        self._owned_rows()

        def rows(r):
            return self._y[r][:npiv * nrhs].view(npiv, nrhs)

        if isinstance(self.comm, LocalComm):
            y0 = rows(self.ranks[0])
            for r in self.ranks[1:]:
                y0[self._own[r]] = rows(r)[self._own[r]]
            ys = [self._y[self.ranks[0]]]
        else:
            me = self.ranks[0]
            send = torch.zeros((self._own_max, nrhs), dtype=torch.float64, device=dp.device)
            send[:len(self._own[me])] = rows(me)[self._own[me]]
            outs = [torch.empty_like(send) for _ in range(self.world)]
            self.comm.allgather(outs, send)
            y0 = rows(me)
            for r in range(self.world):
                if r != me:
                    y0[self._own[r]] = outs[r][:len(self._own[r])]
            ys = [self._y[me]]
        if x.data_ptr() != b.data_ptr():
            x.copy_(b)
        _lib.check(lib.tf_permute_rows(po, dp.n_pivots, C.c_void_p(ys[0].data_ptr()),
                                       C.c_void_p(x.data_ptr()), nrhs, 1, sp), "tf_permute_rows")
