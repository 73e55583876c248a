"""GPU executor: per-level device tables, factor buffers, level launch loops.

`DevicePlan` is the compiled, reusable execution plan (the analogue of the
reference's `compile_execution`, engine.py:335-344): it uploads each level's
pattern table and extend-add maps once, owns the factor buffers, and runs
one Foata class (tree level) per `tf_level_factor` call, in stream order
(the stream is the class barrier of engine.py:330-332).

Device memory layout per level L (all float64, row-major):
  factors[L] : n_fronts x fac_stride   front panel P (m x kp, lower part valid)
                                       followed by the pivots d (kp)
  aux[L]     : n_fronts x aux_stride   large-front levels only: unit-lower
                                       inverses of the 64-wide diagonal blocks
  upd ping-pong: n_fronts x upd_stride packed lower Schur complement (m-k)^2
  solve blocks : n_fronts x max_m x nrhs (forward W / backward X, ping-pong)
"""

from __future__ import annotations

import ctypes as C
import os
from typing import Optional

import numpy as np
import torch

from . import _lib


# Bottom-level subtree fusion is implemented and parity-tested but measured
# slower than the per-level kernels on B200 (tools/fuse_sweep.sh), so it is off
# unless a cap is set.
FUSE_CAP_DEFAULT = 0
# ... except on small trees, where every level is a few microseconds of work and
# the per-launch cost dominates (cfg1: 1024 leaves)
FUSE_AUTO_MAX_LEAVES = 0  # measured: cfg1 fused 0.54 ms vs 0.145 ms per level (graph)


def _tri(n):
    return n * (n + 1) // 2


# Guard mode (tests; race/out-of-bounds detection without compute-sanitizer):
# every kernel-written buffer gets GUARD_DOUBLES canary words on both sides,
# and its interior is filled with a NaN before each factorization / solve, so
# a stray write shows up in check_guards() and a read of unwritten data turns
# the result into NaN.  Off by default (TFB_GUARD=1 or device.GUARD = True).
GUARD = os.environ.get("TFB_GUARD", "0") == "1"
# The public API (run_sequential / run_concurrent(1) / solve) replays cached
# CUDA graphs of the whole factorization and solve (TFB_GRAPHS=0: eager).
USE_GRAPHS = os.environ.get("TFB_GRAPHS", "1") != "0"
GUARD_DOUBLES = 4096
_CANARY = -0x0123456789ABCDF  # int64 bit pattern of the guard words (a NaN-free double)
_guarded: list = []


def _buf(n: int, device, dtype=torch.float64) -> torch.Tensor:
    """Device buffer of n elements (guard bands around it in guard mode)."""
    n = max(1, int(n))
    if not GUARD:
        return torch.empty(n, dtype=dtype, device=device)
    per = 8 // torch.empty(0, dtype=dtype).element_size()
    g = GUARD_DOUBLES * per
    big = torch.empty(n + 2 * g, dtype=dtype, device=device)
    words = big.view(torch.int64) if dtype != torch.uint8 else None
    if words is None:  # byte buffers: whole words of guard on each side
        big.view(torch.uint8).fill_(0xA5)
    else:
        words.fill_(_CANARY)
    inner = big[g:g + n]
    inner.fill_(float("nan") if dtype == torch.float64 else 0)
    _guarded.append((big, g, n, dtype))
    return inner


def check_guards() -> list:
    """Indices of guarded buffers whose canaries were overwritten (guard mode)."""
    bad = []
    for i, (big, g, n, dtype) in enumerate(_guarded):
        if dtype == torch.uint8:
            ok = bool((big[:g] == 0xA5).all() and (big[g + n:] == 0xA5).all())
        else:
            w = big.view(torch.int64)
            per = big.element_size() // 8 or 1
            ok = bool((w[:g // per] == _CANARY).all() and (w[(g + n) // per:] == _CANARY).all())
        if not ok:
            bad.append(i)
    return bad


def poison(*tensors) -> None:
    """Guard mode: fill kernel outputs with NaN so stale reads propagate."""
    if GUARD:
        for t in tensors:
            if t is not None and t.dtype == torch.float64:
                t.fill_(float("nan"))


def require_cuda() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2306_08994_b200 needs a CUDA device (sm_100a); "
                           "there is no CPU fallback")
    return torch.device("cuda", torch.cuda.current_device())


def set_small_front_limit(m: int) -> int:
    """Front order up to which levels use the shared-memory kernels (<= 232).

    Lower values send levels through the blocked large-front kernels; tests
    use this to drive the large path with the reference's small goldens.
    Set it before `compile_execution`.  Returns the previous limit.
    """
    return int(_lib.load().tf_set_small_max_m(int(m)))


class _NoGC:
    """Garbage collection off around a CUDA graph capture: a collector pass
    during the capture can destroy an unreachable earlier graph (another
    DevicePlan's), and destroying a graph while a stream captures invalidates
    the capture ("operation not permitted when stream is capturing")."""

    def __enter__(self):
        import gc
        self._was = gc.isenabled()
        gc.collect()
        gc.disable()
        return self

    def __exit__(self, *exc):
        import gc
        if self._was:
            gc.enable()
        return False


def _ptr(t: Optional[torch.Tensor]):
    return None if t is None else C.c_void_p(t.data_ptr())


class DeviceLevel:
    def __init__(self, lib, lt, device, child_upd_stride: int, elem_stride: int, elem_ld: int):
        self.tables = lt
        m = lt.pat[:, _lib.PAT_M].astype(np.int64)
        k = lt.pat[:, _lib.PAT_K].astype(np.int64)
        self.n_fronts = lt.n_fronts
        self.max_m = lt.max_m
        fac = lt.pat[:, _lib.PAT_FAC].astype(np.int64)
        self.fac_stride = int((fac.max() + 3) // 4 * 4) if len(fac) else 0  # 32-byte slots
        self.upd_stride = int(_tri(m - k).max()) if len(m) else 0
        self.pattern_of = torch.from_numpy(lt.pattern_of).to(device)
        self.piv_off = torch.from_numpy(lt.piv_off).to(device)
        self.pat = torch.from_numpy(np.ascontiguousarray(lt.pat).ravel()).to(device)
        maps = lt.maps if len(lt.maps) else np.zeros(1, np.int32)
        self.maps = torch.from_numpy(maps).to(device)
        v = _lib.LevelView()
        v.level = lt.level
        v.n_fronts = lt.n_fronts
        v.n_patterns = lt.n_patterns
        v.max_m = lt.max_m
        v.max_k = lt.max_k
        v.max_upd = lt.max_upd
        v.is_leaf = 1 if lt.level == 0 else 0
        v.elem_ld = elem_ld
        v.fac_stride = self.fac_stride
        v.upd_stride = self.upd_stride
        v.child_upd_stride = child_upd_stride
        v.elem_stride = elem_stride
        v.pattern_of = self.pattern_of.data_ptr()
        v.piv_off = self.piv_off.data_ptr()
        v.pat = self.pat.data_ptr()
        v.maps = self.maps.data_ptr()
        v.level_fronts = lt.n_fronts
        self.aux_stride = int(lib.tf_level_aux_doubles(C.byref(v)))
        self.aux = None
        if self.aux_stride > 0:
            self.aux = _buf(self.n_fronts * self.aux_stride, device)
            v.aux = self.aux.data_ptr()
            v.aux_stride = self.aux_stride
        self.view = v
        # factor scratch owned by this plan (root-dataflow flags): concurrent
        # factorizations of different plans never share it
        self.ws_bytes = int(lib.tf_level_factor_workspace(C.byref(v)))
        self.ws = _buf(self.ws_bytes, device, torch.uint8) if self.ws_bytes > 0 else None

    @property
    def large(self) -> bool:
        return self.aux_stride > 0


class DevicePlan:
    def __init__(self, plan, fronts, device: Optional[torch.device] = None, values=None):
        self.device = device or require_cuda()
        self.lib = _lib.load()
        self.plan = plan
        native = plan.native
        self.n_dof = plan.n_dof
        self.n_pivots = native.n_pivots
        if isinstance(values, torch.Tensor):  # generated on the device (meshgen)
            elem_ld = int(values.shape[-1])
            elem_stride = 0 if values.dim() == 2 else elem_ld * elem_ld
            self.elem = values.to(device=self.device, dtype=torch.float64).reshape(-1).contiguous()
        else:
            vals = np.ascontiguousarray(fronts.values if values is None else values,
                                        dtype=np.float64)
            elem_ld = vals.shape[-1]
            elem_stride = 0 if vals.ndim == 2 else elem_ld * elem_ld
            self.elem = torch.from_numpy(vals.ravel()).to(self.device)
        self.levels: list[DeviceLevel] = []
        child = 0
        zprev = None
        for lt in native.levels:
            dl = DeviceLevel(self.lib, lt, self.device, child, elem_stride, elem_ld)
            # pivot-free subtrees: the front has no pivots and neither has any
            # descendant, so its forward update block is zero (the solve skips it)
            z = lt.front_k() == 0
            kids = None
            if zprev is not None:
                kids = np.ones(lt.n_fronts, dtype=bool)
                nc = len(zprev)
                i = np.arange(lt.n_fronts)
                kids &= zprev[np.minimum(2 * i, nc - 1)]
                has2 = 2 * i + 1 < nc
                kids[has2] &= zprev[2 * i[has2] + 1]
                z &= kids
            # bit 0: pivot-free subtree; bit 1: every child's subtree is pivot-free
            # (no child reads the front's backward block: it is not written)
            code = z.astype(np.uint8)
            if kids is not None:
                code |= kids.astype(np.uint8) << 1
            dl.zero_upd = torch.from_numpy(code).to(self.device)
            dl.view.zero_upd = dl.zero_upd.data_ptr()
            # implicit forward updates: pivots but no child contribution
            dl.implicit = (lt.front_k() > 0) & (np.ones(lt.n_fronts, dtype=bool) if zprev is None
                                                  else (kids if lt.level > 0 else True))
            zprev = z
            self.levels.append(dl)
            child = dl.upd_stride
        self._setup_implicit()
        self._setup_leaf_direct()
        self.pivot_order = torch.from_numpy(native.pivot_order).to(self.device)
        self._factors = None  # allocated on first single-device factorization
        self._upd = None
        self.err = torch.full((1,), -1, dtype=torch.int64, device=self.device)
        self._solve_nrhs = 0
        self._blk = None
        self._side = None     # second stream of factor_solve (overlapped forward sweep)
        self._lvl_ev = None
        self._fgraph = None   # (threshold, CUDA graph) of factor() (public API path)
        self._sgraphs = {}    # rhs shape -> (graph, static b, static x) of solve_into()
        self.fuse_bottom = True  # run the lowest levels as one subtree kernel when possible
        self.split_top = int(os.environ.get("TFB_SPLIT_TOP", "2"))  # concurrent top slices
        self.split_fronts = int(os.environ.get("TFB_SPLIT_FRONTS", "1024"))
        self._split = None
        self._tiny_ok = None  # whole tree in one launch (tf_tree_small_ok), decided once
        self.fwd_overlap_top = int(os.environ.get("TFB_FWD_OVERLAP_TOP", "1"))
        self.implicit_min_nrhs = int(os.environ.get("TFB_IMPLICIT_MIN_NRHS", "1"))
        self.fuse_cap = FUSE_CAP_DEFAULT  # max fused levels (TFB_FUSE_LEVELS overrides)

    def _setup_implicit(self) -> None:
        """Implicit forward updates (tf_level_view.implicit_upd) on small levels
        whose parent level is small with at most 8 pivots per front (the group
        and column sweeps read them; TFB_IMPLICIT_UPD=0 disables)."""
        on = os.environ.get("TFB_IMPLICIT_UPD", "1") != "0"
        small_max = int(self.lib.tf_set_small_max_m(0)) if on else 0  # query the split
        for L, dl in enumerate(self.levels):
            imp = getattr(dl, "implicit", None)
            dl.implicit_t = None
            dl.view.implicit_upd = None
            if not on or imp is None or L + 1 >= len(self.levels) or not imp.any():
                continue
            par = self.levels[L + 1]
            if dl.max_m > small_max or par.max_m > small_max or par.tables.max_k > 8:
                continue
            dl.implicit_t = torch.from_numpy(imp.astype(np.uint8)).to(self.device)
            dl.view.implicit_upd = dl.implicit_t.data_ptr()

    def _setup_leaf_direct(self) -> None:
        """Leaf pass-through (tf_level_view.leaf_direct): leaves without pivots
        write no update and level 1 reads their element matrices instead --
        the leaf level's update round trip through device memory disappears
        (2D Q1: 99.99% of the leaves).  Needs level 1 on the shared-memory
        path; TFB_LEAF_DIRECT=0 disables."""
        on = os.environ.get("TFB_LEAF_DIRECT", "1") != "0"
        if len(self.levels) < 2:
            return
        small_max = int(self.lib.tf_set_small_max_m(0))  # query the split
        l0, l1 = self.levels[0], self.levels[1]
        use = on and l1.max_m <= small_max
        for dl in (l0, l1):
            dl.view.leaf_direct = 1 if use else 0
        l1.view.src_pattern_of = l0.view.pattern_of if use else None
        l1.view.src_pat = l0.view.pat if use else None
        l1.view.src_maps = None
        if not use:
            return
        # per leaf pattern: entry e = (pa, pb), pa >= pb, of the leaf's packed
        # update (front order) -> index of its element-matrix entry, lower part
        # (rows inv[pa], inv[pb] of the element; inv = the pattern's inverse map)
        lt = l0.tables
        ld = l0.view.elem_ld
        tabs, offs, pos = [], [], lt.n_patterns
        for p in range(lt.n_patterns):
            m = int(lt.pat[p, _lib.PAT_M])
            inv = lt.maps[lt.pat[p, _lib.PAT_IOFF]:lt.pat[p, _lib.PAT_IOFF] + m].astype(np.int64)
            pa, pb = np.tril_indices(m)
            ra, rb = inv[pa], inv[pb]
            tabs.append((np.maximum(ra, rb) * ld + np.minimum(ra, rb)).astype(np.int32))
            offs.append(pos)
            pos += len(tabs[-1])
        arr = np.concatenate([np.asarray(offs, np.int32)] + tabs)
        l1.leaf_index = torch.from_numpy(arr).to(self.device)
        l1.view.src_maps = l1.leaf_index.data_ptr()

    @property
    def factors(self):
        if self._factors is None:
            self._factors = [_buf(dl.n_fronts * dl.fac_stride, self.device)
                             for dl in self.levels]
            for dl, t in zip(self.levels, self._factors):
                dl.view.factors = t.data_ptr()
        return self._factors

    @property
    def upd(self):
        if self._upd is None:
            upd_max = max(dl.n_fronts * dl.upd_stride for dl in self.levels)
            self._upd = [_buf(upd_max, self.device) for _ in range(2)]
        return self._upd

    # ---- factorization -----------------------------------------------------------
    def factor_level(self, L: int, threshold: float, sp, child=None) -> None:
        dl = self.levels[L]
        prev = child if child is not None else (self.upd[(L - 1) & 1] if L > 0 else None)
        rc = self.lib.tf_level_factor(C.byref(dl.view), _ptr(prev), _ptr(self.elem),
                                      _ptr(self.factors[L]), _ptr(self.upd[L & 1]),
                                      C.c_double(threshold), _ptr(self.err), _ptr(dl.ws),
                                      dl.ws_bytes, sp)
        _lib.check(rc, f"tf_level_factor(level {L})")

    @property
    def fused_levels(self) -> int:
        """Bottom levels run as one subtree launch (0: off; tf_subtree_fusable)."""
        if not self.fuse_bottom:
            return 0
        arr = (_lib.LevelView * len(self.levels))(*[dl.view for dl in self.levels])
        n = int(self.lib.tf_subtree_fusable(C.cast(arr, C.c_void_p), len(self.levels)))
        cap = self.fuse_cap
        if cap == 0 and self.levels and self.levels[0].n_fronts <= FUSE_AUTO_MAX_LEAVES:
            cap = 10  # launch-bound trees: one subtree launch instead of one per level
        cap = int(os.environ.get("TFB_FUSE_LEVELS", str(cap)))
        n = min(n, cap)
        return n if n >= 2 else 0

    def factor(self, threshold: float, stream: Optional[torch.cuda.Stream] = None,
               level_hook=None) -> None:
        """Enqueue every level on `stream`; no host synchronisation.

        level_hook(L), if given, runs after the launches that complete level L
        (fused bottom levels complete together)."""
        st = stream or torch.cuda.current_stream(self.device)
        sp = C.c_void_p(st.cuda_stream)
        self.err.fill_(-1)
        if GUARD:
            poison(*self.factors, *self.upd, *[dl.aux for dl in self.levels])
        if self._tiny():
            self._tree_call(threshold, None, None, 1, 0, sp)
            if level_hook is not None:
                for L in range(len(self.levels)):
                    level_hook(L)
            return
        nf = self.fused_levels
        if nf >= 2:
            views = (_lib.LevelView * nf)(*[dl.view for dl in self.levels[:nf]])
            facs = (C.c_void_p * nf)(*[self.factors[L].data_ptr() for L in range(nf)])
            rc = self.lib.tf_subtree_factor(C.cast(views, C.c_void_p), nf,
                                            C.cast(facs, C.c_void_p), _ptr(self.elem),
                                            _ptr(self.upd[(nf - 1) & 1]), C.c_double(threshold),
                                            _ptr(self.err), sp)
            _lib.check(rc, f"tf_subtree_factor(levels 0..{nf - 1})")
            if level_hook is not None:
                for L in range(nf):
                    level_hook(L)
        sp_ = self._split_plan()
        lo = max(nf, 0) if nf >= 2 else 0
        S, R = sp_ if sp_ is not None else (len(self.levels), len(self.levels))
        for L in range(lo, min(S, len(self.levels))):
            self.factor_level(L, threshold, sp)
            if level_hook is not None:
                level_hook(L)
        if sp_ is not None:
            self._factor_split(threshold, st, S, R)
            if level_hook is not None:
                for L in range(S, R):
                    level_hook(L)
            for L in range(R, len(self.levels)):
                # level R reads the slices' last level from the boundary buffer
                self.factor_level(L, threshold, sp, child=self._split[4] if L == R else None)
                if level_hook is not None:
                    level_hook(L)

    # ---- tiny trees: one launch --------------------------------------------------
    def _tiny(self) -> bool:
        """The whole tree qualifies for the one-launch kernel
        (tf_tree_small_ok; TFB_TINY_TREE=0 disables)."""
        if self._tiny_ok is None:
            self.factors  # the kernel reads the factor pointers from the views
            arr = (_lib.LevelView * len(self.levels))(*[dl.view for dl in self.levels])
            self._tiny_ok = (os.environ.get("TFB_TINY_TREE", "1") != "0" and
                             bool(self.lib.tf_tree_small_ok(C.cast(arr, C.c_void_p),
                                                            len(self.levels))))
        return self._tiny_ok

    def _tree_call(self, threshold: float, b, x, do_factor: int, do_solve: int, sp) -> None:
        arr = (_lib.LevelView * len(self.levels))(*[dl.view for dl in self.levels])
        if do_solve:
            blk = self._blocks(1)
            if GUARD:
                poison(*blk, self._y)
        rc = self.lib.tf_tree_factor_solve(
            C.cast(arr, C.c_void_p), len(self.levels), _ptr(self.elem), _ptr(self.upd[0]),
            _ptr(self.upd[1]), C.c_double(threshold), _ptr(self.err),
            _ptr(self.pivot_order) if do_solve else None, self.n_pivots, self.n_dof,
            _ptr(b), _ptr(x), _ptr(self._y) if do_solve else None,
            _ptr(self._blk[0]) if do_solve else None, _ptr(self._blk[1]) if do_solve else None,
            do_factor, do_solve, sp)
        _lib.check(rc, "tf_tree_factor_solve")

    # ---- concurrent top subtrees -------------------------------------------------
    def _split_plan(self):
        """(S, R): levels S .. R-1 are factored as `split_top` concurrent
        slices (independent subtrees of the top levels, each on its own
        stream with its own lookahead streams), the levels from R (fewer
        fronts than slices) after them; None when off (TFB_SPLIT_TOP=1) or
        the tree does not split evenly.  S is the lowest large level with at
        most `split_fronts` fronts from which every level splits evenly (the
        lookahead levels, whose pivot chains leave SMs idle)."""
        H = self.split_top
        n = len(self.levels)
        if H < 2 or n < 3 or self.levels[-1].n_fronts != 1:
            return None
        # R: first level with fewer than H fronts (it and the levels above run whole)
        R = next(L for L in range(n) if self.levels[L].n_fronts < H)

        def even(S):
            for L in range(S, R):
                nl = self.levels[L].n_fronts
                if nl % H or (L > S and self.levels[L - 1].n_fronts != 2 * nl):
                    return False
            return True
        for S in range(1, R):  # the lowest qualifying level from which the top splits evenly
            if self.levels[S].large and self.levels[S].n_fronts <= self.split_fronts and even(S):
                return S, R
        return None

    def _factor_split(self, threshold: float, st, S: int, R: int) -> None:
        from .distributed import _slice_view
        H = self.split_top
        if self._split is None or self._split[0] != (S, R, H):
            streams = [torch.cuda.Stream(self.device) for _ in range(H)]
            per = max([self.levels[L].n_fronts // H * self.levels[L].upd_stride
                       for L in range(S, R - 1)] or [1])
            bufs = [[_buf(per, self.device) for _ in range(2)] for _ in range(H)]
            ws = [[(_buf(self.levels[L].ws_bytes, self.device, torch.uint8)
                    if self.levels[L].ws_bytes > 0 else None) for L in range(n_)]
                  for n_ in [len(self.levels)] * H]
            # the last sliced level writes a buffer of its own: the shared
            # ping-pong buffer of its parity may still be read by the other
            # slice's first level
            bnd = _buf(self.levels[R - 1].n_fronts * self.levels[R - 1].upd_stride, self.device)
            self._split = ((S, R, H), streams, bufs, ws, bnd)
        _, streams, bufs, ws, bnd = self._split
        if GUARD:
            poison(*[b for hb in bufs for b in hb], bnd)
        for h in range(H):
            streams[h].wait_stream(st)
        for L in range(S, R):
            dl = self.levels[L]
            nl = dl.n_fronts // H
            for h in range(H):
                f0 = h * nl
                cb = 0 if L == S else h * self.levels[L - 1].n_fronts // H
                v = _slice_view(dl.view, f0, nl, child_base=cb)
                fac = self.factors[L].data_ptr() + 8 * f0 * dl.fac_stride
                v.factors = fac
                if dl.aux is not None:
                    v.aux = dl.aux.data_ptr() + 8 * f0 * dl.aux_stride
                child = self.upd[(L - 1) & 1] if L == S else bufs[h][(L - 1) & 1]
                if L == R - 1:  # the first whole level reads every child from one buffer
                    out = bnd.data_ptr() + 8 * f0 * dl.upd_stride
                else:
                    out = bufs[h][L & 1].data_ptr()
                w = ws[h][L]
                rc = self.lib.tf_level_factor(C.byref(v), _ptr(child), _ptr(self.elem),
                                              C.c_void_p(fac), C.c_void_p(out),
                                              C.c_double(threshold), _ptr(self.err), _ptr(w),
                                              dl.ws_bytes if w is not None else 0,
                                              C.c_void_p(streams[h].cuda_stream))
                _lib.check(rc, f"tf_level_factor(level {L}, slice {h})")
        for h in range(H):
            st.wait_stream(streams[h])

    def zero_pivot_position(self) -> int:
        """-1, or the pivot-order position of the earliest pivot at/below threshold."""
        return int(self.err.item())

    # ---- solve -------------------------------------------------------------------
    def _blocks(self, nrhs: int):
        if self._solve_nrhs != nrhs:
            n = max(dl.n_fronts * dl.max_m for dl in self.levels) * nrhs
            self._blk = [_buf(n, self.device) for _ in range(2)]
            self._y = _buf(self.n_pivots * nrhs, self.device)
            ws = max(int(self.lib.tf_level_solve_workspace(C.byref(dl.view), nrhs))
                     for dl in self.levels)
            self._ws = _buf(ws // 8, self.device)
            self._ws_bytes = ws
            self._solve_nrhs = nrhs
        return self._blk

    def _solve_begin(self, b: torch.Tensor, x: torch.Tensor, sp) -> int:
        nrhs = 1 if b.dim() == 1 else b.shape[1]
        # implicit forward updates pay off only with several columns (the
        # parent re-reads the child's panel rows, k per update row, instead of
        # one update row per column): on below implicit_min_nrhs columns
        on = nrhs >= self.implicit_min_nrhs
        for dl in self.levels:
            t = getattr(dl, "implicit_t", None)
            dl.view.implicit_upd = t.data_ptr() if (on and t is not None) else None
        blk = self._blocks(nrhs)
        if GUARD:
            poison(*blk, self._y)  # (the workspace's flags must start at zero: not poisoned)
        if x.data_ptr() != b.data_ptr():
            x.copy_(b)  # DOFs outside every front stay as given (engine.py:481)
        _lib.check(self.lib.tf_permute_rows(_ptr(self.pivot_order), self.n_pivots, _ptr(x),
                                            _ptr(self._y), nrhs, 0, sp), "tf_permute_rows")
        return nrhs

    def _solve_fwd_level(self, L: int, nrhs: int, sp) -> None:
        dl = self.levels[L]
        blk = self._blk
        child = self.levels[L - 1] if L > 0 else None
        rc = self.lib.tf_level_solve_fwd(C.byref(dl.view), C.byref(child.view) if child else None,
                                         _ptr(self.factors[L]), _ptr(blk[(L - 1) & 1]) if L else None,
                                         child.max_m if child else 0, _ptr(blk[L & 1]), dl.max_m,
                                         _ptr(self._y), nrhs, _ptr(self._ws), self._ws_bytes, sp)
        _lib.check(rc, f"tf_level_solve_fwd(level {L})")

    def _solve_end(self, x: torch.Tensor, nrhs: int, sp) -> None:
        """Backward sweep (root -> leaves) and the scatter back to natural order."""
        blk = self._blk
        nl = len(self.levels)
        for L in range(nl - 1, -1, -1):
            dl = self.levels[L]
            parent = self.levels[L + 1] if L + 1 < nl else None
            rc = self.lib.tf_level_solve_bwd(C.byref(dl.view),
                                             C.byref(parent.view) if parent else None,
                                             _ptr(self.factors[L]),
                                             _ptr(blk[(L + 1) & 1]) if parent else None,
                                             parent.max_m if parent else 0, _ptr(blk[L & 1]),
                                             dl.max_m, _ptr(self._y), nrhs, _ptr(self._ws),
                                             self._ws_bytes, sp)
            _lib.check(rc, f"tf_level_solve_bwd(level {L})")
        _lib.check(self.lib.tf_permute_rows(_ptr(self.pivot_order), self.n_pivots, _ptr(self._y),
                                            _ptr(x), nrhs, 1, sp), "tf_permute_rows")

    def solve_into(self, b: torch.Tensor, x: torch.Tensor,
                   stream: Optional[torch.cuda.Stream] = None) -> None:
        """x = A^-1 b for row-major (n, nrhs) device tensors (b may alias x)."""
        st = stream or torch.cuda.current_stream(self.device)
        sp = C.c_void_p(st.cuda_stream)
        if (b.dim() == 1 or b.shape[1] == 1) and self._tiny():
            self._tree_call(0.0, b, x, 0, 1, sp)
            return
        nrhs = self._solve_begin(b, x, sp)
        for L in range(len(self.levels)):
            self._solve_fwd_level(L, nrhs, sp)
        self._solve_end(x, nrhs, sp)

    def factor_solve(self, threshold: float, b: torch.Tensor, x: torch.Tensor,
                     stream: Optional[torch.cuda.Stream] = None) -> None:
        """factor(threshold) then x = A^-1 b, with the forward sweep overlapped.

        The forward sweep of level L needs only the factors of levels <= L.
        The top levels' factorization is a latency-bound pivot chain (the
        root's dataflow kernel leaves most SM issue slots idle), so the
        forward sweeps of every level below the top `fwd_overlap_top` levels
        run on a second stream while those top levels are factored
        (TFB_FWD_OVERLAP_TOP, default 1: the root); the top levels' sweeps
        and the backward sweep follow the factorization.  Same kernels and
        order per stream as factor() + solve_into(): identical results."""
        st = stream or torch.cuda.current_stream(self.device)
        if (b.dim() == 1 or b.shape[1] == 1) and self._tiny():
            self.err.fill_(-1)
            if GUARD:
                poison(*self.factors, *self.upd)
            self._tree_call(threshold, b, x, 1, 1, C.c_void_p(st.cuda_stream))
            return
        if self._side is None:
            self._side = torch.cuda.Stream(self.device)
            self._lvl_ev = [torch.cuda.Event() for _ in self.levels]
        ss = self._side
        ssp = C.c_void_p(ss.cuda_stream)
        nrhs = 1 if b.dim() == 1 else b.shape[1]
        self._blocks(nrhs)
        ss.wait_stream(st)                       # b (and everything before) ready
        with torch.cuda.stream(ss):
            self._solve_begin(b, x, ssp)
        nl = len(self.levels)
        top = min(max(self.fwd_overlap_top, 0), nl)
        last = nl - 1 - top  # sweeps of levels <= last overlap the top levels' factorization
        state = {"next": 0}

        def hook(L):
            if L == last:
                self._lvl_ev[L].record(st)
                ss.wait_event(self._lvl_ev[L])
                for n in range(last + 1):
                    self._solve_fwd_level(n, nrhs, ssp)
                state["next"] = last + 1

        self.factor(threshold, st, level_hook=hook if last >= 0 else None)
        ss.wait_stream(st)
        for L in range(state["next"], nl):
            self._solve_fwd_level(L, nrhs, ssp)
        self._solve_end(x, nrhs, ssp)
        st.wait_stream(ss)

    def capture(self, threshold: float, b: torch.Tensor, x: torch.Tensor,
                warmup: bool = True, overlap: bool = False) -> "torch.cuda.CUDAGraph":
        """One CUDA graph of a whole factorization + solve (every level's
        launches, the lookahead streams' fork/join, the wavefront sweeps).

        `b` and `x` are the static right-hand-side / solution buffers and
        `self.elem` the static leaf values: update them in place, then
        `graph.replay()`.  Removes the per-launch host cost (hundreds of
        ctypes launches per step on the large configs, most of the step on
        the small ones).  The zero-pivot flag is still read from `self.err`.
        """
        stream = torch.cuda.Stream(self.device)
        stream.wait_stream(torch.cuda.current_stream(self.device))
        with torch.cuda.stream(stream):
            if warmup or overlap:  # first calls create streams, kernel attributes, workspaces
                if overlap:
                    self.factor_solve(threshold, b, x, stream)
                else:
                    self.factor(threshold, stream)
                    self.solve_into(b, x, stream)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with _NoGC(), torch.cuda.graph(g, stream=stream):
            st = torch.cuda.current_stream(self.device)
            if overlap:  # forward sweep overlapped with the factorization (factor_solve)
                self.factor_solve(threshold, b, x, st)
            else:
                self.factor(threshold, st)
                self.solve_into(b, x, st)
        torch.cuda.current_stream(self.device).wait_stream(stream)
        return g

    # ---- public-API path: cached CUDA graphs ------------------------------------
    def _capture(self, fn) -> "torch.cuda.CUDAGraph":
        cs = torch.cuda.Stream(self.device)
        cs.wait_stream(torch.cuda.current_stream(self.device))
        g = torch.cuda.CUDAGraph()
        with _NoGC(), torch.cuda.graph(g, stream=cs):
            fn(torch.cuda.current_stream(self.device))
        torch.cuda.current_stream(self.device).wait_stream(cs)
        return g

    def factor_graphed(self, threshold: float) -> None:
        """factor() on the current stream through a cached CUDA graph.

        The first call runs eagerly (creating streams, kernel attributes and
        buffers) and captures the launch sequence; later calls with the same
        threshold replay it (the leaf values are read from `self.elem`, which
        callers may overwrite in place).  Guard mode and TFB_GRAPHS=0 launch
        eagerly every time."""
        if not USE_GRAPHS or GUARD:
            return self.factor(threshold)
        if self._fgraph is not None and self._fgraph[0] == threshold:
            self._fgraph[1].replay()
            return
        self.factor(threshold)
        self._fgraph = (threshold, self._capture(lambda st: self.factor(threshold, st)))

    def solve_graphed(self, b: torch.Tensor, x: torch.Tensor) -> None:
        """solve_into() through a cached graph per column count, with static
        right-hand-side / solution buffers (two device copies per call)."""
        if not USE_GRAPHS or GUARD:
            return self.solve_into(b, x)
        shape = tuple(b.shape)
        ent = self._sgraphs.get(shape)
        if ent is None:
            gb = torch.empty_like(b)
            gx = torch.empty_like(b)
            gb.copy_(b)
            self.solve_into(gb, gx)
            g = self._capture(lambda st: self.solve_into(gb, gx, st))
            self._sgraphs[shape] = (g, gb, gx)
            x.copy_(gx)
            return
        g, gb, gx = ent
        gb.copy_(b)
        g.replay()
        x.copy_(gx)

    def factor_solve_graphed(self, threshold: float, b: torch.Tensor, x: torch.Tensor) -> None:
        """factor_solve() through a cached graph per (threshold, rhs shape)."""
        if not USE_GRAPHS or GUARD:
            return self.factor_solve(threshold, b, x)
        key = (threshold, tuple(b.shape))
        ent = self._sgraphs.get(key)
        if ent is None:
            gb, gx = torch.empty_like(b), torch.empty_like(b)
            gb.copy_(b)
            self.factor_solve(threshold, gb, gx)
            g = self._capture(lambda st: self.factor_solve(threshold, gb, gx, st))
            self._sgraphs[key] = (g, gb, gx)
            x.copy_(gx)
            return
        g, gb, gx = ent
        gb.copy_(b)
        g.replay()
        x.copy_(gx)

    def launches_per_factor(self) -> int:
        """Kernel launches one factorization issues (tf_level_launch_count;
        levels factored as concurrent slices launch their sequence per slice)."""
        if self._tiny():
            return 1
        sp_ = self._split_plan()
        n = 0
        for L, dl in enumerate(self.levels):
            c = int(self.lib.tf_level_launch_count(C.byref(dl.view), 1, 0))
            n += c * (self.split_top if sp_ is not None and sp_[0] <= L < sp_[1] else 1)
        return n

    def launches_per_solve(self, nrhs: int) -> int:
        if nrhs == 1 and self._tiny():
            return 1
        n = 2  # permutations
        for dl in self.levels:
            n += int(self.lib.tf_level_launch_count(C.byref(dl.view), nrhs, 1))
            n += int(self.lib.tf_level_launch_count(C.byref(dl.view), nrhs, 2))
        return n
