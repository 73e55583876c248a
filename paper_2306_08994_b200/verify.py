"""Debug-mode structural checks (analogue of engine.py:426-461).

The reference checks that every dependency edge advances Foata classes and
that no class writes a cell twice.  At front granularity the same contracts
are: every front's children sit exactly one class below it, the schedule
covers every node once, and within a class each front writes a disjoint
factor slot and update slot (guaranteed by fixed strides) while its
extend-add maps are injective (no two child entries land on one front cell).
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .errors import ContractViolationError


def check_level_schedule(plan, schedule) -> None:
    from .schedule import AtomicFoataSchedule
    native = plan.native
    if isinstance(schedule, AtomicFoataSchedule):
        # the atomic FNF of the same plan: its task count must be the plan's
        st = native.atomic_fnf()[0] if native.keep_lists else None
        if st is not None and int(st.n_tasks) != sum(schedule.widths):
            raise ContractViolationError("atomic schedule does not belong to this plan")
    elif schedule is not None and tuple(schedule.level_sizes) != tuple(plan.tree.level_sizes):
        raise ContractViolationError("schedule classes do not match the tree levels")
    for L, lt in enumerate(native.levels):
        if L > 0 and lt.n_fronts != (native.levels[L - 1].n_fronts + 1) // 2:
            raise ContractViolationError(f"level {L}: not a pairwise join of level {L - 1}")
        for p in range(lt.n_patterns):
            row = lt.pat[p]
            m, k = int(row[_lib.PAT_M]), int(row[_lib.PAT_K])
            if not 0 <= k <= m:
                raise ContractViolationError(f"level {L} pattern {p}: k={k} m={m}")
            for c in range(int(row[_lib.PAT_NSRC])):
                off, ln = int(row[_lib.PAT_OFF0 + c]), int(row[_lib.PAT_LEN0 + c])
                mp = lt.maps[off:off + ln]
                if len(np.unique(mp)) != ln or (ln and (mp.min() < 0 or mp.max() >= m)):
                    raise ContractViolationError(
                        f"level {L} pattern {p} source {c}: extend-add map not injective")
