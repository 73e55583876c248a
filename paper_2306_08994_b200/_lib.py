"""ctypes binding of libtfb200.so (C ABI: include/tracefront_b200.h).

The shared library is built in-tree by `__graft_entry__.build()` (or
`make -C paper_2306_08994_b200/csrc`).  There is no fallback: if the library
is missing, importing the numeric path raises.
"""

from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

LIB_PATH = Path(os.environ.get("TFB_LIB", Path(__file__).resolve().parent / "libtfb200.so"))

TF_OK = 0
TF_ZERO_PIVOT = 2
TF_ERR_INVALID = -1
TF_ERR_CUDA = -2
TF_ERR_STRAY = -3

PAT_WIDTH = 12
(PAT_M, PAT_K, PAT_NSRC, PAT_LEN0, PAT_LEN1, PAT_OFF0, PAT_OFF1, PAT_LEAF, PAT_IOFF, PAT_KP,
 PAT_FAC, PAT_SOFF) = range(12)


class PlanSummary(C.Structure):
    _fields_ = [
        ("n_dof", C.c_int64), ("n_leaves", C.c_int64), ("n_nodes", C.c_int64),
        ("n_pivots", C.c_int64), ("n_levels", C.c_int32), ("max_m", C.c_int32),
        ("max_k", C.c_int32), ("keep_lists", C.c_int32),
    ]


class FnfStats(C.Structure):
    _fields_ = [
        ("n_tasks", C.c_int64), ("n_edges", C.c_int64), ("n_cells", C.c_int64),
        ("max_width", C.c_int64), ("n_classes", C.c_int32), ("singular", C.c_int32),
        ("n_divisions", C.c_int64), ("n_multiplications", C.c_int64),
    ]


class LevelHost(C.Structure):
    _fields_ = [
        ("level", C.c_int32), ("n_fronts", C.c_int32), ("n_patterns", C.c_int32),
        ("max_m", C.c_int32), ("max_k", C.c_int32), ("max_upd", C.c_int32),
        ("node_base", C.c_int64), ("piv_base", C.c_int64), ("n_pivots", C.c_int64),
        ("maps_len", C.c_int64),
        ("pattern_of", C.POINTER(C.c_int32)), ("piv_off", C.POINTER(C.c_int64)),
        ("pat", C.POINTER(C.c_int32)), ("maps", C.POINTER(C.c_int32)),
    ]


class LevelView(C.Structure):
    _fields_ = [
        ("level", C.c_int32), ("n_fronts", C.c_int32), ("n_patterns", C.c_int32),
        ("max_m", C.c_int32), ("max_k", C.c_int32), ("max_upd", C.c_int32),
        ("is_leaf", C.c_int32), ("elem_ld", C.c_int32),
        ("fac_stride", C.c_int64), ("upd_stride", C.c_int64),
        ("child_upd_stride", C.c_int64), ("elem_stride", C.c_int64),
        ("pattern_of", C.c_void_p), ("piv_off", C.c_void_p),
        ("pat", C.c_void_p), ("maps", C.c_void_p),
        ("aux", C.c_void_p), ("aux_stride", C.c_int64),
        ("front_base", C.c_int64), ("child_base", C.c_int64),
        ("level_fronts", C.c_int64), ("zero_upd", C.c_void_p),
        ("implicit_upd", C.c_void_p), ("factors", C.c_void_p),
        ("leaf_direct", C.c_int32), ("src_pattern_of", C.c_void_p),
        ("src_pat", C.c_void_p), ("src_maps", C.c_void_p),
    ]


# every symbol the header declares (checked by tests/test_capi.py)
EXPORTS = (
    "tf_mesh_tensor", "tf_plan_create", "tf_plan_destroy", "tf_plan_summary_get",
    "tf_plan_level", "tf_plan_pivot_order", "tf_plan_node_lists", "tf_plan_node_lists_len",
    "tf_level_factor_workspace", "tf_level_factor", "tf_level_solve_fwd",
    "tf_level_solve_bwd", "tf_permute_rows", "tf_level_launch_count", "tf_set_small_max_m", "tf_set_jitter",
    "tf_level_aux_doubles", "tf_level_solve_workspace", "tf_subtree_fusable",
    "tf_subtree_factor", "tf_timing_enable", "tf_timing_collect", "tf_timing_class_name",
    "tf_build_info", "tf_atomic_fnf", "tf_mesh_tensor_device_workspace",
    "tf_mesh_tensor_device", "tf_mesh_element_values_device", "tf_level_solve_cooperative",
    "tf_tree_small_ok", "tf_tree_factor_solve",
)

_lib = None


def load() -> C.CDLL:
    """Load the in-tree library once; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not LIB_PATH.exists():
        raise ImportError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
            "g.build()'` or `make -C paper_2306_08994_b200/csrc` (no CPU fallback exists)"
        )
    lib = C.CDLL(os.fspath(LIB_PATH))
    i32, i64, vp = C.c_int32, C.c_int64, C.c_void_p
    P_i64, P_i32 = C.POINTER(C.c_int64), C.POINTER(C.c_int32)
    lib.tf_mesh_tensor.argtypes = [i32, P_i64, i32, P_i64, P_i64, P_i32]
    lib.tf_mesh_tensor.restype = C.c_int
    lib.tf_plan_create.argtypes = [i64, i64, P_i64, i32, P_i32, i32, C.POINTER(vp)]
    lib.tf_plan_create.restype = C.c_int
    lib.tf_plan_destroy.argtypes = [vp]
    lib.tf_plan_destroy.restype = None
    lib.tf_plan_summary_get.argtypes = [vp, C.POINTER(PlanSummary)]
    lib.tf_plan_summary_get.restype = C.c_int
    lib.tf_plan_level.argtypes = [vp, i32, C.POINTER(LevelHost)]
    lib.tf_plan_level.restype = C.c_int
    lib.tf_plan_pivot_order.argtypes = [vp, P_i32]
    lib.tf_plan_pivot_order.restype = C.c_int
    lib.tf_plan_node_lists.argtypes = [vp, i32, P_i64, P_i32, P_i32]
    lib.tf_plan_node_lists.restype = C.c_int
    lib.tf_plan_node_lists_len.argtypes = [vp, i32]
    lib.tf_plan_node_lists_len.restype = i64
    lib.tf_atomic_fnf.argtypes = [vp, C.POINTER(FnfStats), P_i64, P_i32, i32]
    lib.tf_atomic_fnf.restype = C.c_int
    lib.tf_level_factor_workspace.argtypes = [C.POINTER(LevelView)]
    lib.tf_level_factor_workspace.restype = i64
    lib.tf_level_aux_doubles.argtypes = [C.POINTER(LevelView)]
    lib.tf_level_aux_doubles.restype = i64
    lib.tf_level_factor.argtypes = [C.POINTER(LevelView), vp, vp, vp, vp, C.c_double, vp, vp,
                                    i64, vp]
    lib.tf_level_factor.restype = C.c_int
    lib.tf_level_solve_fwd.argtypes = [C.POINTER(LevelView), C.POINTER(LevelView), vp, vp, i64,
                                       vp, i64, vp, i32, vp, i64, vp]
    lib.tf_level_solve_fwd.restype = C.c_int
    lib.tf_level_solve_bwd.argtypes = [C.POINTER(LevelView), C.POINTER(LevelView), vp, vp, i64,
                                       vp, i64, vp, i32, vp, i64, vp]
    lib.tf_level_solve_bwd.restype = C.c_int
    lib.tf_level_solve_workspace.argtypes = [C.POINTER(LevelView), i32]
    lib.tf_level_solve_workspace.restype = i64
    lib.tf_permute_rows.argtypes = [vp, i64, vp, vp, i32, i32, vp]
    lib.tf_permute_rows.restype = C.c_int
    lib.tf_level_launch_count.argtypes = [C.POINTER(LevelView), i32, i32]
    lib.tf_level_launch_count.restype = i32
    lib.tf_mesh_tensor_device_workspace.argtypes = [i32, C.POINTER(i64), i32]
    lib.tf_mesh_tensor_device_workspace.restype = i64
    lib.tf_mesh_tensor_device.argtypes = [i32, C.POINTER(i64), i32, vp, vp, vp, i64, vp]
    lib.tf_mesh_tensor_device.restype = C.c_int
    lib.tf_mesh_element_values_device.argtypes = [i32, C.POINTER(i64), i32, vp, vp, vp, vp, vp, vp]
    lib.tf_mesh_element_values_device.restype = C.c_int
    lib.tf_level_solve_cooperative.argtypes = [C.POINTER(LevelView), i32, i32]
    lib.tf_level_solve_cooperative.restype = i32
    lib.tf_tree_small_ok.argtypes = [vp, i32]
    lib.tf_tree_small_ok.restype = i32
    lib.tf_tree_factor_solve.argtypes = [vp, i32, vp, vp, vp, C.c_double, vp, vp, i64, i64, vp,
                                         vp, vp, vp, vp, i32, i32, vp]
    lib.tf_tree_factor_solve.restype = C.c_int
    lib.tf_set_jitter.argtypes = [C.c_uint32]
    lib.tf_set_jitter.restype = C.c_int
    lib.tf_set_small_max_m.argtypes = [i32]
    lib.tf_set_small_max_m.restype = i32
    lib.tf_subtree_fusable.argtypes = [vp, i32]
    lib.tf_subtree_fusable.restype = i32
    lib.tf_subtree_factor.argtypes = [vp, i32, vp, vp, vp, C.c_double, vp, vp]
    lib.tf_subtree_factor.restype = C.c_int
    lib.tf_timing_enable.argtypes = [i32]
    lib.tf_timing_enable.restype = None
    lib.tf_timing_collect.argtypes = [vp, vp, i32]
    lib.tf_timing_collect.restype = i32
    lib.tf_timing_class_name.argtypes = [i32]
    lib.tf_timing_class_name.restype = C.c_char_p
    lib.tf_build_info.argtypes = []
    lib.tf_build_info.restype = C.c_char_p
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    if rc == TF_OK:
        return
    if rc == TF_ERR_CUDA:
        raise RuntimeError(f"{what}: CUDA error (see stderr)")
    raise ValueError(f"{what}: invalid input (status {rc})")


def i64p(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_int64))


def i32p(arr):
    return arr.ctypes.data_as(C.POINTER(C.c_int32))


def kernel_timing(lib, n: int = 32):
    """Collect tf_timing: {class name: (total ms, launches)} (non-zero classes)."""
    import numpy as np
    ms = np.zeros(n)
    cnt = np.zeros(n, dtype=np.int64)
    k = lib.tf_timing_collect(ms.ctypes.data, cnt.ctypes.data, n)
    return {lib.tf_timing_class_name(i).decode(): (float(ms[i]), int(cnt[i]))
            for i in range(k) if cnt[i] > 0}
