"""Tensor-mesh generation on the GPU.

`element_table_device` builds the Morton-ordered element DOF table with the
CUDA kernels of csrc/mesh.cu (Morton keys, CUB radix sort, an exclusive scan
of owned-point counts, one thread per (element, local point)); it is bitwise
the host table of `TensorMesh.element_table` (tf_mesh_tensor).
`element_values_device` writes the per-element matrices of graded / weighted
meshes (width products x density x the unit reference matrix), bitwise the
host `TensorMesh.element_values`.  Both stay on the device: a `DevicePlan`
accepts the values tensor directly (no host stack, no upload).
"""

from __future__ import annotations

import ctypes as C
from typing import Optional

import numpy as np
import torch

from . import _lib
from .fem import TensorMesh, element_mass_matrix


def _dims(mesh: TensorMesh):
    return np.ascontiguousarray(mesh.shape, dtype=np.int64)


def element_table_device(mesh: TensorMesh, device: Optional[torch.device] = None):
    """(dofs int32 (n_el, (p+1)^d), order int64 (n_el,)) on the GPU, Morton order."""
    dev = device or torch.device("cuda", torch.cuda.current_device())
    lib = _lib.load()
    ns = _dims(mesh)
    ws_bytes = int(lib.tf_mesh_tensor_device_workspace(mesh.dim, _lib.i64p(ns), mesh.degree))
    if ws_bytes < 0:
        raise ValueError(f"mesh {mesh.shape} too large for the device generator")
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    dofs = torch.empty((mesh.n_elements, mesh.nloc), dtype=torch.int32, device=dev)
    order = torch.empty(mesh.n_elements, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev)
    rc = lib.tf_mesh_tensor_device(mesh.dim, _lib.i64p(ns), mesh.degree,
                                   C.c_void_p(dofs.data_ptr()), C.c_void_p(order.data_ptr()),
                                   C.c_void_p(ws.data_ptr()), ws_bytes, C.c_void_p(st.cuda_stream))
    _lib.check(rc, "tf_mesh_tensor_device")
    return dofs, order


def element_values_device(mesh: TensorMesh, order: torch.Tensor) -> torch.Tensor:
    """(n_el, nloc, nloc) float64 element matrices on the GPU (Morton order)."""
    dev = order.device
    lib = _lib.load()
    ref = [element_mass_matrix(1.0, mesh.degree) for _ in mesh.shape]
    out = ref[0]
    for m in ref[1:]:
        out = np.kron(m, out)
    ref_d = torch.from_numpy(np.ascontiguousarray(out)).to(dev)
    nodes = None
    if mesh.nodes is not None:
        nodes = torch.from_numpy(np.concatenate(mesh.nodes)).to(dev)
    dens = None if mesh.density is None else torch.from_numpy(mesh.density).to(dev)
    vals = torch.empty((mesh.n_elements, mesh.nloc, mesh.nloc), dtype=torch.float64, device=dev)
    ns = _dims(mesh)
    st = torch.cuda.current_stream(dev)
    ptr = lambda t: None if t is None else C.c_void_p(t.data_ptr())
    rc = lib.tf_mesh_element_values_device(mesh.dim, _lib.i64p(ns), mesh.degree, ptr(order),
                                           ptr(nodes), ptr(dens), ptr(ref_d), ptr(vals),
                                           C.c_void_p(st.cuda_stream))
    _lib.check(rc, "tf_mesh_element_values_device")
    return vals
