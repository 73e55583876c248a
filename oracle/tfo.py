"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of tf_oracle.c (see its header)."""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "_ref" / "libtforacle.so"
_lib = None


def load():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
        lib = C.CDLL(str(LIB))
        vp, i64, i32 = C.c_void_p, C.c_int64, C.c_int32
        lib.oracle_factor.argtypes = [i64, i64, i32, vp, vp, i64, C.POINTER(vp)]
        lib.oracle_factor.restype = C.c_int
        lib.oracle_free.argtypes = [vp]
        lib.oracle_solve.argtypes = [vp, vp]
        for f in ("oracle_n_piv", "oracle_n_u", "oracle_n_l"):
            getattr(lib, f).argtypes = [vp]
            getattr(lib, f).restype = i64
        lib.oracle_zero_pivot.argtypes = [vp, C.POINTER(i64), C.POINTER(i64)]
        lib.oracle_get.argtypes = [vp] + [vp] * 8
        _lib = lib
    return _lib


class OracleFactors:
    """Reference-arithmetic factors (bitwise equal to engine.py:500-552)."""

    def __init__(self, n_dof, elem_dofs, elem_vals):
        lib = load()
        dofs = np.ascontiguousarray(elem_dofs, dtype=np.int32)
        vals = np.ascontiguousarray(elem_vals, dtype=np.float64)
        n_elem, nloc = dofs.shape
        stride = 0 if vals.ndim == 2 else nloc * nloc
        h = C.c_void_p()
        rc = lib.oracle_factor(int(n_dof), n_elem, nloc, dofs.ctypes.data, vals.ctypes.data,
                               stride, C.byref(h))
        self._h, self._lib, self.n_dof = h, lib, int(n_dof)
        self.status = rc
        if rc < 0:
            raise MemoryError("oracle_factor failed")
        fr, pv = C.c_int64(), C.c_int64()
        lib.oracle_zero_pivot(h, C.byref(fr), C.byref(pv))
        self.zero_pivot = None if rc != 2 else (int(fr.value), int(pv.value))

    def arrays(self):
        lib, h = self._lib, self._h
        npiv, nu, nl = lib.oracle_n_piv(h), lib.oracle_n_u(h), lib.oracle_n_l(h)
        piv = np.empty(npiv, np.int32)
        uz, uy, uv = np.empty(nu, np.int32), np.empty(nu, np.int32), np.empty(nu)
        lx, lz, lv = np.empty(nl, np.int32), np.empty(nl, np.int32), np.empty(nl)
        diag = np.empty(npiv)
        p = lambda a: a.ctypes.data
        lib.oracle_get(h, p(piv), p(uz), p(uy), p(uv), p(lx), p(lz), p(lv), p(diag))
        return dict(pivot_order=piv, u_z=uz, u_y=uy, u_v=uv, l_x=lx, l_z=lz, l_v=lv, diag=diag)

    def dicts(self):
        a = self.arrays()
        u = {(int(z), int(y)): float(v) for z, y, v in zip(a["u_z"], a["u_y"], a["u_v"])}
        for z, d in zip(a["pivot_order"], a["diag"]):
            u[(int(z), int(z))] = float(d)
        l = {(int(x), int(z)): float(v) for x, z, v in zip(a["l_x"], a["l_z"], a["l_v"])}
        return u, l

    def solve(self, rhs):
        rhs = np.asarray(rhs, dtype=np.float64)
        if rhs.ndim == 2:
            return np.stack([self.solve(rhs[:, j]) for j in range(rhs.shape[1])], axis=1)
        b = np.ascontiguousarray(rhs.copy())
        self._lib.oracle_solve(self._h, b.ctypes.data)
        return b

    def __del__(self):
        try:
            if self._h:
                self._lib.oracle_free(self._h)
        except Exception:
            pass
