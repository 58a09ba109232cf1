"""ctypes wrapper of liboracle.so (plain C++ oracle, lfem_oracle.cpp).

TEST INFRASTRUCTURE ONLY — see the header of lfem_oracle.cpp.
Argument marshalling only; every number comes from the C++ oracle.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lfem_oracle.cpp")
_SO = os.path.join(_HERE, "liboracle.so")
_LIB = None

K_MASS, K_STIFF, K_STIFF_COEF = 1, 2, 4
KIND_BITS = {"M": K_MASS, "A": K_STIFF, "Aa": K_STIFF_COEF}
RHS_LOAD, RHS_KLL = 1, 2
RHS_KINDS = {"load": RHS_LOAD, "kll": RHS_KLL}
RHS_NCOMP = {RHS_LOAD: 1, RHS_KLL: 4}


class OracleError(RuntimeError):
    def __init__(self, code: int, elem: int = -1):
        super().__init__(f"oracle status {code} (element {elem})")
        self.code = code
        self.elem = elem


def build(force: bool = False) -> str:
    """Compile liboracle.so: -O2, no fast-math, no FP contraction."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < os.path.getmtime(_SRC):
        cmd = ["g++", "-std=c++17", "-O2", "-ffp-contract=off", "-fno-fast-math", "-pthread",
               "-shared", "-fPIC", "-o", _SO + ".tmp", _SRC]
        subprocess.run(cmd, check=True)
        os.replace(_SO + ".tmp", _SO)
    return _SO


class _Csr(ctypes.Structure):
    _fields_ = [("n_rows", ctypes.c_int64), ("nnz", ctypes.c_int64),
                ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
                ("col_idx", ctypes.POINTER(ctypes.c_int32)),
                ("vals", ctypes.POINTER(ctypes.c_double) * 3),
                ("bad_elem", ctypes.c_int64)]


def lib():
    global _LIB
    if _LIB is None:
        L = ctypes.CDLL(build())
        vp = ctypes.c_void_p
        L.oracle_assemble_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp,
                                           ctypes.c_int64, vp, vp, ctypes.c_int, ctypes.c_int64, vp,
                                           ctypes.c_int, ctypes.POINTER(_Csr)]
        L.oracle_free.argtypes = [ctypes.POINTER(_Csr)]
        L.oracle_element.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int, vp, vp, vp]
        L.oracle_rule.argtypes = [ctypes.c_int, vp, vp, vp]
        L.oracle_basis.argtypes = [ctypes.c_int, ctypes.c_int, vp, vp, vp]
        L.oracle_element_rhs.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, vp, vp, ctypes.c_int,
                                         ctypes.c_int, vp]
        L.oracle_assemble_rhs_rows.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int64, vp,
                                               ctypes.c_int64, vp, vp, ctypes.c_int, ctypes.c_int64, vp,
                                               ctypes.c_int, vp, vp, ctypes.POINTER(ctypes.c_int64)]
        _LIB = L
    return _LIB


def _p(a: Optional[np.ndarray]):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


@dataclass
class CsrRows:
    rows: np.ndarray        # global row ids (int64)
    row_ptr: np.ndarray     # int64, len(rows)+1
    col_idx: np.ndarray     # int32
    vals: dict              # kind name -> float64 array

    @property
    def nnz(self) -> int:
        return int(self.col_idx.size)


def assemble_rows(mesh, kinds: Sequence[str] = ("M", "A"), rows=None, coeff=None,
                  nthreads: Optional[int] = None) -> CsrRows:
    """Oracle CSR of the given global rows (default: all rows)."""
    L = lib()
    kmask = 0
    for k in kinds:
        kmask |= KIND_BITS[k]
    if rows is None:
        rows = np.arange(mesh.n_nodes, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
    if coeff is None:
        coeff = mesh.coeff
    cf = None if coeff is None else np.ascontiguousarray(coeff, dtype=np.float64)
    out = _Csr()
    nt = nthreads or (os.cpu_count() or 1)
    st = L.oracle_assemble_rows(mesh.domain, mesh.order, mesh.quad, mesh.n_nodes, _p(coords),
                                mesh.n_elems, _p(conn), _p(cf), kmask, rows.size, _p(rows), nt,
                                ctypes.byref(out))
    if st != 0:
        raise OracleError(st, out.bad_elem)
    try:
        n = out.n_rows
        nnz = out.nnz
        rp = np.ctypeslib.as_array(out.row_ptr, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(out.col_idx, shape=(max(nnz, 1),))[:nnz].copy()
        vals = {}
        for name, bit in KIND_BITS.items():
            if kmask & bit:
                idx = bit.bit_length() - 1
                vals[name] = np.ctypeslib.as_array(out.vals[idx], shape=(max(nnz, 1),))[:nnz].copy()
    finally:
        L.oracle_free(ctypes.byref(out))
    return CsrRows(rows, rp, ci, vals)


def element_matrices(domain: int, order: int, quad: int, X, u=None, formulation: int = 0):
    """Full local (M, A, Aa) of one element with nodes X (nref x 3)."""
    L = lib()
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = X.shape[0]
    uu = None if u is None else np.ascontiguousarray(u, dtype=np.float64)
    M = np.zeros((n, n))
    A = np.zeros((n, n))
    Aa = np.zeros((n, n))
    st = L.oracle_element(domain, order, quad, _p(X), _p(uu), formulation, _p(M), _p(A), _p(Aa))
    if st != 0:
        raise OracleError(st)
    return M, A, Aa


def _rhs_kind(kind) -> int:
    return RHS_KINDS[kind] if isinstance(kind, str) else int(kind)


def element_rhs(domain: int, order: int, quad: int, X, U, kind="load", formulation: int = 0) -> np.ndarray:
    """Local right-hand side (nref x ncomp) of one element; U is nref x ncomp nodal data
    (load: f; kll: (nu_1, nu_2, nu_3, H))."""
    L = lib()
    k = _rhs_kind(kind)
    X = np.ascontiguousarray(X, dtype=np.float64)
    n = X.shape[0]
    nc = RHS_NCOMP.get(k, 1)
    U = np.ascontiguousarray(np.asarray(U, dtype=np.float64).reshape(n, nc))
    F = np.zeros((n, nc))
    st = L.oracle_element_rhs(domain, order, quad, _p(X), _p(U), k, formulation, _p(F))
    if st != 0:
        raise OracleError(st)
    return F


def assemble_rhs_rows(mesh, u, kind="load", rows=None, nthreads: Optional[int] = None,
                      with_abs: bool = False):
    """Oracle right-hand side of the given global rows (default all): returns an
    (ncomp, n_rows) array (and the matching sum of |local entries| if with_abs).
    u: (ncomp, n_nodes) nodal data, component-major."""
    L = lib()
    k = _rhs_kind(kind)
    nc = RHS_NCOMP.get(k, 1)
    if rows is None:
        rows = np.arange(mesh.n_nodes, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64)
    coords = np.ascontiguousarray(mesh.coords, dtype=np.float64)
    conn = np.ascontiguousarray(mesh.conn, dtype=np.int32)
    uu = np.ascontiguousarray(np.asarray(u, dtype=np.float64).reshape(nc, mesh.n_nodes))
    out = np.zeros((nc, rows.size))
    oabs = np.zeros((nc, rows.size)) if with_abs else None
    bad = ctypes.c_int64(-1)
    nt = nthreads or (os.cpu_count() or 1)
    st = L.oracle_assemble_rhs_rows(mesh.domain, mesh.order, mesh.quad, mesh.n_nodes, _p(coords),
                                    mesh.n_elems, _p(conn), _p(uu), k, rows.size, _p(rows), nt,
                                    _p(out), _p(oabs), ctypes.byref(bad))
    if st != 0:
        raise OracleError(st, bad.value)
    return (out, oabs) if with_abs else out


def rule(quad: int):
    """(lam (nq,4), w (nq,)) of the oracle's quadrature rule."""
    L = lib()
    lam = np.zeros((64, 4))
    w = np.zeros(64)
    nq = ctypes.c_int(0)
    st = L.oracle_rule(quad, ctypes.byref(nq), _p(lam), _p(w))
    if st != 0:
        raise OracleError(st)
    return lam[:nq.value].copy(), w[:nq.value].copy()


def basis(domain: int, order: int, lam):
    """(phi (10,), grad (10,3)) at barycentric point lam."""
    L = lib()
    lam = np.ascontiguousarray(np.pad(np.asarray(lam, dtype=np.float64), (0, 4 - len(lam))))
    phi = np.zeros(10)
    grad = np.zeros((10, 3))
    st = L.oracle_basis(domain, order, _p(lam), _p(phi), _p(grad))
    if st != 0:
        raise OracleError(st)
    return phi, grad


def to_dense(c: CsrRows, n_cols: int, kind: str) -> np.ndarray:
    D = np.zeros((c.rows.size, n_cols))
    for i in range(c.rows.size):
        s, e = c.row_ptr[i], c.row_ptr[i + 1]
        D[i, c.col_idx[s:e]] = c.vals[kind][s:e]
    return D
