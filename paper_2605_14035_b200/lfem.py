"""Thin Python binding of liblfem.so (include/lfem.h).

Argument marshalling only: every step of the assembly runs in the CUDA
kernels of liblfem.so.  Same names as the C ABI.  PyTorch is used for device
memory and streams (torch.cuda tensors in, torch.cuda tensors out).

There is NO CPU fallback: if liblfem.so is missing, importing this module
raises; if no GPU is present, the entry points raise from CUDA.
"""
from __future__ import annotations

import ctypes
import os
from typing import Optional, Sequence

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
SO_PATH = os.environ.get("LFEM_SO") or os.path.join(_HERE, "liblfem.so")

LFEM_OK = 0
STATUS = {0: "LFEM_OK", 1: "LFEM_ERR_INVALID_ARG", 2: "LFEM_ERR_UNSUPPORTED", 3: "LFEM_ERR_INDEX",
          4: "LFEM_ERR_DEGENERATE", 5: "LFEM_ERR_NOMEM", 6: "LFEM_ERR_CUDA", 7: "LFEM_ERR_STATE"}
LFEM_SURFACE_TRI, LFEM_BULK_TET = 0, 1
LFEM_QUAD_DEFAULT, LFEM_QUAD_TRI3_DEG2, LFEM_QUAD_TRI6_DEG4, LFEM_QUAD_TET4_DEG2, LFEM_QUAD_TET11_DEG4 = range(5)
LFEM_QUAD_TRI16_DEG8, LFEM_QUAD_LINE2_DEG3, LFEM_QUAD_LINE3_DEG5, LFEM_QUAD_TET35_DEG7, LFEM_QUAD_LINE6_DEG11 = range(5, 10)
LFEM_MASS, LFEM_STIFF, LFEM_STIFF_COEF = 1, 2, 4
LFEM_NUMERIC_AUTO, LFEM_NUMERIC_V0, LFEM_NUMERIC_TILED, LFEM_NUMERIC_ROWS = 0, 1, 2, 3
LFEM_RHS_LOAD, LFEM_RHS_KLL = 1, 2
RHS_KINDS = {"load": LFEM_RHS_LOAD, "kll": LFEM_RHS_KLL}
KIND_BITS = {"M": LFEM_MASS, "A": LFEM_STIFF, "Aa": LFEM_STIFF_COEF}
KIND_INDEX = {"M": 0, "A": 1, "Aa": 2}

# symbols declared in include/lfem.h (the CPU test checks they are all exported)
EXPORTED = ("lfem_mesh_create", "lfem_mesh_destroy", "lfem_assemble_symbolic", "lfem_plan_destroy",
            "lfem_plan_info", "lfem_plan_set_variant", "lfem_assemble_numeric", "lfem_assemble_numeric_coords",
            "lfem_assemble_numeric_host", "lfem_csr_get", "lfem_spmv", "lfem_plan_check", "lfem_axpby",
            "lfem_numeric_launches", "lfem_error_element", "lfem_last_error", "lfem_version",
            "lfem_profile_enable", "lfem_profile_read", "lfem_set_allocator", "lfem_assemble_rhs",
            "lfem_rhs_ncomp", "lfem_rhs_launches", "lfem_cg_solve", "lfem_mcf_step",
            "lfem_solve_meanfree", "lfem_numeric_stats")


class LfemError(RuntimeError):
    def __init__(self, status: int, where: str):
        self.status = status
        self.element = int(_lib().lfem_error_element())
        msg = _lib().lfem_last_error().decode()
        super().__init__(f"{where}: {STATUS.get(status, status)}: {msg} (element {self.element})")


_LIB = None


def _lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(SO_PATH):
            raise ImportError(f"{SO_PATH} is missing: run paper_2605_14035_b200/build.py (no CPU fallback exists)")
        L = ctypes.CDLL(SO_PATH)
        vp, i64, u32, c_int = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint, ctypes.c_int
        pp = ctypes.POINTER(ctypes.c_void_p)
        L.lfem_mesh_create.argtypes = [c_int, c_int, c_int, i64, vp, i64, vp, vp, pp]
        L.lfem_mesh_destroy.argtypes = [vp]
        L.lfem_mesh_destroy.restype = None
        L.lfem_assemble_symbolic.argtypes = [vp, i64, i64, vp, pp]
        L.lfem_plan_destroy.argtypes = [vp]
        L.lfem_plan_destroy.restype = None
        L.lfem_plan_info.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.lfem_plan_set_variant.argtypes = [vp, c_int]
        L.lfem_assemble_numeric.argtypes = [vp, u32, vp, ctypes.c_void_p * 3, vp]
        L.lfem_assemble_numeric_coords.argtypes = [vp, u32, vp, vp, ctypes.c_void_p * 3, vp]
        L.lfem_assemble_numeric_host.argtypes = [vp, u32, vp, vp, ctypes.c_void_p * 3, vp]
        L.lfem_csr_get.argtypes = [vp, pp, pp]
        L.lfem_spmv.argtypes = [vp, vp, vp, vp, vp]
        L.lfem_plan_check.argtypes = [vp, vp]
        L.lfem_axpby.argtypes = [i64, ctypes.c_double, vp, ctypes.c_double, vp, vp, vp]
        L.lfem_numeric_launches.argtypes = [vp, u32]
        L.lfem_numeric_stats.argtypes = [vp, ctypes.POINTER(i64), ctypes.POINTER(i64)]
        L.lfem_profile_enable.argtypes = [vp, c_int]
        L.lfem_profile_read.argtypes = [vp, c_int, ctypes.POINTER(ctypes.c_char_p), ctypes.POINTER(ctypes.c_double),
                                        ctypes.POINTER(i64), ctypes.POINTER(c_int)]
        L.lfem_error_element.restype = i64
        L.lfem_last_error.restype = ctypes.c_char_p
        L.lfem_version.restype = ctypes.c_char_p
        L.lfem_set_allocator.argtypes = [vp, vp, vp]
        L.lfem_assemble_rhs.argtypes = [vp, c_int, vp, vp, vp, vp]
        L.lfem_rhs_ncomp.argtypes = [c_int]
        L.lfem_rhs_launches.argtypes = [vp, c_int]
        L.lfem_cg_solve.argtypes = [vp, vp, vp, vp, ctypes.c_double, c_int, ctypes.POINTER(c_int), vp]
        L.lfem_solve_meanfree.argtypes = [vp, vp, vp, vp, ctypes.c_double, c_int, ctypes.POINTER(c_int), vp]
        L.lfem_mcf_step.argtypes = [vp, ctypes.c_double, vp, vp, ctypes.c_double, c_int, ctypes.POINTER(c_int), vp]
        _LIB = L
    return _LIB


def _check(st: int, where: str):
    if st != LFEM_OK:
        raise LfemError(st, where)


def _dptr(t: Optional[torch.Tensor]):
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


def kinds_mask(kinds: Sequence[str]) -> int:
    m = 0
    for k in kinds:
        m |= KIND_BITS[k]
    return m


class Mesh:
    """lfem_mesh handle; keeps the borrowed coords/conn tensors alive."""

    def __init__(self, handle, coords, conn, domain, order, quad):
        self.handle = handle
        self.coords = coords
        self.conn = conn
        self.domain, self.order, self.quad = domain, order, quad
        self.n_nodes = int(coords.shape[0])
        self.n_elems = int(conn.shape[0])

    def __del__(self):
        if getattr(self, "handle", None) and _LIB is not None:
            _LIB.lfem_mesh_destroy(self.handle)
            self.handle = None


class Plan:
    """lfem_plan handle (keeps its mesh alive)."""

    def __init__(self, handle, mesh: Mesh, row_begin: int, row_end: int):
        self.handle = handle
        self.mesh = mesh
        self.row_begin, self.row_end = row_begin, row_end
        n_rows, nnz, nel = lfem_plan_info(self)
        self.n_rows, self.nnz, self.n_elems_local = n_rows, nnz, nel

    def destroy(self):
        if getattr(self, "handle", None) and _LIB is not None:
            _LIB.lfem_plan_destroy(self.handle)
            self.handle = None

    def __del__(self):
        self.destroy()


def lfem_mesh_create(domain: int, order: int, quad: int, coords: torch.Tensor, conn: torch.Tensor,
                     stream=None) -> Mesh:
    assert coords.is_cuda and coords.dtype == torch.float64 and coords.is_contiguous() and coords.dim() == 2
    assert conn.is_cuda and conn.dtype == torch.int32 and conn.is_contiguous() and conn.dim() == 2
    h = ctypes.c_void_p()
    st = _lib().lfem_mesh_create(domain, order, quad, coords.shape[0], _dptr(coords), conn.shape[0], _dptr(conn),
                                 _stream(stream), ctypes.byref(h))
    _check(st, "lfem_mesh_create")
    return Mesh(h, coords, conn, domain, order, quad)


def lfem_assemble_symbolic(mesh: Mesh, row_begin: int = 0, row_end: Optional[int] = None, stream=None) -> Plan:
    if row_end is None:
        row_end = mesh.n_nodes
    h = ctypes.c_void_p()
    st = _lib().lfem_assemble_symbolic(mesh.handle, row_begin, row_end, _stream(stream), ctypes.byref(h))
    _check(st, "lfem_assemble_symbolic")
    return Plan(h, mesh, row_begin, row_end)


def lfem_plan_info(plan: Plan):
    a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
    _check(_lib().lfem_plan_info(plan.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)), "lfem_plan_info")
    return a.value, b.value, c.value


def lfem_plan_set_variant(plan: Plan, variant: int):
    _check(_lib().lfem_plan_set_variant(plan.handle, variant), "lfem_plan_set_variant")


def _vals_array(vals):
    arr = (ctypes.c_void_p * 3)()
    for k in range(3):
        v = vals[k] if vals is not None else None
        arr[k] = None if v is None else (v.data_ptr() if isinstance(v, torch.Tensor) else v.ctypes.data)
    return arr


def lfem_assemble_numeric(plan: Plan, kinds: int, coeff: Optional[torch.Tensor], vals, stream=None):
    """vals: list of 3 (torch.cuda float64 nnz tensors or None) -> [M, A, A_a]."""
    st = _lib().lfem_assemble_numeric(plan.handle, kinds, _dptr(coeff), _vals_array(vals), _stream(stream))
    _check(st, "lfem_assemble_numeric")


def lfem_assemble_numeric_coords(plan: Plan, kinds: int, coords: torch.Tensor, coeff: Optional[torch.Tensor], vals,
                                 stream=None):
    st = _lib().lfem_assemble_numeric_coords(plan.handle, kinds, _dptr(coords), _dptr(coeff), _vals_array(vals),
                                             _stream(stream))
    _check(st, "lfem_assemble_numeric_coords")


def lfem_assemble_numeric_host(plan: Plan, kinds: int, coords_h, coeff_h, vals_h, stream=None):
    """Host buffers (pinned torch CPU tensors or numpy arrays); synchronises."""
    def hp(a):
        if a is None:
            return None
        return ctypes.c_void_p(a.data_ptr() if isinstance(a, torch.Tensor) else a.ctypes.data)
    st = _lib().lfem_assemble_numeric_host(plan.handle, kinds, hp(coords_h), hp(coeff_h), _vals_array(vals_h),
                                           _stream(stream))
    _check(st, "lfem_assemble_numeric_host")


class _DevView:
    """Zero-copy __cuda_array_interface__ view of a plan-owned device array."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False), "version": 3,
                                         "strides": None}


def lfem_csr_get(plan: Plan):
    """(row_ptr int64 [n_rows+1], col_idx int32 [nnz]) as torch views of PLAN-OWNED memory
    (clone them to keep them past lfem_plan_destroy)."""
    rp, ci = ctypes.c_void_p(), ctypes.c_void_p()
    _check(_lib().lfem_csr_get(plan.handle, ctypes.byref(rp), ctypes.byref(ci)), "lfem_csr_get")
    dev = plan.mesh.coords.device
    row_ptr = torch.as_tensor(_DevView(rp.value, plan.n_rows + 1, "<i8"), device=dev)
    col_idx = torch.as_tensor(_DevView(ci.value or 0, plan.nnz, "<i4"), device=dev) if plan.nnz else \
        torch.empty(0, dtype=torch.int32, device=dev)
    return row_ptr, col_idx


def lfem_spmv(plan: Plan, vals: torch.Tensor, x_full: torch.Tensor, y_rows: torch.Tensor, stream=None):
    _check(_lib().lfem_spmv(plan.handle, _dptr(vals), _dptr(x_full), _dptr(y_rows), _stream(stream)), "lfem_spmv")


def lfem_rhs_ncomp(kind: int) -> int:
    return int(_lib().lfem_rhs_ncomp(kind))


def lfem_rhs_launches(plan: Plan, kind: int) -> int:
    return int(_lib().lfem_rhs_launches(plan.handle, kind))


def lfem_assemble_rhs(plan: Plan, kind: int, coords: Optional[torch.Tensor], u: torch.Tensor, out: torch.Tensor,
                      stream=None):
    """Right-hand side `kind` (LFEM_RHS_LOAD / LFEM_RHS_KLL): u is (ncomp, n_nodes) fp64 on the device,
    out (ncomp, n_rows) fp64 on the device (component-major); coords None = the mesh's."""
    st = _lib().lfem_assemble_rhs(plan.handle, kind, _dptr(coords), _dptr(u), _dptr(out), _stream(stream))
    _check(st, "lfem_assemble_rhs")


def lfem_cg_solve(plan: Plan, vals_K: torch.Tensor, b: torch.Tensor, x: torch.Tensor, tol: float = 1e-12,
                  max_it: int = 10000, stream=None) -> int:
    """K x = b for the three AoS columns of b (n_nodes x 3); x: initial guess in, solution out.
    Returns the iterations used."""
    it = ctypes.c_int(0)
    st = _lib().lfem_cg_solve(plan.handle, _dptr(vals_K), _dptr(b), _dptr(x), tol, max_it, ctypes.byref(it),
                              _stream(stream))
    _check(st, "lfem_cg_solve")
    return it.value


def lfem_solve_meanfree(plan: Plan, vals_A: torch.Tensor, b: torch.Tensor, u: torch.Tensor, tol: float = 1e-12,
                        max_it: int = 20000, stream=None) -> int:
    """Mean-free Poisson for the three AoS columns of b; u (n_nodes x 3) is overwritten."""
    it = ctypes.c_int(0)
    st = _lib().lfem_solve_meanfree(plan.handle, _dptr(vals_A), _dptr(b), _dptr(u), tol, max_it, ctypes.byref(it),
                                    _stream(stream))
    _check(st, "lfem_solve_meanfree")
    return it.value


def lfem_mcf_step(plan: Plan, tau: float, x_prev: torch.Tensor, x_next: torch.Tensor, tol: float = 1e-12,
                  max_it: int = 10000, stream=None) -> int:
    """One step of Dziuk's MCF on the device; returns the CG iterations."""
    it = ctypes.c_int(0)
    st = _lib().lfem_mcf_step(plan.handle, tau, _dptr(x_prev), _dptr(x_next), tol, max_it, ctypes.byref(it),
                              _stream(stream))
    _check(st, "lfem_mcf_step")
    return it.value


def lfem_plan_check(plan: Plan, stream=None):
    _check(_lib().lfem_plan_check(plan.handle, _stream(stream)), "lfem_plan_check")


def lfem_axpby(ca: float, a: torch.Tensor, cb: float, b: torch.Tensor, out: torch.Tensor, stream=None):
    _check(_lib().lfem_axpby(a.numel(), ca, _dptr(a), cb, _dptr(b), _dptr(out), _stream(stream)), "lfem_axpby")


def lfem_numeric_launches(plan: Plan, kinds: int) -> int:
    return int(_lib().lfem_numeric_launches(plan.handle, kinds))


def lfem_numeric_stats(plan: Plan):
    """(element evaluations per numeric call incl. tile halo, row tiles) of the last call."""
    ev, nt = ctypes.c_int64(), ctypes.c_int64()
    _check(_lib().lfem_numeric_stats(plan.handle, ctypes.byref(ev), ctypes.byref(nt)), "lfem_numeric_stats")
    return int(ev.value), int(nt.value)


def lfem_profile_enable(plan: Plan, enable: bool = True):
    _check(_lib().lfem_profile_enable(plan.handle, 1 if enable else 0), "lfem_profile_enable")


def lfem_profile_read(plan: Plan):
    """{kernel name: (total ms, launches)} since the last read (synchronises)."""
    names = (ctypes.c_char_p * 16)()
    ms = (ctypes.c_double * 16)()
    cnt = (ctypes.c_int64 * 16)()
    n = ctypes.c_int()
    _check(_lib().lfem_profile_read(plan.handle, 16, names, ms, cnt, ctypes.byref(n)), "lfem_profile_read")
    return {names[i].decode(): (ms[i], cnt[i]) for i in range(n.value)}


ALLOC_FN = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
FREE_FN = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)
_ALLOC_KEEP = []  # keep the ctypes callbacks alive while installed


def lfem_set_allocator(alloc=None, dealloc=None) -> None:
    """Install Python callables alloc(bytes, stream) -> int device pointer and
    dealloc(ptr, stream) as the library's device allocator (None, None: cudaMalloc)."""
    if alloc is None and dealloc is None:
        _check(_lib().lfem_set_allocator(None, None, None), "lfem_set_allocator")
        _ALLOC_KEEP.clear()
        return
    a = ALLOC_FN(lambda n, s, ctx: alloc(int(n), s) or None)
    f = FREE_FN(lambda p, s, ctx: dealloc(int(p), s))
    _check(_lib().lfem_set_allocator(a, f, None), "lfem_set_allocator")
    _ALLOC_KEEP[:] = [a, f]


def torch_caching_allocator():
    """(alloc, dealloc) pair backed by PyTorch's caching allocator on the current
    device, stream-ordered on the stream the library hands over (the block is
    allocated from, and returned to, that stream's pool)."""
    def alloc(n, stream):
        dev = torch.cuda.current_device()
        return torch.cuda.caching_allocator_alloc(max(int(n), 1), dev, stream or 0)

    def dealloc(p, stream):
        torch.cuda.caching_allocator_delete(int(p))

    return alloc, dealloc


def lfem_version() -> str:
    return _lib().lfem_version().decode()


# ----------------------------------------------------------------------------
# convenience: one call from host arrays to device CSR
# ----------------------------------------------------------------------------
def assemble(mesh_arrays, kinds=("M", "A"), coeff=None, row_begin=0, row_end=None, variant=LFEM_NUMERIC_AUTO,
             device="cuda"):
    """Upload a lfem_inputs.Mesh-like object (coords, conn, domain, order, quad),
    run symbolic + numeric, return (plan, row_ptr, col_idx, {kind: vals})."""
    coords = torch.as_tensor(mesh_arrays.coords, device=device).contiguous()
    conn = torch.as_tensor(mesh_arrays.conn, device=device).contiguous()
    m = lfem_mesh_create(mesh_arrays.domain, mesh_arrays.order, mesh_arrays.quad, coords, conn)
    plan = lfem_assemble_symbolic(m, row_begin, row_end)
    lfem_plan_set_variant(plan, variant)
    km = kinds_mask(kinds)
    vals = [None, None, None]
    for k in kinds:
        vals[KIND_INDEX[k]] = torch.empty(plan.nnz, dtype=torch.float64, device=device)
    cf = None
    if "Aa" in kinds:
        src = coeff if coeff is not None else mesh_arrays.coeff
        cf = torch.as_tensor(src, device=device).contiguous()
    lfem_assemble_numeric(plan, km, cf, vals)
    lfem_plan_check(plan)
    row_ptr, col_idx = lfem_csr_get(plan)
    plan._keep = (coords, conn, cf)
    return plan, row_ptr, col_idx, {k: vals[KIND_INDEX[k]] for k in kinds}


def assemble_rhs(mesh_arrays, u, kind="load", row_begin=0, row_end=None, device="cuda", plan=None,
                 variant=None):
    """Upload a lfem_inputs.Mesh-like object and nodal data u ((ncomp, n_nodes), component-major),
    run symbolic (unless `plan` is given) + the right-hand side; returns (plan, out (ncomp, n_rows))."""
    k = RHS_KINDS[kind] if isinstance(kind, str) else int(kind)
    nc = lfem_rhs_ncomp(k)
    if plan is None:
        coords = torch.as_tensor(mesh_arrays.coords, device=device).contiguous()
        conn = torch.as_tensor(mesh_arrays.conn, device=device).contiguous()
        m = lfem_mesh_create(mesh_arrays.domain, mesh_arrays.order, mesh_arrays.quad, coords, conn)
        plan = lfem_assemble_symbolic(m, row_begin, row_end)
        plan._keep = (coords, conn)
    if variant is not None:
        lfem_plan_set_variant(plan, variant)
    uu = torch.as_tensor(u, dtype=torch.float64, device=device).reshape(nc, -1).contiguous()
    out = torch.empty((nc, plan.n_rows), dtype=torch.float64, device=device)
    lfem_assemble_rhs(plan, k, None, uu, out)
    lfem_plan_check(plan)
    return plan, out
