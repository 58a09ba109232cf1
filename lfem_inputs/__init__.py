"""Seeded synthetic inputs shared by the CUDA path and the CPU oracle.

This module is the ONLY code both sides use.  It builds meshes (node
coordinates + element connectivity) and nodal coefficient fields; it holds
none of the assembly method's arithmetic (no basis functions, no quadrature,
no Jacobians, no sparse accumulation).  Conventions are the readings listed
in DESIGN.md §3:

* RNG: splitmix64, uniforms (x >> 11) * 2^-53, normals by Box-Muller (cos
  branch, two uniforms per normal).                               (G18)
* Icosphere: icosahedron, midpoint subdivision, every new vertex projected to
  the unit sphere after every level; P2 edge node of (a, b) =
  normalize((x_a + x_b)/2); local order 4=(1,2), 5=(2,3), 6=(3,1).  (G15, G26;
  PAPER.md Fig. "notation" P:211-216 for the P2 node order)
* Kuhn cube: 6 tets per cell, (v0, v0+e_p1, v0+e_p1+e_p2, v0+1); for odd
  permutations local vertices 2,3 swapped so det J > 0; P2 edge order
  (1,2),(2,3),(3,1),(1,4),(2,4),(3,4).                               (G17, G26)
* Spherical harmonics: real, orthonormal on S^2, no Condon-Shortley phase,
  coefficients drawn in order l ascending, m = -l..l.               (G13, G14)
* Canonical numbering: nodes sorted by a 3-D Hilbert key of their
  coordinates, elements by the key of their corner centroid, ties by old id.
  (SURVEY.md §8(d).2 "Canonical numbering")

Arrays: coords float64 (n_nodes, 3) C-contiguous (AoS xyz); conn int32
(n_elems, nref) C-contiguous, 0-based (Table 1 P:426-435 is 1-based;
G22).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

# ---------------------------------------------------------------------------
# optional compiled fast path (lfem_inputs/_fast.cpp); bitwise identical to
# the numpy code below (same operation order, no FP contraction)
# ---------------------------------------------------------------------------
import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
_FAST = None


def build_fast(force: bool = False) -> Optional[str]:
    src = os.path.join(_HERE, "_fast.cpp")
    so = os.path.join(_HERE, "_fast.so")
    if force or not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(src):
        cmd = ["g++", "-O2", "-ffp-contract=off", "-fno-fast-math", "-fopenmp", "-shared",
               "-fPIC", "-o", so + ".tmp", src]
        subprocess.run(cmd, check=True)
        os.replace(so + ".tmp", so)
    return so


def _fast():
    global _FAST
    if _FAST is None:
        try:
            lib = ctypes.CDLL(build_fast())
            lib.lfin_hilbert_keys.restype = None
            lib.lfin_sh_field.restype = None
            _FAST = lib
        except Exception:  # no compiler: numpy path (identical results)
            _FAST = False
    return _FAST


def _ptr(a):
    return ctypes.c_void_p(a.ctypes.data)

# ---------------------------------------------------------------------------
# RNG: splitmix64
# ---------------------------------------------------------------------------
_M64 = (1 << 64) - 1


class SplitMix64:
    """Sequential splitmix64 stream (G18).  Deterministic across platforms."""

    def __init__(self, seed: int = 0):
        self.state = seed & _M64

    def next_u64(self, n: int) -> np.ndarray:
        # vectorised: state_k = seed + k*gamma, then the mixing function
        gamma = np.uint64(0x9E3779B97F4A7C15)
        k = np.arange(1, n + 1, dtype=np.uint64)
        with np.errstate(over="ignore"):
            z = np.uint64(self.state) + k * gamma
            z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
            z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
            z = z ^ (z >> np.uint64(31))
        self.state = (self.state + n * 0x9E3779B97F4A7C15) & _M64
        return z

    def uniform(self, n: int) -> np.ndarray:
        """n uniforms in [0, 1): (x >> 11) * 2^-53."""
        return (self.next_u64(n) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)

    def normal(self, n: int) -> np.ndarray:
        """n standard normals, Box-Muller cos branch, uniforms taken pairwise."""
        u = self.uniform(2 * n).reshape(n, 2)
        u1 = 1.0 - u[:, 0]  # (0, 1]: log is finite
        return np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u[:, 1])


# ---------------------------------------------------------------------------
# Mesh container
# ---------------------------------------------------------------------------
SURFACE_TRI = 0
BULK_TET = 1

# quadrature enum values of include/lfem.h (lfem_quad)
QUAD_DEFAULT = 0
QUAD_TRI3_DEG2 = 1
QUAD_TRI6_DEG4 = 2
QUAD_TET4_DEG2 = 3
QUAD_TET11_DEG4 = 4
QUAD_TRI16_DEG8 = 5  # Dunavant degree 8 (the paper's load-vector rule)
QUAD_LINE2_DEG3 = 6  # 2-point Gauss-Legendre (curves)
QUAD_LINE3_DEG5 = 7  # 3-point Gauss-Legendre
QUAD_TET35_DEG7 = 8  # 35-point symmetric degree-7 tet rule (stands in for Jaskowiec-Sukumar degree 7)
QUAD_LINE6_DEG11 = 9  # 6-point Gauss-Legendre (the paper's order-10 Gauss rule for curves)
SURFACE_LINE = 2     # curves in R^3 (Table 4 "surface 1D")


@dataclass
class Mesh:
    domain: int            # SURFACE_TRI | BULK_TET
    order: int             # 1 | 2
    coords: np.ndarray     # (n_nodes, 3) float64
    conn: np.ndarray       # (n_elems, nref) int32
    quad: int = QUAD_DEFAULT
    coeff: Optional[np.ndarray] = None      # (n_nodes,) float64 nodal u
    extra: dict = field(default_factory=dict)

    @property
    def n_nodes(self) -> int:
        return int(self.coords.shape[0])

    @property
    def n_elems(self) -> int:
        return int(self.conn.shape[0])

    @property
    def nref(self) -> int:
        return int(self.conn.shape[1])

    @property
    def n_corners(self) -> int:
        return 3 if self.domain == SURFACE_TRI else 4


def _finish(m: Mesh) -> Mesh:
    m.coords = np.ascontiguousarray(m.coords, dtype=np.float64)
    m.conn = np.ascontiguousarray(m.conn, dtype=np.int32)
    if m.coeff is not None:
        m.coeff = np.ascontiguousarray(m.coeff, dtype=np.float64)
    return m


# ---------------------------------------------------------------------------
# Icosphere (G15)
# ---------------------------------------------------------------------------
def _normalize(x: np.ndarray) -> np.ndarray:
    return x / np.sqrt(np.einsum("ij,ij->i", x, x))[:, None]


def icosahedron():
    p = (1.0 + math.sqrt(5.0)) / 2.0
    v = np.array([
        [-1, p, 0], [1, p, 0], [-1, -p, 0], [1, -p, 0],
        [0, -1, p], [0, 1, p], [0, -1, -p], [0, 1, -p],
        [p, 0, -1], [p, 0, 1], [-p, 0, -1], [-p, 0, 1]], dtype=np.float64)
    f = np.array([
        [0, 11, 5], [0, 5, 1], [0, 1, 7], [0, 7, 10], [0, 10, 11],
        [1, 5, 9], [5, 11, 4], [11, 10, 2], [10, 7, 6], [7, 1, 8],
        [3, 9, 4], [3, 4, 2], [3, 2, 6], [3, 6, 8], [3, 8, 9],
        [4, 9, 5], [2, 4, 11], [6, 2, 10], [8, 6, 7], [9, 8, 1]], dtype=np.int64)
    return _normalize(v), f


def _unique_edges(f: np.ndarray, nv: int):
    """Unique undirected edges of triangles f; returns (edges (ne,2), inv (3m,))
    where inv indexes edges for f[:, (0,1)], f[:, (1,2)], f[:, (2,0)] stacked."""
    e = np.concatenate([f[:, [0, 1]], f[:, [1, 2]], f[:, [2, 0]]], axis=0)
    lo = np.minimum(e[:, 0], e[:, 1])
    hi = np.maximum(e[:, 0], e[:, 1])
    key = lo.astype(np.int64) * nv + hi
    uniq, inv = np.unique(key, return_inverse=True)
    edges = np.stack([uniq // nv, uniq % nv], axis=1)
    return edges, inv.reshape(-1)


def icosphere_p1(level: int):
    """Natural-order icosphere: vertices of level l keep their ids at level l+1."""
    v, f = icosahedron()
    for _ in range(level):
        nv = v.shape[0]
        m = f.shape[0]
        edges, inv = _unique_edges(f, nv)
        mid = _normalize(0.5 * (v[edges[:, 0]] + v[edges[:, 1]]))
        v = np.concatenate([v, mid], axis=0)
        m01 = nv + inv[0:m]
        m12 = nv + inv[m:2 * m]
        m20 = nv + inv[2 * m:3 * m]
        f = np.concatenate([
            np.stack([f[:, 0], m01, m20], 1),
            np.stack([f[:, 1], m12, m01], 1),
            np.stack([f[:, 2], m20, m12], 1),
            np.stack([m01, m12, m20], 1)], axis=0)
    return v, f


def p2_from_p1_triangles(v: np.ndarray, f: np.ndarray, project_sphere: bool):
    """Insert one node per unique edge; local order 4=(1,2),5=(2,3),6=(3,1)."""
    nv = v.shape[0]
    m = f.shape[0]
    edges, inv = _unique_edges(f, nv)
    mid = 0.5 * (v[edges[:, 0]] + v[edges[:, 1]])
    if project_sphere:
        mid = _normalize(mid)
    nodes = np.concatenate([v, mid], axis=0)
    conn = np.concatenate([f, np.stack([nv + inv[0:m], nv + inv[m:2 * m],
                                        nv + inv[2 * m:3 * m]], 1)], axis=1)
    return nodes, conn


# ---------------------------------------------------------------------------
# Kuhn cube (G16, G17)
# ---------------------------------------------------------------------------
_PERMS = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]


def _perm_sign(p):
    s = 1
    p = list(p)
    for i in range(3):
        for j in range(i + 1, 3):
            if p[i] > p[j]:
                s = -s
    return s


def kuhn_cube(n: int, order: int):
    """Unit cube, n^3 cells, 6 tets each.  P1 nodes: (n+1)^3 grid; P2 nodes:
    the full (2n+1)^3 half grid.  Returns (coords, conn) in natural order
    (x fastest).  Tets have positive orientation."""
    s = order  # grid refinement of the node lattice
    g = s * n + 1
    ii, jj, kk = np.meshgrid(np.arange(g), np.arange(g), np.arange(g), indexing="ij")
    # node id = i + g*(j + g*k)
    coords = np.stack([ii.transpose(2, 1, 0).ravel(), jj.transpose(2, 1, 0).ravel(),
                       kk.transpose(2, 1, 0).ravel()], 1).astype(np.float64) / (s * n)

    def nid(i, j, k):
        return i + g * (j + g * k)

    cx, cy, cz = np.meshgrid(np.arange(n), np.arange(n), np.arange(n), indexing="ij")
    cx = cx.transpose(2, 1, 0).ravel()
    cy = cy.transpose(2, 1, 0).ravel()
    cz = cz.transpose(2, 1, 0).ravel()
    base = np.stack([cx, cy, cz], 1) * s  # lattice coords of v0
    tets = []
    unit = np.eye(3, dtype=np.int64) * s
    for p in _PERMS:
        v0 = base
        v1 = v0 + unit[p[0]]
        v2 = v1 + unit[p[1]]
        v3 = v0 + s
        vs = [v0, v1, v2, v3]
        if _perm_sign(p) < 0:
            vs = [v0, v2, v1, v3]
        tets.append(vs)
    # interleave so that the 6 tets of a cell are consecutive
    elems = []
    for c in range(6):
        vs = tets[c]
        cols = [nid(v[:, 0], v[:, 1], v[:, 2]) for v in vs]
        if order == 2:
            pairs = [(0, 1), (1, 2), (2, 0), (0, 3), (1, 3), (2, 3)]
            for a, b in pairs:
                mv = (vs[a] + vs[b]) // 2
                cols.append(nid(mv[:, 0], mv[:, 1], mv[:, 2]))
        elems.append(np.stack(cols, 1))
    conn = np.stack(elems, 1).reshape(-1, 4 if order == 1 else 10)
    return coords, conn


# ---------------------------------------------------------------------------
# Real spherical harmonics (G14)
# ---------------------------------------------------------------------------
def real_sh(xyz: np.ndarray, lmax: int = 4) -> np.ndarray:
    """Real orthonormal spherical harmonics on S^2 at unit vectors xyz.
    Columns ordered l ascending, m = -l..l.  No Condon-Shortley phase.
    Y_l0 = N_l0 P_l(z); Y_lm = sqrt2 N_lm P_l^m(z) cos(m phi) (m>0),
    Y_l,-m = sqrt2 N_lm P_l^m(z) sin(m phi), with P_l^m(z) = (1-z^2)^{m/2} Q_l^m(z)
    and (x+iy)^m = (sin th)^m e^{i m phi}."""
    x, y, z = xyz[:, 0], xyz[:, 1], xyz[:, 2]
    n = xyz.shape[0]
    out = np.zeros((n, (lmax + 1) ** 2))
    # powers (x + i y)^m
    cm = [np.ones(n)]
    sm = [np.zeros(n)]
    for m in range(1, lmax + 1):
        c, s_ = cm[-1], sm[-1]
        cm.append(c * x - s_ * y)
        sm.append(c * y + s_ * x)
    for m in range(0, lmax + 1):
        # Q_m^m = (2m-1)!!, Q_{m+1}^m = z (2m+1) Q_m^m, Q_l^m recursion
        dfact = 1.0
        for k in range(1, 2 * m, 2):
            dfact *= k
        q_prev2 = None
        q_prev = np.full(n, dfact)
        for l in range(m, lmax + 1):
            if l == m:
                q = q_prev
            elif l == m + 1:
                q = z * (2 * m + 1) * q_prev
                q_prev2, q_prev = q_prev, q
            else:
                q = ((2 * l - 1) * z * q_prev - (l + m - 1) * q_prev2) / (l - m)
                q_prev2, q_prev = q_prev, q
            norm = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
            if m == 0:
                out[:, l * l + l] = norm * q
            else:
                out[:, l * l + l + m] = math.sqrt(2.0) * norm * q * cm[m]
                out[:, l * l + l - m] = math.sqrt(2.0) * norm * q * sm[m]
    return out


def _sh_norms(lmax: int) -> np.ndarray:
    nrm = np.zeros((lmax + 1) ** 2)
    for l in range(lmax + 1):
        for m in range(0, l + 1):
            v = math.sqrt((2 * l + 1) / (4 * math.pi) * math.factorial(l - m) / math.factorial(l + m))
            if m == 0:
                nrm[l * l + l] = v
            else:
                nrm[l * l + l + m] = math.sqrt(2.0) * v
                nrm[l * l + l - m] = math.sqrt(2.0) * v
    return nrm


def sh_field(xyz: np.ndarray, coef: np.ndarray, normalize: bool = True, lmax: int = 4,
             use_fast: bool = True) -> np.ndarray:
    """u(x) = sum_lm coef_lm Y_lm(x/|x|), accumulated m-major then l (same
    order in the compiled and numpy paths, so the values are identical)."""
    xyz = np.ascontiguousarray(xyz, dtype=np.float64)
    coef = np.ascontiguousarray(coef, dtype=np.float64)
    norms = _sh_norms(lmax)
    lib = _fast() if use_fast else False
    if lib:
        out = np.empty(xyz.shape[0])
        lib.lfin_sh_field(ctypes.c_int64(xyz.shape[0]), _ptr(xyz), ctypes.c_int(lmax), _ptr(coef),
                          _ptr(norms), ctypes.c_int(1 if normalize else 0), _ptr(out))
        return out
    x, y, z = xyz[:, 0].copy(), xyz[:, 1].copy(), xyz[:, 2].copy()
    if normalize:
        r = np.sqrt(x * x + y * y + z * z)
        x, y, z = x / r, y / r, z / r
    n = xyz.shape[0]
    cm = [np.ones(n)]
    sm = [np.zeros(n)]
    for m in range(1, lmax + 1):
        cm.append(cm[-1] * x - sm[-1] * y)
        sm.append(cm[-2] * y + sm[-1] * x)
    acc = np.zeros(n)
    for m in range(0, lmax + 1):
        dfact = 1.0
        for k in range(1, 2 * m, 2):
            dfact *= k
        qp2 = np.zeros(n)
        qp = np.full(n, dfact)
        for l in range(m, lmax + 1):
            if l == m:
                q = qp
            elif l == m + 1:
                q = z * float(2 * m + 1) * qp
                qp2, qp = qp, q
            else:
                q = (float(2 * l - 1) * z * qp - float(l + m - 1) * qp2) / float(l - m)
                qp2, qp = qp, q
            if m == 0:
                acc = acc + coef[l * l + l] * (norms[l * l + l] * q)
            else:
                acc = acc + coef[l * l + l + m] * (norms[l * l + l + m] * q * cm[m])
                acc = acc + coef[l * l + l - m] * (norms[l * l + l - m] * q * sm[m])
    return acc


def sh_coefficients(rng: SplitMix64, lmax: int = 4) -> np.ndarray:
    """c_lm ~ N(0,1)/(1+l^2), order l asc, m=-l..l (G13)."""
    z = rng.normal((lmax + 1) ** 2)
    ls = np.concatenate([[l] * (2 * l + 1) for l in range(lmax + 1)])
    return z / (1.0 + ls.astype(np.float64) ** 2)


# ---------------------------------------------------------------------------
# Hilbert ordering
# ---------------------------------------------------------------------------
_HBITS = 16


def _part1by2(x: np.ndarray) -> np.ndarray:
    x = x.astype(np.uint64) & np.uint64(0x1FFFFF)
    x = (x | (x << np.uint64(32))) & np.uint64(0x1F00000000FFFF)
    x = (x | (x << np.uint64(16))) & np.uint64(0x1F0000FF0000FF)
    x = (x | (x << np.uint64(8))) & np.uint64(0x100F00F00F00F00F)
    x = (x | (x << np.uint64(4))) & np.uint64(0x10C30C30C30C30C3)
    x = (x | (x << np.uint64(2))) & np.uint64(0x1249249249249249)
    return x


def hilbert_keys(pts: np.ndarray, lo: np.ndarray, hi: np.ndarray, bits: int = _HBITS,
                 use_fast: bool = True) -> np.ndarray:
    """3-D Hilbert index of points quantised to `bits` bits per axis over the
    box [lo, hi] (compiled path if available, else numpy; identical keys)."""
    lib = _fast() if use_fast else False
    if lib:
        pts = np.ascontiguousarray(pts, dtype=np.float64)
        lo = np.ascontiguousarray(lo, dtype=np.float64)
        hi = np.ascontiguousarray(hi, dtype=np.float64)
        keys = np.empty(pts.shape[0], dtype=np.uint64)
        lib.lfin_hilbert_keys(ctypes.c_int64(pts.shape[0]), _ptr(pts), _ptr(lo), _ptr(hi),
                              ctypes.c_int(bits), _ptr(keys))
        return keys
    return hilbert_keys_np(pts, lo, hi, bits)


def hilbert_keys_np(pts: np.ndarray, lo: np.ndarray, hi: np.ndarray, bits: int = _HBITS) -> np.ndarray:
    """3-D Hilbert index (Skilling's transpose algorithm) of points quantised
    to `bits` bits per axis over the box [lo, hi]."""
    span = np.where(hi > lo, hi - lo, 1.0)
    q = np.floor((pts - lo) / span * ((1 << bits) - 1) + 0.5)
    X = [np.clip(q[:, i], 0, (1 << bits) - 1).astype(np.uint32) for i in range(3)]
    M = np.uint32(1 << (bits - 1))
    Q = M
    while Q > 1:
        P = np.uint32(Q - 1)
        for i in range(3):
            mask = (X[i] & Q) != 0
            X[0] = np.where(mask, X[0] ^ P, X[0])
            t = np.where(mask, np.uint32(0), (X[0] ^ X[i]) & P)
            X[0] = X[0] ^ t
            X[i] = X[i] ^ t
        Q = np.uint32(Q >> 1)
    X[1] = X[1] ^ X[0]
    X[2] = X[2] ^ X[1]
    t = np.zeros_like(X[0])
    Q = M
    while Q > 1:
        t = np.where((X[2] & Q) != 0, t ^ np.uint32(Q - 1), t)
        Q = np.uint32(Q >> 1)
    X = [xi ^ t for xi in X]
    # interleave: bit b of X0 is the most significant of each triple
    return (_part1by2(X[0]) << np.uint64(2)) | (_part1by2(X[1]) << np.uint64(1)) | _part1by2(X[2])


def sfc_reorder(coords: np.ndarray, conn: np.ndarray, n_corners: int, coeffs=()):
    """Renumber nodes by Hilbert key of coordinates and elements by the key
    of their corner centroid (stable: ties by old id)."""
    lo = coords.min(axis=0)
    hi = coords.max(axis=0)
    nkey = hilbert_keys(coords, lo, hi)
    norder = np.argsort(nkey, kind="stable")
    newid = np.empty_like(norder)
    newid[norder] = np.arange(norder.size)
    cent = coords[conn[:, :n_corners]].mean(axis=1)
    ekey = hilbert_keys(cent, lo, hi)
    eorder = np.argsort(ekey, kind="stable")
    new_conn = newid[conn[eorder]]
    out = [coords[norder], new_conn]
    out.extend(c[norder] for c in coeffs)
    return out


# ---------------------------------------------------------------------------
# Tiny fixtures
# ---------------------------------------------------------------------------
def table12_mesh() -> Mesh:
    """PAPER.md Tables 1-2, 2-element P2 half-disk, embedded at
    z = 0 as a flat P2 surface.  Reading G5: node 6 = (-sqrt2/2, sqrt2/2),
    node 9 = (+sqrt2/2, sqrt2/2); 0-based (G22)."""
    r = math.sqrt(2.0) / 2.0
    nodes = np.array([[-1, 0, 0], [0, 0, 0], [0, 1, 0], [-0.5, 0, 0], [0, 0.5, 0],
                      [-r, r, 0], [1, 0, 0], [0.5, 0, 0], [r, r, 0]], dtype=np.float64)
    elems = np.array([[1, 2, 3, 4, 5, 6], [2, 7, 3, 8, 9, 5]], dtype=np.int32) - 1
    return _finish(Mesh(SURFACE_TRI, 2, nodes, elems, QUAD_TRI6_DEG4))


def single_triangle(p, order: int = 1) -> Mesh:
    p = np.asarray(p, dtype=np.float64).reshape(3, 3)
    f = np.array([[0, 1, 2]])
    if order == 1:
        return _finish(Mesh(SURFACE_TRI, 1, p, f, QUAD_TRI3_DEG2))
    nodes, conn = p2_from_p1_triangles(p, f, project_sphere=False)
    return _finish(Mesh(SURFACE_TRI, 2, nodes, conn, QUAD_TRI6_DEG4))


def sphere_mesh(level: int, order: int, sfc: bool = True) -> Mesh:
    v, f = icosphere_p1(level)
    if order == 2:
        v, f = p2_from_p1_triangles(v, f, project_sphere=True)
    if sfc:
        v, f = sfc_reorder(v, f, 3)
    return _finish(Mesh(SURFACE_TRI, order, v, f,
                        QUAD_TRI3_DEG2 if order == 1 else QUAD_TRI6_DEG4))


def cube_mesh(n: int, order: int, sfc: bool = True, displace_seed: Optional[int] = None) -> Mesh:
    x, t = kuhn_cube(n, order)
    if displace_seed is not None:
        x = displace_cube(x, SplitMix64(displace_seed))
    if sfc:
        x, t = sfc_reorder(x, t, 4)
    return _finish(Mesh(BULK_TET, order, x, t,
                        QUAD_TET4_DEG2 if order == 1 else QUAD_TET11_DEG4))


def displace_cube(x: np.ndarray, rng: SplitMix64) -> np.ndarray:
    """G16: x <- x + sum_i 0.05 sin(2 pi x_i) v_i, three seeded unit vectors."""
    v = rng.normal(9).reshape(3, 3)
    v = v / np.linalg.norm(v, axis=1)[:, None]
    d = np.zeros_like(x)
    for i in range(3):
        d += 0.05 * np.sin(2.0 * math.pi * x[:, i])[:, None] * v[i][None, :]
    return x + d


# ---------------------------------------------------------------------------
# BASELINE.json configs
# ---------------------------------------------------------------------------
CONFIG_NAMES = ("C1", "C2", "C3", "C4", "C5")  # BASELINE.json; "C4P1" = N2's P1 tets at scale


def make_config(name: str, seed: int = 0, level_override: Optional[int] = None, natural: bool = False) -> Mesh:
    """Build BASELINE.json configs[i] (C1..C5) as a Mesh.  `level_override`
    builds the same recipe at a smaller size (tests only).  `natural` keeps C2 in the
    generator's own node / element numbering (the SURVEY §8(d).2 sensitivity point)
    instead of the space-filling-curve order."""
    rng = SplitMix64(seed)
    if name == "C1":
        L = 3 if level_override is None else level_override
        v, f = icosphere_p1(L)
        u = rng.uniform(v.shape[0])
        v = v * (1.0 + 1e-3 * (2.0 * u - 1.0))[:, None]
        v, f = sfc_reorder(v, f, 3)
        m = Mesh(SURFACE_TRI, 1, v, f, QUAD_TRI3_DEG2)
        m.extra["kinds"] = ("M", "A")
    elif name == "C2":
        L = 7 if level_override is None else level_override
        v, f = icosphere_p1(L)
        v, f = p2_from_p1_triangles(v, f, project_sphere=True)
        if not natural:
            v, f = sfc_reorder(v, f, 3)
        m = Mesh(SURFACE_TRI, 2, v, f, QUAD_TRI6_DEG4)
        m.extra["kinds"] = ("M", "A")
    elif name == "C3":
        L = 9 if level_override is None else level_override
        xh, f = icosphere_p1(L)
        c = sh_coefficients(rng)
        dA = sh_coefficients(rng)
        dB = sh_coefficients(rng)
        r = 1.0 + 0.2 * sh_field(xh, c)
        if r.min() <= 0.5:
            raise ValueError("C3 radius field min r <= 0.5 (SURVEY §8(d).2 guard)")
        v = xh * r[:, None]
        uA = sh_field(xh, dA)
        uB = sh_field(xh, dB)
        v, f, uA, uB = sfc_reorder(v, f, 3, coeffs=(uA, uB))
        m = Mesh(SURFACE_TRI, 1, v, f, QUAD_TRI3_DEG2, coeff=uA)
        m.extra.update(kinds=("M", "Aa"), uA=np.ascontiguousarray(uA),
                       uB=np.ascontiguousarray(uB), reps=100)
    elif name == "C4":
        n = 96 if level_override is None else level_override
        x, t = kuhn_cube(n, 2)
        x = displace_cube(x, rng)
        x, t = sfc_reorder(x, t, 4)
        m = Mesh(BULK_TET, 2, x, t, QUAD_TET11_DEG4)
        m.extra["kinds"] = ("M", "A")
    elif name == "C4P1":
        # SURVEY §8(f) N2 "P1 tets at scale": the C4 recipe with P1 tetrahedra (TET4_DEG2)
        n = 96 if level_override is None else level_override
        x, t = kuhn_cube(n, 1)
        x = displace_cube(x, rng)
        x, t = sfc_reorder(x, t, 4)
        m = Mesh(BULK_TET, 1, x, t, QUAD_TET4_DEG2)
        m.extra["kinds"] = ("M", "A")
    elif name == "CURVE2":
        # SURVEY §8(f) N2 curves at scale: the P2 unit circle with 2^23 elements (16.8M nodes)
        n = (1 << 23) if level_override is None else level_override
        m = circle_mesh(n, 2)
        m.extra["kinds"] = ("M", "A")
    elif name == "C5":
        L = 10 if level_override is None else level_override
        v, f = icosphere_p1(L)
        v, f = p2_from_p1_triangles(v, f, project_sphere=True)
        d = sh_coefficients(rng)
        u = sh_field(v, d)
        v, f, u = sfc_reorder(v, f, 3, coeffs=(u,))
        m = Mesh(SURFACE_TRI, 2, v, f, QUAD_TRI6_DEG4, coeff=u)
        m.extra["kinds"] = ("M", "A", "Aa")
    else:
        raise ValueError(f"unknown config {name!r}")
    m.extra["name"] = name
    return _finish(m)


def coeff_at_rep(m: Mesh, t: int, reps: int = 100) -> np.ndarray:
    """C3 coefficient at repetition t (G12): cos(2 pi t/reps) uA + sin(2 pi t/reps) uB."""
    th = 2.0 * math.pi * t / reps
    return math.cos(th) * m.extra["uA"] + math.sin(th) * m.extra["uB"]


def random_field(m: Mesh, seed: int) -> np.ndarray:
    """Seeded smooth-ish nodal field for small tests (uniform in [-1,1])."""
    return 2.0 * SplitMix64(seed).uniform(m.n_nodes) - 1.0


def perturb(m: Mesh, seed: int, eps: float) -> Mesh:
    """Copy of m with every node moved by eps*U(-1,1)^3 (test meshes)."""
    u = SplitMix64(seed).uniform(3 * m.n_nodes).reshape(-1, 3)
    c = m.coords + eps * (2.0 * u - 1.0)
    return _finish(Mesh(m.domain, m.order, c, m.conn.copy(), m.quad,
                        None if m.coeff is None else m.coeff.copy()))


def dziuk_surface(level: int, order: int = 2, sfc: bool = True) -> Mesh:
    """PAPER.md P:842 (Dziuk's MCF example): the sphere's nodes mapped by
    x -> (1 + 0.5 sin(2 pi (x + y)) cos(0.25 z pi)) x."""
    m = sphere_mesh(level, order, sfc=sfc)
    x = m.coords
    s = 1.0 + 0.5 * np.sin(2.0 * math.pi * (x[:, 0] + x[:, 1])) * np.cos(0.25 * x[:, 2] * math.pi)
    return _finish(Mesh(m.domain, m.order, s[:, None] * x, m.conn, m.quad))


def circle_mesh(n: int, order: int = 1, radius: float = 1.0) -> Mesh:
    """Unit circle in the z = 0 plane: n vertices, n line elements; P2 inserts each
    element's midpoint node projected to the circle (nodes: vertices first)."""
    t = 2.0 * math.pi * np.arange(n) / n
    v = radius * np.stack([np.cos(t), np.sin(t), np.zeros(n)], axis=1)
    e = np.stack([np.arange(n), (np.arange(n) + 1) % n], axis=1).astype(np.int32)
    if order == 1:
        return _finish(Mesh(SURFACE_LINE, 1, v, e, QUAD_LINE2_DEG3))
    tm = t + math.pi / n
    mid = radius * np.stack([np.cos(tm), np.sin(tm), np.zeros(n)], axis=1)
    conn = np.concatenate([e, (n + np.arange(n))[:, None]], axis=1).astype(np.int32)
    return _finish(Mesh(SURFACE_LINE, 2, np.vstack([v, mid]), conn, QUAD_LINE3_DEG5))
