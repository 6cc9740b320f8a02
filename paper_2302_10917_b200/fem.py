"""Reference-element tables for the device assembly of the 2-D HDG blocks.

Host side of SURVEY.md 8(f) row 2 (real HDG block assembly on the GPU): the
small constant tables the per-macro kernel (csrc/assembly.cu) needs -- basis
values / gradients / Hessians at the quadrature points, the C0 patch dof map,
the face trace tables -- plus the problem data evaluated at the quadrature
points (the data are Python callables, as in the reference).  Everything that
scales with the number of macros runs on the device.

Restates mehdg/fem_basis.py (Lagrange bases by inverting the monomial
Vandermonde matrix on the equispaced lattice, Duffy-collapsed Gauss rules,
patch dof maps, piecewise trace bases) and the quadrature / projection helpers
of mehdg/assembly.py, following the same formulas so the tables agree with the
reference's to rounding.
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache

import numpy as np

EDGE_VERTS = ((1, 2), (2, 0), (0, 1))  # local edge k is opposite vertex k (mesh.py:68)


def simplex_lattice(d: int, p: int) -> list:
    """fem_basis.py:30-37: lattice multi-indices in the reference order."""
    if d == 1:
        return [(i,) for i in range(p + 1)]
    if d == 2:
        return [(i, j) for j in range(p + 1) for i in range(p + 1 - j)]
    raise ValueError("d must be 1 or 2")


class Lagrange:
    """fem_basis.py:40-125: nodal basis = monomials @ inv(Vandermonde)."""

    def __init__(self, d: int, p: int):
        self.d, self.p = d, p
        self.exps = np.array(simplex_lattice(d, p))
        self.n = len(self.exps)
        nodes = self.exps.astype(float) / p
        self.coeff = np.linalg.inv(self._mono(nodes))

    def _mono(self, x, deriv=()):
        """Monomials (or their derivatives along the axes listed in deriv)."""
        x = np.atleast_2d(x)
        out = np.ones((x.shape[0], self.n))
        for c in range(self.d):
            e = self.exps[:, c].astype(float)
            order = deriv.count(c)
            fac = np.ones_like(e)
            for k in range(order):
                fac *= np.maximum(e - k, 0.0)
            out *= fac[None, :] * x[:, c, None] ** np.maximum(self.exps[None, :, c] - order, 0)
        return out

    def eval(self, x):
        return self._mono(x) @ self.coeff

    def grad(self, x):
        x = np.atleast_2d(x)
        return np.stack([self._mono(x, (c,)) @ self.coeff for c in range(self.d)], axis=2)

    def hess(self, x):
        x = np.atleast_2d(x)
        out = np.empty((x.shape[0], self.n, self.d, self.d))
        for a in range(self.d):
            for b in range(a, self.d):
                tab = self._mono(x, (a, b)) @ self.coeff
                out[:, :, a, b] = tab
                out[:, :, b, a] = tab
        return out


def _gauss01(n: int):
    x, w = np.polynomial.legendre.leggauss(n)
    return 0.5 * (x + 1.0), 0.5 * w


def triangle_rule(degree: int):
    """fem_basis.py:183-215 (d = 2): (points_ref (n, 2), weights)."""
    if degree <= 1:
        return np.array([[1.0 / 3.0, 1.0 / 3.0]]), np.array([0.5])
    n = (degree + 3) // 2 + 1
    x, wx = _gauss01(n)
    e, we = _gauss01(n)
    X, E = np.meshgrid(x, e, indexing="ij")
    WX, WE = np.meshgrid(wx, we, indexing="ij")
    px = (X * (1.0 - E)).ravel()
    py = E.ravel()
    w = (WX * WE * (1.0 - E)).ravel()
    return np.column_stack((px, py)), w


def sub_cells(m: int):
    """mesh.py:71-77: red-pattern sub-triangles in the reference order."""
    for j in range(m):
        for i in range(m - j):
            yield ("up", i, j)
            if i + j <= m - 2:
                yield ("down", i, j)


@lru_cache(maxsize=None)
def patch_dof_map(m: int, p: int):
    """fem_basis.py:140-170: (cell kinds, cell (i, j), cell maps, edge nodes)."""
    L = m * p
    index = {ab: i for i, ab in enumerate(simplex_lattice(2, L))}
    loc = simplex_lattice(2, p)
    kinds, ij, maps = [], [], []
    for kind, i, j in sub_cells(m):
        arr = []
        for r, s in loc:
            ab = (i * p + r, j * p + s) if kind == "up" else ((i + 1) * p - s, j * p + r + s)
            arr.append(index[ab])
        kinds.append(0 if kind == "up" else 1)
        ij.append((i, j))
        maps.append(arr)
    edge = np.empty((3, L + 1), dtype=np.int64)
    for k in range(L + 1):
        edge[0, k] = index[(L - k, k)]
        edge[1, k] = index[(0, L - k)]
        edge[2, k] = index[(k, 0)]
    return (np.array(kinds, np.int32), np.array(ij, np.int32), np.array(maps, np.int32),
            edge.astype(np.int32), len(index))


def trace_eval(m_f: int, p: int, s):
    """fem_basis.py:228-250: C0 piecewise degree-p basis on [0, 1], m_f segments."""
    s = np.atleast_1d(np.asarray(s, dtype=float))
    out = np.zeros((s.size, m_f * p + 1))
    seg = np.clip(np.floor(s * m_f).astype(int), 0, m_f - 1)
    vals = Lagrange(1, p).eval((s * m_f - seg)[:, None])
    for r in range(p + 1):
        out[np.arange(s.size), seg * p + r] = vals[:, r]
    return out


def piecewise_quad(breaks, npts: int):
    """assembly.py:120-130: Gauss points subordinate to the breakpoints."""
    x, w = _gauss01(npts)
    pts, wts = [], []
    for lo, hi in zip(breaks[:-1], breaks[1:]):
        if hi - lo < 1e-14:
            continue
        pts.append(lo + (hi - lo) * x)
        wts.append((hi - lo) * w)
    return np.concatenate(pts), np.concatenate(wts)


JSUB = (np.array([[1.0, 0.0], [0.0, 1.0]]), np.array([[0.0, -1.0], [1.0, 1.0]]))  # up, down


# side orientations of a face on a macro edge: (t0, t1) of FaceSide (mesh.py:130-135);
# the last four are the coarse side of a 2:1 hanging face (mesh.py:264-302)
SIDE_VARIANTS = ((0.0, 1.0), (1.0, 0.0), (0.0, 0.5), (0.5, 0.0), (0.5, 1.0), (1.0, 0.5))


@dataclass
class AsmTables:
    m: int
    p: int
    Q: int
    nb: int
    t: int
    qp: np.ndarray     # (nq, 2) reference points
    qw: np.ndarray     # (nq,)
    val: np.ndarray    # (nq, nb)
    gref: np.ndarray   # (nq, nb, 2)
    href: np.ndarray   # (nq, nb, 2, 2)
    cell_kind: np.ndarray
    cell_ij: np.ndarray
    cell_map: np.ndarray   # (ncell, nb)
    edge_nodes: np.ndarray  # (3, t)
    fw: np.ndarray     # (nvar, nfq) assemble_macro's face rule per side variant (zero padded)
    th: np.ndarray     # (nvar, nfq, t) macro-edge trace basis at t0 + (t1 - t0) s
    ps: np.ndarray     # (nvar, nfq, t) face trace basis at s
    ffw: np.ndarray    # (nffq,) face-block quadrature (assemble_face)
    fps: np.ndarray    # (nffq, t)

    @property
    def fs(self):  # conforming forward side: the rule's parameters (tests)
        return self._fs

    @property
    def th_fwd(self):
        return self.th[0, :self._nfq0]


def face_rule(m_f: int, m: int, p: int, t0: float, t1: float):
    """assemble_macro's quadrature on one face side (assembly.py:134-143, 292):
    breakpoints of the face's trace subdivision united with the macro-edge
    subdivision mapped to the face parameter, the latter rounded to 12 digits
    (so for m = 3, 5, ... the set also holds a sliver segment, kept as in the
    reference)."""
    breaks = set(np.arange(m_f + 1) / m_f)
    dt = t1 - t0
    for c in range(m + 1):
        sc = (c / m - t0) / dt
        if 1e-12 < sc < 1 - 1e-12:
            breaks.add(round(sc, 12))
    return piecewise_quad(np.array(sorted(breaks)), p + 1)


@lru_cache(maxsize=None)
def asm_tables(m: int, p: int, quad_degree: int) -> AsmTables:
    """Constant tables of assemble_macro / assemble_face (assembly.py:176-322) for a
    structured mesh of one subdivision m (m_f = m on every face)."""
    qp, qw = triangle_rule(quad_degree)
    basis = Lagrange(2, p)
    kinds, ij, maps, edge, Q = patch_dof_map(m, p)
    t = m * p + 1
    rules = [face_rule(m, m, p, t0, t1) for t0, t1 in SIDE_VARIANTS]
    nfq = max(s.size for s, _ in rules)
    fw = np.zeros((len(rules), nfq))
    th = np.zeros((len(rules), nfq, t))
    ps = np.zeros((len(rules), nfq, t))
    for v, ((s, w), (t0, t1)) in enumerate(zip(rules, SIDE_VARIANTS)):
        fw[v, :s.size] = w
        th[v, :s.size] = trace_eval(m, p, t0 + (t1 - t0) * s)
        ps[v, :s.size] = trace_eval(m, p, s)
    ffs, ffw = piecewise_quad(np.arange(m + 1) / m, p + 1)  # assemble_face (assembly.py:302)
    tab = AsmTables(m=m, p=p, Q=Q, nb=basis.n, t=t, qp=qp, qw=qw,
                    val=basis.eval(qp), gref=basis.grad(qp), href=basis.hess(qp),
                    cell_kind=kinds, cell_ij=ij, cell_map=maps, edge_nodes=edge,
                    fw=fw, th=th, ps=ps, ffw=ffw, fps=trace_eval(m, p, ffs))
    tab._fs, tab._nfq0 = rules[0][0], rules[0][0].size
    return tab


def side_variant(t0, t1):
    """Index into SIDE_VARIANTS of FaceSide parameters (t0, t1); arrays accepted."""
    t0, t1 = np.asarray(t0, float), np.asarray(t1, float)
    out = np.full(t0.shape, -1, np.int64)
    for v, (a, b) in enumerate(SIDE_VARIANTS):
        out[(np.abs(t0 - a) < 1e-12) & (np.abs(t1 - b) < 1e-12)] = v
    if (out < 0).any():
        raise NotImplementedError("face side parameters are not a conforming or 2:1 hanging "
                                  "configuration")
    return int(out) if out.ndim == 0 else out


def macro_geometry(mesh) -> np.ndarray:
    """(N, 3, 2) physical vertex coordinates of every macro."""
    if hasattr(mesh, "elem_verts"):
        return mesh.vertices[mesh.elem_verts]
    return np.stack([np.asarray(e.verts, float) for e in mesh.macro_elements])


def quad_points(verts: np.ndarray, tab: AsmTables) -> np.ndarray:
    """(N, ncell, nq, 2) physical quadrature points of every sub-cell
    (assembly.py:218-222: pts = points_ref @ Jc^T + v0 of the sub-cell)."""
    m = tab.m
    J = np.stack((verts[:, 1] - verts[:, 0], verts[:, 2] - verts[:, 0]), axis=2)  # (N,2,2)
    out = np.empty((verts.shape[0], len(tab.cell_kind), tab.qp.shape[0], 2))
    for c, (kind, (i, j)) in enumerate(zip(tab.cell_kind, tab.cell_ij)):
        h = 1.0 / m
        v0ref = np.array([i * h, j * h]) if kind == 0 else np.array([(i + 1) * h, j * h])
        Jc = J @ (JSUB[kind] / m)
        v0 = verts[:, 0] + J @ v0ref
        out[:, c] = np.swapaxes(Jc @ tab.qp.T, 1, 2) + v0[:, None, :]
    return out


def dirichlet_projection(face_verts: np.ndarray, g, p: int, m_f: int) -> np.ndarray:
    """assembly.py:153-165 for many faces at once: L2 projection of g onto the
    face trace space; face_verts (nD, 2, 2) canonical endpoints."""
    psi_breaks = np.arange(m_f + 1) / m_f
    s, w = piecewise_quad(psi_breaks, max(p + 2, 6))
    V = trace_eval(m_f, p, s)
    M = V.T @ (w[:, None] * V)
    x = face_verts[:, None, 0, :] + s[None, :, None] * (face_verts[:, 1] - face_verts[:, 0])[:, None]
    G = np.asarray(g(x.reshape(-1, 2)), dtype=float).reshape(x.shape[0], s.size)
    r = (G * w[None, :]) @ V
    return np.linalg.solve(M, r.T).T


def neumann_rhs(face_verts: np.ndarray, g, p: int, m_f: int) -> np.ndarray:
    """assembly.py:313-321: R_hat of Neumann faces."""
    s, w = piecewise_quad(np.arange(m_f + 1) / m_f, max(p + 2, 6))
    V = trace_eval(m_f, p, s)
    length = np.linalg.norm(face_verts[:, 1] - face_verts[:, 0], axis=1)
    x = face_verts[:, None, 0, :] + s[None, :, None] * (face_verts[:, 1] - face_verts[:, 0])[:, None]
    G = np.asarray(g(x.reshape(-1, 2)), dtype=float).reshape(x.shape[0], s.size)
    return ((G * w[None, :]) * length[:, None]) @ V


def supg_parameter(h: float, a, kappa: float, variant: str) -> float:
    """assembly.py:94-111 (used on the host only to document the formula; the
    device computes it per macro sub-cell class)."""
    anorm = float(np.linalg.norm(a))
    if anorm == 0.0:
        return 0.0
    pe = anorm * h / (2.0 * kappa)
    sign = -1.0 if variant == "classical-minus" else 1.0
    if pe > 30.0:
        g = 1.0 + sign / pe
    elif pe < 1e-4:
        g = pe / 3.0 - pe ** 3 / 45.0
        if sign > 0:
            g += 2.0 / pe
    else:
        g = 1.0 / math.tanh(pe) + sign / pe
    return h / (2.0 * anorm) * g
