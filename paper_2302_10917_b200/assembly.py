"""``mehdg.assembly`` on the B200 path.

* The block containers of the drop-in boundary (assembly.py:63-82).
* Device assembly of the 2-D HDG blocks:
  ``assemble_system_device`` is ``assemble_system`` (schur_solver.py:482-492)
  with assemble_macro / assemble_face (assembly.py:170-322) computed by the
  csrc/assembly.cu kernels.  The host builds the reference-element tables
  (fem.py), evaluates the problem data (Python callables) at the quadrature
  points and projects the Dirichlet data; the blocks never leave the device.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import fem


@dataclass
class LocalOperators:
    """assembly.py:63-72: per-macro blocks A (nloc x nloc), B (nloc x nc),
    C (nc x nloc), R_u (nloc) and face_slots [(face id, slice)]."""

    macro_id: int
    A: object
    B: np.ndarray
    C: np.ndarray
    R_u: np.ndarray
    face_slots: list
    storage: str = "dense"
    lu = None  # the reference stores scipy factors here; the B200 path keeps them on the device


@dataclass
class FaceOperator:
    """assembly.py:75-82: per unknown face D (t x t) and R_hat (t)."""

    face_id: int
    D: np.ndarray
    R_hat: np.ndarray
    tag: str = "interior"
    factor = None
    factor_kind: str = ""


def operators_from_problem(prob: dict):
    """LocalOperators / FaceOperator views of a synthetic problem (the
    reference's injection recipe)."""
    t = prob["t"]
    mesh = prob["mesh"]
    nfe = prob["d"] + 1
    local_ops = []
    for e in range(prob["N"]):
        slots = [(int(mesh.elem_face[e, k]), slice(k * t, (k + 1) * t)) for k in range(nfe)]
        local_ops.append(LocalOperators(macro_id=e, A=prob["A"][e], B=prob["B"][e],
                                        C=prob["C"][e], R_u=prob["R_u"][e], face_slots=slots))
    face_ops = {}
    for fid in range(mesh.n_face):
        u = prob["uidx"][fid]
        if u >= 0:
            face_ops[fid] = FaceOperator(face_id=fid, D=prob["D"][u], R_hat=prob["R_hat"][u],
                                         tag=str(mesh.face_tag[fid]))
    return local_ops, face_ops


@dataclass
class ProblemData:
    """assembly.py:36-50: constant-velocity advection-diffusion data; f, g_D, g_N
    map (npts, 2) points to (npts,) values."""

    a: np.ndarray
    kappa: float
    f: Callable
    g_D: Callable
    g_N: Optional[Callable] = None

    def __post_init__(self):
        self.a = np.asarray(self.a, dtype=float)
        if self.kappa <= 0:
            raise ValueError("kappa must be positive")


@dataclass
class StabilizationConfig:
    """assembly.py:53-60."""

    supg: bool = False
    supg_variant: str = "classical-minus"  # or "paper-plus"

    def __post_init__(self):
        if self.supg_variant not in ("classical-minus", "paper-plus"):
            raise ValueError(f"unknown supg variant {self.supg_variant!r}")


def manufactured_tanh(kappa: float = 0.4, a=(1.0, 1.0), g_N: Optional[Callable] = None):
    """The reference's "tanh" manufactured case (mehdg/bench.py:46-70): interior
    layer u = (1 + tanh((y - 2x + 0.4) / kappa)) / 2 on the unit square."""
    if kappa <= 0:
        raise ValueError("kappa must be positive")
    k = float(kappa)
    ax, ay = float(a[0]), float(a[1])

    def sech2(z):
        return 1.0 / np.cosh(np.clip(z, -350.0, 350.0)) ** 2

    def u_exact(x):
        x = np.atleast_2d(x)
        return 0.5 * (1.0 + np.tanh((x[:, 1] - 2.0 * x[:, 0] + 0.4) / k))

    def f(x):
        x = np.atleast_2d(x)
        z = (x[:, 1] - 2.0 * x[:, 0] + 0.4) / k
        s2 = sech2(z)
        return 0.5 * s2 * (ay - 2.0 * ax) / k - k * (-5.0 * s2 * np.tanh(z) / k ** 2)

    return ProblemData(a=np.array([ax, ay]), kappa=k, f=f, g_D=u_exact, g_N=g_N)


class _Tables(C.Structure):
    """mh_hdg2d_tables (include/mehdg_b200.h)."""

    _fields_ = [(n, C.c_int32) for n in ("m", "p", "Q", "nb", "t", "nq", "ncell", "nfq",
                                         "nffq", "supg", "supg_plus")] + \
               [(n, C.c_double) for n in ("kappa", "ax", "ay")] + \
               [(n, C.c_void_p) for n in ("qw", "val", "gref", "href", "cell_kind", "cell_map",
                                          "edge_nodes", "fw", "th", "ps", "ffw", "fps")]


@dataclass
class DeviceBlocks:
    """Assembled blocks on the device (torch float64 CUDA tensors), in the
    layouts of LocalOperators / FaceOperator: A (N, nloc, nloc), B (N, nloc, nc)
    = op.B, C (N, nc, nloc) = op.C, R_u (N, nloc); D (F, t, t), R_hat (F, t) in
    unknown-face order."""

    A: object
    B: object
    C: object
    R_u: object
    D: object
    R_hat: object
    nloc: int
    t: int
    p: int
    m: int
    tables: dict


def _side_params(mesh, tables: dict) -> np.ndarray:
    """(F, 2, 2) FaceSide (t0, t1) of every face's left / right side (mesh.py:130-135):
    for our structured mesh from the exact lattice order of the edge end points
    (the face vertices are in canonical lexicographic order, mesh.py:222-223);
    for the reference MacroMesh read from its FaceSide records."""
    F = len(tables["face_left"])
    tt = np.zeros((F, 2, 2))
    if hasattr(mesh, "vertices_lattice"):
        lat = mesh.vertices_lattice[mesh.elem_verts]  # (N, 3, 2)
        for c, fs in enumerate((tables["face_left"], tables["face_right"])):
            e, k = fs[:, 0], fs[:, 1]
            ok = e >= 0
            a = np.array([ev[0] for ev in fem.EDGE_VERTS])[k[ok]]
            b = np.array([ev[1] for ev in fem.EDGE_VERTS])[k[ok]]
            pa, pb = lat[e[ok], a], lat[e[ok], b]
            rev = (pa[:, 0] > pb[:, 0]) | ((pa[:, 0] == pb[:, 0]) & (pa[:, 1] > pb[:, 1]))
            tt[ok, c, 0] = rev.astype(float)
            tt[ok, c, 1] = 1.0 - rev
        return tt
    for face in mesh.skeleton:
        for c, side in enumerate(face.sides()):
            tt[face.id, c] = (side.t0, side.t1)
    return tt


def _face_verts(mesh, fids: np.ndarray) -> np.ndarray:
    if hasattr(mesh, "face_verts"):
        return mesh.vertices[mesh.face_verts[fids]]
    return np.stack([np.asarray(mesh.skeleton[int(f)].verts, float) for f in fids]) \
        if len(fids) else np.zeros((0, 2, 2))


def assemble_system_device(mesh, problem: ProblemData, stab: StabilizationConfig, p: int,
                           quad_degree: Optional[int] = None, device: int = 0,
                           tables: Optional[dict] = None,
                           timings: Optional[dict] = None) -> DeviceBlocks:
    """assemble_system (schur_solver.py:482-492) on the device, for a conforming
    2-D structured macro mesh (ours or the reference's).  ``timings`` (optional
    dict) receives host_s (tables, data evaluation, uploads) and kernel_ms (the
    two assembly kernels, CUDA events)."""
    import time as _time

    t_host0 = _time.perf_counter()
    from . import _lib
    from ._lib import check, lib
    from .mesh import condense_tables, mesh_tables
    import torch

    _lib.require_gpu()
    if getattr(mesh, "d", 2) != 2:
        raise NotImplementedError("the HDG block assembly is two-dimensional (assembly.py)")
    ms = {int(e.m) for e in mesh.macro_elements} if not hasattr(mesh, "m") else {int(mesh.m)}
    if len(ms) != 1:
        raise NotImplementedError("mixed macro subdivisions (adaptive meshes) are not on the "
                                  "B200 path (SURVEY.md 8(f) row 4)")
    m = ms.pop()
    if tables is None:
        tables = mesh_tables(mesh)
        tables.update(condense_tables(tables))
    if quad_degree is None:
        quad_degree = 2 * p + 2 if stab.supg else 2 * p + 1  # assembly.py:188-189
    tab = fem.asm_tables(m, p, quad_degree)
    dev = torch.device(f"cuda:{device}")
    verts = fem.macro_geometry(mesh)
    N = verts.shape[0]
    Q, t = tab.Q, tab.t
    nloc = 3 * Q

    def d(x, dtype=torch.float64):
        return torch.as_tensor(np.ascontiguousarray(x), dtype=dtype, device=dev)

    # problem data at the quadrature points (host; the data are Python callables)
    pts = fem.quad_points(verts, tab)
    fq = np.asarray(problem.f(pts.reshape(-1, 2)), dtype=float).reshape(pts.shape[:3])
    face_tag = np.array([str(tg) for tg in (mesh.face_tag if hasattr(mesh, "face_tag")
                                            else [f.tag for f in mesh.skeleton])])
    elem_face = np.asarray(tables["elem_face"])  # (N, S) faces in slot order, -1 = none
    S = elem_face.shape[1]
    dfaces = np.nonzero(face_tag == "D")[0]
    drow = np.full(face_tag.size, -1, np.int32)
    drow[dfaces] = np.arange(dfaces.size, dtype=np.int32)
    slot_dir = np.where(elem_face >= 0, drow[np.maximum(elem_face, 0)], -1).astype(np.int32)
    ghat = fem.dirichlet_projection(_face_verts(mesh, dfaces), problem.g_D, p, m) \
        if dfaces.size else np.zeros((1, t))
    # per slot: local edge, side variant (t0, t1) and face length
    F_all = face_tag.size
    fverts = _face_verts(mesh, np.arange(F_all))
    flen = np.linalg.norm(fverts[:, 1] - fverts[:, 0], axis=1)
    tt = _side_params(mesh, tables)
    slot_edge = np.full((N, S), -1, np.int8)
    slot_var = np.zeros((N, S), np.int8)
    slot_len = np.zeros((N, S))
    for c, fs in enumerate((np.asarray(tables["face_left"]), np.asarray(tables["face_right"]))):
        ok = np.nonzero(fs[:, 0] >= 0)[0]
        e, j = fs[ok, 0], fs[ok, 1]
        slot_edge[e, j] = np.asarray(tables["face_edge"])[ok, c]
        slot_var[e, j] = fem.side_variant(tt[ok, c, 0], tt[ok, c, 1])
        slot_len[e, j] = flen[ok]

    keep = dict(qw=d(tab.qw), val=d(tab.val), gref=d(tab.gref), href=d(tab.href),
                cell_kind=d(tab.cell_kind, torch.int32), cell_map=d(tab.cell_map, torch.int32),
                edge_nodes=d(tab.edge_nodes, torch.int32), fw=d(tab.fw), th=d(tab.th),
                ps=d(tab.ps), ffw=d(tab.ffw), fps=d(tab.fps))
    T = _Tables(m=m, p=p, Q=Q, nb=tab.nb, t=t, nq=tab.qw.size, ncell=len(tab.cell_kind),
                nfq=tab.fw.shape[1], nffq=tab.ffw.size, supg=int(stab.supg),
                supg_plus=int(stab.supg_variant == "paper-plus"), kappa=float(problem.kappa),
                ax=float(problem.a[0]), ay=float(problem.a[1]),
                **{k: v.data_ptr() for k, v in keep.items()})
    nc = S * t
    A = torch.empty((N, nloc, nloc), dtype=torch.float64, device=dev)
    B = torch.empty((N, nloc, nc), dtype=torch.float64, device=dev)
    Cm = torch.empty((N, nc, nloc), dtype=torch.float64, device=dev)
    Ru = torch.empty((N, nloc), dtype=torch.float64, device=dev)
    verts_d = d(verts)
    se_d, sv_d, sd_d, sl_d = (d(slot_edge, torch.int8), d(slot_var, torch.int8),
                              d(slot_dir, torch.int32), d(slot_len))
    ghat_d, fq_d = d(ghat), d(fq)
    stream = torch.cuda.current_stream(dev).cuda_stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    uidx = np.asarray(tables["uidx"])
    ufaces = np.nonzero(uidx >= 0)[0]
    ufaces = ufaces[np.argsort(uidx[ufaces])]
    F = ufaces.size
    fe = np.asarray(tables["face_edge"])[ufaces]
    sides = np.stack((np.asarray(tables["face_left"])[ufaces, 0], fe[:, 0],
                      np.asarray(tables["face_right"])[ufaces, 0], fe[:, 1]), axis=1)
    sides = np.ascontiguousarray(sides, dtype=np.int32)
    flen_d = d(flen[ufaces])
    D = torch.empty((F, t, t), dtype=torch.float64, device=dev)
    sides_d = d(sides, torch.int32)
    t_host = _time.perf_counter() - t_host0
    ev0.record(torch.cuda.current_stream(dev))
    check(lib.mh_assemble_macros_2d(C.addressof(T), N, S, verts_d.data_ptr(), se_d.data_ptr(),
                                    sv_d.data_ptr(), sd_d.data_ptr(), sl_d.data_ptr(),
                                    ghat_d.data_ptr(), fq_d.data_ptr(), A.data_ptr(),
                                    B.data_ptr(), Cm.data_ptr(), Ru.data_ptr(), stream),
          "mh_assemble_macros_2d")
    # face blocks in unknown-face order (the order of condense's offsets)
    check(lib.mh_assemble_faces_2d(C.addressof(T), F, verts_d.data_ptr(), sides_d.data_ptr(),
                                   flen_d.data_ptr(), D.data_ptr(), stream),
          "mh_assemble_faces_2d")
    ev1.record(torch.cuda.current_stream(dev))
    Rh = np.zeros((F, t))
    nfaces = np.nonzero(face_tag[ufaces] == "N")[0]
    if nfaces.size:
        if problem.g_N is None:
            raise ValueError("Neumann face present but g_N not provided")
        Rh[nfaces] = fem.neumann_rhs(_face_verts(mesh, ufaces[nfaces]), problem.g_N, p, m)
    torch.cuda.current_stream(dev).synchronize()
    if timings is not None:
        timings["host_s"] = t_host
        timings["kernel_ms"] = ev0.elapsed_time(ev1)
    return DeviceBlocks(A=A, B=B, C=Cm, R_u=Ru, D=D, R_hat=d(Rh), nloc=nloc, t=t, p=p, m=m,
                        tables=tables)
