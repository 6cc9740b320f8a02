"""Structured macro mesh connectivity, built by the C++ skeleton builder.

Mirrors the parts of ``mehdg.mesh`` (/root/reference/pkg/src/mehdg/mesh.py)
that the solver consumes: ``build_structured_macro_mesh`` (mesh.py:359-389),
``MacroMesh.skeleton`` with ``SkeletonFace.{id, tag, sides()}``
(mesh.py:139-171) and ``FaceSide.{macro, edge}`` (mesh.py:130-135).  The
integer tables are bit-identical to the reference's 2-D skeleton; d=3 adds
the Kuhn-tet skeleton the reference only counts (mesh.py:392-425).
Geometry (affine maps, normals, VTK export) is not on the operator path and
is not reproduced.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Callable, Optional

import numpy as np

from . import _lib
from ._lib import check, lib, ptr


@dataclass
class FaceSide:
    """mesh.py:130-135 (t0/t1 are 0/1 on the conforming structured mesh)."""

    macro: int
    edge: int
    t0: float = 0.0
    t1: float = 1.0


@dataclass
class SkeletonFace:
    """mesh.py:139-171, connectivity fields only."""

    id: int
    left: FaceSide
    right: Optional[FaceSide]
    tag: str
    m_f: int
    vertex_ids: tuple = ()

    @property
    def is_boundary(self) -> bool:
        return self.right is None

    def sides(self) -> list:
        return [self.left] if self.right is None else [self.left, self.right]


@dataclass
class MacroElement:
    id: int
    vertex_ids: tuple
    m: int
    level: int = 0


class StructuredMacroMesh:
    """Array-backed ``MacroMesh``: the skeleton objects are built lazily."""

    def __init__(self, d, n, m, verts, elem_verts, face_verts, face_left, face_right,
                 face_boundary, elem_face, face_tag):
        self.d, self.n, self.m = d, n, m
        self.vertices_lattice = verts
        self.elem_verts = elem_verts
        self.face_verts = face_verts
        self.face_left = face_left
        self.face_right = face_right
        self.face_boundary = face_boundary
        self.elem_face = elem_face
        self.face_tag = face_tag  # np.array of "interior" / "D" / "N"
        self._skeleton = None
        self._macros = None

    @property
    def vertices(self) -> np.ndarray:
        return self.vertices_lattice / float(self.n)

    @property
    def n_elem(self) -> int:
        return int(self.elem_verts.shape[0])

    @property
    def n_face(self) -> int:
        return int(self.face_left.shape[0])

    @property
    def face_unknown(self) -> np.ndarray:
        return (self.face_tag != "D").astype(np.int8)

    @property
    def macro_elements(self) -> list:
        if self._macros is None:
            self._macros = [MacroElement(i, tuple(int(v) for v in row), self.m)
                            for i, row in enumerate(self.elem_verts)]
        return self._macros

    @property
    def skeleton(self) -> list:
        if self._skeleton is None:
            sk = []
            for f in range(self.n_face):
                l = self.face_left[f]
                r = self.face_right[f]
                right = FaceSide(int(r[0]), int(r[1])) if r[0] >= 0 else None
                sk.append(SkeletonFace(f, FaceSide(int(l[0]), int(l[1])), right,
                                       str(self.face_tag[f]), self.m,
                                       tuple(int(v) for v in self.face_verts[f])))
            self._skeleton = sk
        return self._skeleton

    def interior_faces(self) -> list:
        return [f for f in self.skeleton if f.tag == "interior"]

    def boundary_faces(self) -> list:
        return [f for f in self.skeleton if f.tag != "interior"]


def skeleton_sizes(d: int, n: int) -> tuple:
    ne, nv, nf = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib.mh_skeleton_sizes(d, n, C.byref(ne), C.byref(nv), C.byref(nf)),
          "mh_skeleton_sizes")
    return ne.value, nv.value, nf.value


def build_structured_macro_mesh(d: int, n: int, m: int,
                                boundary_tagger: Optional[Callable] = None,
                                counting_only: bool = False) -> StructuredMacroMesh:
    """Structured macro mesh of [0,1]^d with d! n^d macro simplices
    (mesh.py:359-389); d=3 carries the Kuhn-tet skeleton as well."""
    if d not in (2, 3):
        raise ValueError(f"unsupported dimension {d}")
    if n < 1 or m < 1:
        raise ValueError("n and m must be >= 1")
    ne, nv, nf = skeleton_sizes(d, n)
    verts = np.empty((nv, d), np.int32)
    elem_verts = np.empty((ne, d + 1), np.int32)
    face_verts = np.empty((nf, d), np.int32)
    face_left = np.empty((nf, 2), np.int32)
    face_right = np.empty((nf, 2), np.int32)
    face_boundary = np.empty(nf, np.int8)
    elem_face = np.empty((ne, d + 1), np.int32)
    check(lib.mh_build_skeleton(d, n, ptr(verts), ptr(elem_verts), ptr(face_verts),
                                ptr(face_left), ptr(face_right), ptr(face_boundary),
                                ptr(elem_face)), "mh_build_skeleton")
    tags = np.where(face_boundary == 1, "D", "interior").astype(object)
    if boundary_tagger is not None:
        for f in np.nonzero(face_boundary)[0]:
            mid = verts[face_verts[f]].mean(axis=0) / float(n)
            t = boundary_tagger(mid)
            if t not in ("D", "N"):
                raise ValueError(f"invalid boundary tag {t!r}")
            tags[f] = t
    return StructuredMacroMesh(d, n, m, verts, elem_verts, face_verts, face_left, face_right,
                               face_boundary, elem_face, tags)


def mesh_tables(mesh) -> dict:
    """Integer skeleton tables of any mesh exposing ``skeleton`` with
    ``id``/``tag``/``sides()`` (ours or the reference ``MacroMesh``)."""
    if isinstance(mesh, StructuredMacroMesh):
        return dict(nfe=mesh.d + 1, n_elem=mesh.n_elem, face_unknown=mesh.face_unknown,
                    elem_face=mesh.elem_face, face_left=mesh.face_left,
                    face_right=mesh.face_right,
                    face_edge=np.stack((mesh.face_left[:, 1], mesh.face_right[:, 1]), axis=1),
                    hanging=False)
    skel = list(mesh.skeleton)
    macros = list(mesh.macro_elements)
    n_elem = len(macros)
    nfe = getattr(mesh, "d", 2) + 1
    F = len(skel)
    face_left = np.full((F, 2), -1, np.int32)
    face_right = np.full((F, 2), -1, np.int32)
    face_edge = np.full((F, 2), -1, np.int32)
    face_unknown = np.zeros(F, np.int8)
    # 2:1 hanging faces (mesh.py:264-302): a macro edge carries two faces; the
    # macro's slots are then its face lists in order, edge by edge
    # (assemble_macro's face_slots, assembly.py:241-249), up to 6 in 2-D
    hanging = all(hasattr(e, "faces") for e in macros) and \
        any(len(fl) > 1 for e in macros for fl in e.faces)
    if hanging:
        slots = [[int(fid) for k in range(nfe) for fid in e.faces[k]] for e in macros]
        nfe = max(len(sl) for sl in slots)
        elem_face = np.full((n_elem, nfe), -1, np.int32)
        slot_of = {}
        for e, sl in enumerate(slots):
            elem_face[e, :len(sl)] = sl
            for j, fid in enumerate(sl):
                slot_of[(e, fid)] = j
    else:
        elem_face = np.full((n_elem, nfe), -1, np.int32)
    for pos, face in enumerate(skel):
        if face.id != pos:
            raise ValueError("skeleton face ids must be 0..F-1 in order")
        for col, side in enumerate(face.sides()):
            slot = slot_of[(side.macro, pos)] if hanging else side.edge
            (face_left if col == 0 else face_right)[pos] = (side.macro, slot)
            face_edge[pos, col] = side.edge
            if not hanging:
                if elem_face[side.macro, side.edge] != -1:
                    raise ValueError("two faces on one macro edge without face lists")
                elem_face[side.macro, side.edge] = pos
        face_unknown[pos] = 0 if face.tag == "D" else 1
    return dict(nfe=nfe, n_elem=n_elem, face_unknown=face_unknown, elem_face=elem_face,
                face_left=face_left, face_right=face_right, face_edge=face_edge,
                hanging=hanging)


def condense_tables(tables: dict) -> dict:
    """``condense``'s integer tables (schur_solver.py:198-241) via the C++ builder."""
    nfe, n_elem = tables["nfe"], tables["n_elem"]
    fu = np.ascontiguousarray(tables["face_unknown"], np.int8)
    ef = np.ascontiguousarray(tables["elem_face"], np.int32)
    fl = np.ascontiguousarray(tables["face_left"], np.int32)
    fr = np.ascontiguousarray(tables["face_right"], np.int32)
    F_all = fu.size
    uidx = np.empty(F_all, np.int32)
    elem_ufac = np.empty((n_elem, nfe), np.int32)
    Fu = int(fu.astype(bool).sum())
    face_elem = np.empty((Fu, 2), np.int32)
    face_slot = np.empty((Fu, 2), np.int32)
    nu = C.c_int64()
    check(lib.mh_condense_tables(nfe, n_elem, F_all, ptr(fu), ptr(ef), ptr(fl), ptr(fr),
                                 ptr(uidx), ptr(elem_ufac), ptr(face_elem), ptr(face_slot),
                                 C.byref(nu)), "mh_condense_tables")
    assert nu.value == Fu
    return dict(uidx=uidx, elem_ufac=elem_ufac, face_elem=face_elem, face_slot=face_slot, F=Fu)


def slab_partition(n_elem: int, elems_per_slab: int, nranks: int) -> np.ndarray:
    out = np.empty(nranks + 1, np.int64)
    check(lib.mh_slab_partition(n_elem, elems_per_slab, nranks, ptr(out)), "mh_slab_partition")
    return out


def elems_per_slab(d: int, n: int) -> int:
    """Macros per mesh slab: 2n per row in 2-D (mesh.py:376-387), 6n^2 per
    x-slab in 3-D (mesh.py:407-417)."""
    return 2 * n if d == 2 else 6 * n * n
