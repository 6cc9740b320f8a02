"""Oracle (test infrastructure): structured macro-mesh skeleton on integer lattices.

Restates the connectivity half of ``/root/reference/pkg/src/mehdg/mesh.py``:

* d=2 macro enumeration  -- ``build_structured_macro_mesh`` (mesh.py:359-389):
  cells row-major (j outer, i inner), two triangles per cell with the diagonal
  (i,j)->(i+1,j+1): ``[p00, p10, p11]`` then ``[p00, p11, p01]`` (mesh.py:381-387).
* vertex ids by first visit in macro order -- ``_dedup_vertices`` (mesh.py:331-345).
* local edge k opposite vertex k, directed as ``EDGE_VERTS`` (mesh.py:68).
* face matching by the snapped vertex pair (mesh.py:207-245); the left side is
  the record with the lower macro id (mesh.py:235); unmatched edges on the
  square boundary are tagged ``"D"`` unless a tagger says otherwise (mesh.py:248-258).
* face ids = lexicographic order of the canonical (sorted) snapped vertex
  tuple (mesh.py:304).  Coordinates are ``i*h`` snapped to 12 digits
  (``_key``, mesh.py:28-29); on a structured lattice that order is the integer
  lattice order, which is what we sort on.
* d=3: tets exactly as ``_build_kuhn_counting_mesh`` (mesh.py:392-425): cubes in
  (i, j, k) loop order, ``sorted(permutations(range(3)))`` paths, vertex ids by
  first visit.  The reference carries no 3-D skeleton (mesh.py:372-375); the
  skeleton here generalises the 2-D rules (face k opposite vertex k, sorted
  vertex-triple key, left = lower tet id, cube-surface faces tagged ``"D"``).
  This is the decision SURVEY.md section 8(c) asks the build to document.

Outputs are plain int64 numpy arrays so that the CUDA library's connectivity
builder can be compared bit-for-bit.
"""

from __future__ import annotations

from itertools import permutations

import numpy as np

# mesh.py:68 -- local edge k is opposite vertex k; direction (a, b)
EDGE_VERTS = ((1, 2), (2, 0), (0, 1))


def _macros_2d(n: int):
    """Lattice vertex triples of the 2n^2 triangles (mesh.py:376-387)."""
    out = []
    for j in range(n):
        for i in range(n):
            p00, p10 = (i, j), (i + 1, j)
            p11, p01 = (i + 1, j + 1), (i, j + 1)
            out.append((p00, p10, p11))
            out.append((p00, p11, p01))
    return out


def _macros_3d(n: int):
    """Lattice vertex quadruples of the 6n^3 Kuhn tets (mesh.py:407-417)."""
    out = []
    perms = sorted(permutations(range(3)))
    for i in range(n):
        for j in range(n):
            for k in range(n):
                for perm in perms:
                    path = [(i, j, k)]
                    for axis in perm:
                        nxt = list(path[-1])
                        nxt[axis] += 1
                        path.append(tuple(nxt))
                    out.append(tuple(path))
    return out


def _on_boundary(pts, n: int) -> bool:
    """Face lies in one plane x_c in {0, n} (mesh.py:194-199 generalised)."""
    d = len(pts[0])
    for c in range(d):
        for v in (0, n):
            if all(p[c] == v for p in pts):
                return True
    return False


def structured_skeleton(d: int, n: int, tagger=None) -> dict:
    """Skeleton tables of the structured macro mesh of [0,1]^d.

    Returns a dict of int64 arrays:
      verts (nv, d) lattice coords; elem_verts (N, d+1);
      face_verts (F, d) vertex ids in canonical (sorted) order;
      face_left (F, 2) = (macro, local face); face_right (F, 2) (-1 if none);
      face_tag (F,) 0 interior / 1 "D" / 2 "N"; elem_face (N, d+1).
    For d=2 also face_left_t / face_right_t (F, 2): the FaceSide (t0, t1)
    edge parameters of mesh.py:226-230 (0 or 1 on a conforming mesh).
    ``tagger(midpoint_xy) -> "D" | "N"`` mirrors the boundary_tagger hook.
    """
    if d not in (2, 3):
        raise ValueError(f"unsupported dimension {d}")
    if n < 1:
        raise ValueError("n must be >= 1")
    macros = _macros_2d(n) if d == 2 else _macros_3d(n)

    vid: dict = {}
    coords = []
    elem_verts = np.empty((len(macros), d + 1), dtype=np.int64)
    for e, pts in enumerate(macros):
        for a, pt in enumerate(pts):
            if pt not in vid:
                vid[pt] = len(coords)
                coords.append(pt)
            elem_verts[e, a] = vid[pt]

    # records: (macro, local face, ordered vertex list) -- mesh.py:211-218
    by_key: dict = {}
    records = []
    for e, pts in enumerate(macros):
        for k in range(d + 1):
            if d == 2:
                a, b = EDGE_VERTS[k]
                fpts = (pts[a], pts[b])
            else:
                fpts = tuple(pts[a] for a in range(4) if a != k)
            rid = len(records)
            records.append((e, k, fpts))
            by_key.setdefault(tuple(sorted(fpts)), []).append(rid)

    raw = []  # (key, left rid, right rid or -1, tag)
    for key, rids in by_key.items():
        if len(rids) == 2:
            r0, r1 = sorted(rids, key=lambda r: records[r][0])  # mesh.py:235
            raw.append((key, r0, r1, 0))
        elif len(rids) == 1:
            if not _on_boundary(key, n):
                raise ValueError("unmatched interior face")
            tag = 1
            if tagger is not None:
                mid = np.mean(np.asarray(key, float), axis=0) / n
                t = tagger(mid)
                if t not in ("D", "N"):
                    raise ValueError(f"invalid boundary tag {t!r}")
                tag = 1 if t == "D" else 2
            raw.append((key, rids[0], -1, tag))
        else:
            raise ValueError("more than two macros share a face")
    raw.sort(key=lambda r: r[0])  # mesh.py:304

    F = len(raw)
    face_verts = np.empty((F, d), dtype=np.int64)
    face_left = np.empty((F, 2), dtype=np.int64)
    face_right = np.full((F, 2), -1, dtype=np.int64)
    face_tag = np.empty(F, dtype=np.int64)
    elem_face = np.full((len(macros), d + 1), -1, dtype=np.int64)
    face_left_t = np.zeros((F, 2))
    face_right_t = np.zeros((F, 2))
    for fid, (key, rl, rr, tag) in enumerate(raw):
        face_verts[fid] = [vid[p] for p in key]
        face_tag[fid] = tag
        for col, rid in ((0, rl), (1, rr)):
            if rid < 0:
                continue
            e, k, fpts = records[rid]
            if col == 0:
                face_left[fid] = (e, k)
            else:
                face_right[fid] = (e, k)
            elem_face[e, k] = fid
            if d == 2:
                # FaceSide t0/t1: edge parameter of canonical v0, v1 (mesh.py:226-230)
                pa, _ = fpts
                tt = (0.0, 1.0) if pa == key[0] else (1.0, 0.0)
                (face_left_t if col == 0 else face_right_t)[fid] = tt
    out = dict(
        d=d, n=n, verts=np.asarray(coords, dtype=np.int64), elem_verts=elem_verts,
        face_verts=face_verts, face_left=face_left, face_right=face_right,
        face_tag=face_tag, elem_face=elem_face,
    )
    if d == 2:
        out["face_left_t"] = face_left_t
        out["face_right_t"] = face_right_t
    return out


def kuhn_tets(n: int) -> tuple:
    """(vertices lattice coords, tets vertex ids) as ``_build_kuhn_counting_mesh``."""
    sk = structured_skeleton(3, n)
    return sk["verts"], sk["elem_verts"]


def interior_face_count(d: int, n: int) -> int:
    """Cost-model face count D = A_d n^d + B_d d n^(d-1) (n-1) (costmodel.py:14, 53)."""
    A_d, B_d = {2: (1, 1), 3: (6, 2)}[d]
    return A_d * n**d + B_d * d * n ** (d - 1) * (n - 1)
