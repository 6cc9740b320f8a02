"""Hot-path data contract of ``mehdg.assembly`` (assembly.py:63-82).

Only the block containers cross the drop-in boundary; FEM quadrature
assembly itself is outside the B200 path.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


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
