"""2:1 hanging faces: adaptive meshes from the reference's
refine_macros, rebuilt here from tests/golden/adaptive_tanh_*.npz (made by
tests/golden/make_golden.py adaptive from mehdg itself).  A macro then carries
up to 6 face slots (two faces on a refined neighbour's edge); the B200 path
pads the narrower macros with empty slots."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2302_10917_b200 as P
from paper_2302_10917_b200.assembly import (StabilizationConfig, assemble_system_device,
                                            manufactured_tanh)
from paper_2302_10917_b200.mesh import condense_tables, mesh_tables
from conftest import golden, rel

pytestmark = pytest.mark.gpu

FIXTURES = ["adaptive_tanh_n2m2p2.npz", "adaptive_tanh_n2m1p3_2lev.npz"]
APPLY_TOL = 1e-12
SOLVE_TOL = 1e-9


class Side:
    def __init__(self, macro, edge, t0, t1):
        self.macro, self.edge, self.t0, self.t1 = int(macro), int(edge), float(t0), float(t1)


class Face:
    def __init__(self, fid, sides, tag, verts, m_f):
        self.id, self._sides, self.tag, self.verts, self.m_f = fid, sides, tag, verts, m_f

    def sides(self):
        return self._sides


class Macro:
    def __init__(self, eid, verts, m, faces):
        self.id, self.verts, self.m, self.faces = eid, verts, m, faces


class AdaptiveMesh:
    """Duck-typed mehdg MacroMesh with hanging faces, from the fixture arrays."""

    d = 2

    def __init__(self, g):
        fs = g["face_side"]
        self.skeleton = []
        for f in range(fs.shape[0]):
            sides = [Side(*fs[f, c]) for c in range(2) if fs[f, c, 0] >= 0]
            self.skeleton.append(Face(f, sides, str(g["face_tag"][f]), g["face_verts"][f],
                                      int(g["face_mf"][f])))
        self.macro_elements = []
        for e in range(g["mesh_verts"].shape[0]):
            per_edge = [[], [], []]
            for fid in g["mesh_faces"][e]:
                if fid < 0:
                    continue
                side = next(s for s in self.skeleton[fid].sides() if s.macro == e)
                per_edge[side.edge].append(int(fid))
            self.macro_elements.append(Macro(e, g["mesh_verts"][e], int(g["mesh_m"][e]), per_edge))
        self.n = int(g["n"])


def local_ops_from(g, mesh):
    t = g["D"].shape[1]
    ops = []
    for e in range(g["A"].shape[0]):
        ns = int(g["nslot"][e])
        fids = [fid for k in range(3) for fid in mesh.macro_elements[e].faces[k]]
        slots = [(fid, slice(k * t, (k + 1) * t)) for k, fid in enumerate(fids)]
        ops.append(P.LocalOperators(macro_id=e, A=g["A"][e], B=g["B"][e][:, :ns * t],
                                    C=g["C"][e][:ns * t], R_u=g["R_u"][e], face_slots=slots))
    fops = {int(f): P.FaceOperator(face_id=int(f), D=g["D"][i], R_hat=g["R_hat"][i])
            for i, f in enumerate(g["face_ids"])}
    return ops, fops


@pytest.mark.parametrize("fx", FIXTURES)
def test_slot_tables(fx):
    g = golden(fx)
    mesh = AdaptiveMesh(g)
    tab = mesh_tables(mesh)
    assert tab["hanging"] and tab["nfe"] == int((g["mesh_faces"] >= 0).sum(axis=1).max())
    assert int(g["face_hanging"].sum()) > 0
    tab.update(condense_tables(tab))
    assert tab["F"] == g["D"].shape[0]


@pytest.mark.parametrize("fx", FIXTURES)
def test_condense_apply_solve_with_hanging_faces(fx):
    """The reference's own blocks through condense / apply / D^-1 / GMRES / reconstruct."""
    g = golden(fx)
    mesh = AdaptiveMesh(g)
    ops, fops = local_ops_from(g, mesh)
    sys_ = P.condense(mesh, ops, fops, P.SolverConfig(tol=1e-12))
    assert rel(sys_.f_vec, g["f"]) <= APPLY_TOL
    for i in range(g["xs"].shape[0]):
        assert rel(P.apply_schur(sys_, g["xs"][i]), g["w"][i]) <= APPLY_TOL
        assert rel(P.apply_preconditioner(sys_, g["xs"][i]), g["z"][i]) <= APPLY_TOL
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, P.SolverConfig(tol=1e-12),
                      precond=P.Preconditioner(sys_))
    assert abs(info["iterations"] - int(g["iterations"])) <= 1
    assert rel(x, g["x"]) <= SOLVE_TOL
    assert rel(np.stack(P.reconstruct_interior(sys_, x)), g["U"]) <= SOLVE_TOL


@pytest.mark.parametrize("fx", FIXTURES)
def test_device_assembly_with_hanging_faces(fx):
    """assemble_macro on half-edge faces (side parameters (0, .5), (.5, 1), ...)."""
    g = golden(fx)
    mesh = AdaptiveMesh(g)
    p = int(g["p"])
    blk = assemble_system_device(mesh, manufactured_tanh(0.4, (1.0, 1.0)),
                                 StabilizationConfig(), p)
    A, B, Cm, Ru = (x.cpu().numpy() for x in (blk.A, blk.B, blk.C, blk.R_u))
    assert B.shape == g["B"].shape
    for e in range(A.shape[0]):
        for x, ref in ((A[e], g["A"][e]), (B[e], g["B"][e]), (Cm[e], g["C"][e]),
                       (Ru[e], g["R_u"][e])):
            assert np.abs(x - ref).max() <= 1e-12 * np.abs(ref).max(), e
    D = blk.D.cpu().numpy()
    assert np.abs(D - g["D"]).max() <= 1e-12 * np.abs(g["D"]).max()
    sol, _ = P.solve(mesh, manufactured_tanh(0.4, (1.0, 1.0)), StabilizationConfig(),
                     P.SolverConfig(tol=1e-12), p)
    assert abs(sol.report.iterations - int(g["iterations"])) <= 1
    assert rel(sol.uhat, g["x"]) <= SOLVE_TOL
    assert rel(np.stack(sol.local), g["U"]) <= SOLVE_TOL
