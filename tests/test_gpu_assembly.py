"""Device assembly of the 2-D HDG blocks against the
reference's own assemble_system output (tests/golden/real_tanh_*.npz, made by
tests/golden/make_golden.py from mehdg itself), and the full solve() driver
(assembly -> condense -> GMRES -> reconstruct, all on the device)."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2302_10917_b200 as P
from paper_2302_10917_b200.assembly import (StabilizationConfig, assemble_system_device,
                                            manufactured_tanh)
from conftest import golden, rel

pytestmark = pytest.mark.gpu

BLOCK_TOL = 1e-12   # assembled entries, relative to the block's max |entry|
SOLVE_TOL = 1e-9    # converged traces / interior unknowns (north_star)


def tanh_problem(neumann=False):
    """The fixtures' problem: the reference's tanh case (kappa 0.4, a = (1, 1)) and,
    for the Neumann fixture, g_N = sin(3y) + x/2 (make_golden.py)."""
    def g_n(x):
        x = np.atleast_2d(x)
        return np.sin(3.0 * x[:, 1]) + 0.5 * x[:, 0]

    return manufactured_tanh(0.4, (1.0, 1.0), g_N=g_n if neumann else None)


FIXTURES = ["real_tanh_n2m2p2.npz", "real_tanh_n3m1p3.npz", "real_tanh_n2m3p2.npz",
            "real_tanh_n2m2p2_supg.npz", "real_tanh_n2m2p3_supgplus.npz",
            "real_tanh_n2m2p2_neumann.npz"]


def case(fx):
    g = golden(fx)
    n, m, p = int(g["n"]), int(g["m"]), int(g["p"])
    neumann = bool(g["neumann"]) if "neumann" in g.files else False
    supg = str(g["supg"]) if "supg" in g.files else ""
    tagger = (lambda x: "N" if x[0] < 1e-12 else "D") if neumann else None
    mesh = P.build_structured_macro_mesh(2, n, m, boundary_tagger=tagger)
    stab = StabilizationConfig(supg=bool(supg), supg_variant=supg or "classical-minus")
    return g, mesh, tanh_problem(neumann=neumann), stab, p


def brel(x, ref):
    return np.abs(x - ref).max() / max(np.abs(ref).max(), 1e-300)


@pytest.mark.parametrize("fx", FIXTURES)
def test_device_blocks_match_reference_assembly(fx):
    g, mesh, problem, stab, p = case(fx)
    blk = assemble_system_device(mesh, problem, stab, p)
    A, B, Cm, Ru = (x.cpu().numpy() for x in (blk.A, blk.B, blk.C, blk.R_u))
    D, Rh = blk.D.cpu().numpy(), blk.R_hat.cpu().numpy()
    assert A.shape == g["A"].shape and B.shape == g["B"].shape and D.shape == g["D"].shape
    for e in range(A.shape[0]):
        assert brel(A[e], g["A"][e]) <= BLOCK_TOL, e
        assert brel(B[e], g["B"][e]) <= BLOCK_TOL, e
        assert brel(Cm[e], g["C"][e]) <= BLOCK_TOL, e
        assert brel(Ru[e], g["R_u"][e]) <= BLOCK_TOL, e
    assert brel(D, g["D"]) <= BLOCK_TOL
    assert brel(Rh, g["R_hat"]) <= BLOCK_TOL if np.abs(g["R_hat"]).max() > 0 else \
        np.abs(Rh).max() == 0.0


@pytest.mark.parametrize("fx", FIXTURES)
def test_solve_with_device_assembly_matches_reference(fx):
    """P.solve(mesh, problem, stab, config, p) -- the reference's top-level entry
    (schur_solver.py:495-541) -- end to end on the device."""
    g, mesh, problem, stab, p = case(fx)
    sol, sys_ = P.solve(mesh, problem, stab, P.SolverConfig(tol=1e-12), p)
    rec = sol.report.to_record()
    assert rec["converged"]
    assert abs(rec["iterations"] - int(g["iterations"])) <= 1
    assert rel(sol.uhat, g["x"]) <= SOLVE_TOL
    assert rel(np.stack(sol.local), g["U"]) <= SOLVE_TOL


def test_device_assembly_is_deterministic():
    g, mesh, problem, stab, p = case("real_tanh_n2m2p2_supg.npz")
    a1 = assemble_system_device(mesh, problem, stab, p)
    a2 = assemble_system_device(mesh, problem, stab, p)
    for x, y in ((a1.A, a2.A), (a1.B, a2.B), (a1.C, a2.C), (a1.R_u, a2.R_u), (a1.D, a2.D)):
        assert bool((x == y).all())


def test_device_assembly_on_the_reference_mesh_object():
    """The reference's MacroMesh is accepted duck-typed (macro verts, FaceSide t0/t1)."""
    g, mesh, problem, stab, p = case("real_tanh_n3m1p3.npz")

    class Side:
        def __init__(self, macro, edge, t0):
            self.macro, self.edge, self.t0, self.t1 = macro, edge, t0, 1.0 - t0

    class Face:
        def __init__(self, fid, sides, tag, verts):
            self.id, self._s, self.tag, self.verts = fid, sides, tag, verts

        def sides(self):
            return self._s

    class Macro:
        def __init__(self, verts, m):
            self.verts, self.m = verts, m

    V = mesh.vertices
    macros = [Macro(V[row], mesh.m) for row in mesh.elem_verts]
    skel = []
    for f in range(mesh.n_face):
        fv = V[mesh.face_verts[f]]
        sides = []
        for (e, k) in (mesh.face_left[f], mesh.face_right[f]):
            if e < 0:
                continue
            a = V[mesh.elem_verts[e][[1, 2, 0][k]]]
            sides.append(Side(int(e), int(k), 0.0 if np.allclose(a, fv[0]) else 1.0))
        skel.append(Face(f, sides, str(mesh.face_tag[f]), fv))

    class Duck:
        d = 2
        macro_elements = macros
        skeleton = skel

    blk = assemble_system_device(Duck(), problem, stab, p)
    for e in range(g["A"].shape[0]):
        assert brel(blk.A[e].cpu().numpy(), g["A"][e]) <= BLOCK_TOL
    assert brel(blk.D.cpu().numpy(), g["D"]) <= BLOCK_TOL


def test_device_assembly_rejects_3d_and_missing_neumann_data():
    mesh3 = P.build_structured_macro_mesh(3, 1, 1)
    with pytest.raises(NotImplementedError):
        assemble_system_device(mesh3, tanh_problem(), StabilizationConfig(), 1)
    mesh = P.build_structured_macro_mesh(2, 2, 1, boundary_tagger=lambda x: "N")
    with pytest.raises(ValueError):
        assemble_system_device(mesh, tanh_problem(), StabilizationConfig(), 1)
