"""Pin the CPU oracle against the reference's own outputs (tests/golden)
and against the reference's counting KATs.  CPU only."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel
from oracle import mesh_oracle as MO
from oracle import solver_oracle as SO
from paper_2302_10917_b200 import synthetic as S


@pytest.mark.parametrize("n", [1, 2, 3, 4, 8])
def test_oracle_2d_skeleton_matches_reference(n):
    g = golden("skeleton_2d.npz")
    o = MO.structured_skeleton(2, n)
    for k in ("face_left", "face_right", "face_tag", "elem_verts", "elem_face", "verts"):
        assert np.array_equal(o[k], g[f"n{n}_{k}"]), k
    assert np.array_equal(o["face_left_t"], g[f"n{n}_face_left_t"])
    assert np.array_equal(o["face_right_t"], g[f"n{n}_face_right_t"])


@pytest.mark.parametrize("n", [1, 2, 3, 4])
def test_oracle_kuhn_tets_match_reference(n):
    g = golden("kuhn_3d.npz")
    verts, tets = MO.kuhn_tets(n)
    assert np.array_equal(tets, g[f"n{n}_elem_verts"])
    assert np.array_equal(verts, g[f"n{n}_verts"])


@pytest.mark.parametrize("d,n", [(2, 1), (2, 2), (2, 5), (3, 1), (3, 2), (3, 3), (3, 4)])
def test_face_count_formulas(d, n):
    """Interior faces = cost-model D (costmodel.py:53; test_mesh.py:16-50,
    test_costmodel.py:28-38); every interior face has exactly two sides and
    the left side is the lower macro id (mesh.py:235)."""
    o = MO.structured_skeleton(d, n)
    interior = int((o["face_tag"] == 0).sum())
    assert interior == MO.interior_face_count(d, n)
    boundary = int((o["face_tag"] != 0).sum())
    assert boundary == (4 * n if d == 2 else 12 * n * n)
    inner = o["face_tag"] == 0
    assert (o["face_right"][inner, 0] > o["face_left"][inner, 0]).all()
    assert (o["face_right"][~inner, 0] == -1).all()
    assert o["elem_verts"].shape[0] == (2 * n * n if d == 2 else 6 * n**3)


def test_3d_interface_faces_per_slab():
    """each x-slab interface of the Kuhn mesh has 2n^2 faces,
    left side in the lower slab."""
    for n in (2, 3, 4):
        o = MO.structured_skeleton(3, n)
        slab = 6 * n * n
        inner = o["face_tag"] == 0
        l = o["face_left"][inner, 0] // slab
        r = o["face_right"][inner, 0] // slab
        cross = l != r
        assert cross.sum() == (n - 1) * 2 * n * n
        assert (r[cross] == l[cross] + 1).all()


def _oracle_c1():
    prob = S.config_problem("c1")
    sysO = SO.system_from_problem(prob).factorize()
    return prob, sysO


def test_oracle_c1_matches_reference_outputs():
    g = golden("synthetic_c1.npz")
    prob, o = _oracle_c1()
    assert o.zhat == int(g["zhat"])
    f = o.rhs()
    assert rel(f, g["f"]) <= 1e-13
    w = o.apply(prob["uhat"])
    assert rel(w, g["w"]) <= 1e-13
    z = o.precond(w)
    assert rel(z, g["z"]) <= 1e-13
    assert np.array_equal(o.face_kind, g["face_kinds"])
    x, info = SO.gmres(o.apply, f, tol=1e-10, precond=o.precond)
    assert info["iterations"] == int(g["iterations"])
    assert rel(x, g["x"]) <= 1e-12
    U = o.reconstruct(x)
    assert rel(U[g["esel"]], g["U"]) <= 1e-12
    for k, e in enumerate(g["esel"][:8]):
        assert np.array_equal(o.lu[e][1], g["piv"][k])
        assert np.abs(o.lu[e][0] - g["lu"][k]).max() <= 1e-13 * np.abs(g["lu"][k]).max()


def test_oracle_c1_tables_match_reference():
    g = golden("synthetic_c1.npz")
    prob = S.config_problem("c1", with_blocks=False)
    o = MO.structured_skeleton(2, 8)
    tab = SO.condense_tables(o["face_tag"] == 0, o["elem_face"], o["face_left"],
                             o["face_right"], prob["t"])
    fid = np.nonzero(tab["uidx"] >= 0)[0]
    assert np.array_equal(fid, g["offsets_fid"])
    assert np.array_equal(tab["starts"], g["offsets_start"])
    assert np.array_equal(np.concatenate(tab["gather_idx"]), g["gather_idx_concat"])
    fp = []
    for f, start, nd, order in tab["face_plan"]:
        row = [f, start]
        for e, sl in order:
            row += [e, sl.start]
        row += [-1, -1] * (2 - len(order))
        fp.append(row)
    assert np.array_equal(np.array(fp), g["face_plan"])


def test_oracle_explicit_schur_matches_reference():
    g = golden("synthetic_c1.npz")
    prob, o = _oracle_c1()
    Sx = o.explicit_schur()
    for x, ref_mb, ref_mf in zip(g["mb_x"], g["mb_Sx"], g["mf_Sx"]):
        assert rel(Sx @ x, ref_mb) <= 1e-13
        assert rel(o.apply(x), ref_mf) <= 1e-13


@pytest.mark.parametrize("fx", ["real_tanh_n2m2p2.npz", "real_tanh_n3m1p3.npz"])
def test_oracle_real_hdg_blocks(fx):
    """Reference-assembled HDG blocks: pivoting LU, chol-neg faces, C != B^T."""
    g = golden(fx)
    n = int(g["n"])
    sk = MO.structured_skeleton(2, n)
    t = g["D"].shape[1]
    tab = SO.condense_tables(sk["face_tag"] == 0, sk["elem_face"], sk["face_left"],
                             sk["face_right"], t)
    assert np.array_equal(np.nonzero(tab["uidx"] >= 0)[0], g["face_ids"])
    assert np.array_equal(sk["elem_face"], g["slot_faces"])
    o = SO.OracleSystem(g["A"], g["B"], g["C"], g["R_u"], g["D"], g["R_hat"],
                        tab["elem_face"], tab["face_elem"], tab["face_slot"], t).factorize()
    assert np.array_equal(o.face_kind, g["face_kinds"])
    for e in range(o.N):
        assert np.array_equal(o.lu[e][1], g["piv"][e])
    assert rel(o.rhs(), g["f"]) <= 1e-13
    for x, w, z in zip(g["xs"], g["w"], g["z"]):
        assert rel(o.apply(x), w) <= 1e-12
        assert rel(o.precond(x), z) <= 1e-12
    x, info = SO.gmres(o.apply, o.rhs(), tol=1e-12, precond=o.precond)
    assert info["iterations"] == int(g["iterations"])
    assert rel(x, g["x"]) <= 1e-10
    assert rel(o.reconstruct(x), g["U"]) <= 1e-10


def test_oracle_gmres_kats():
    """schur_solver KATs (test_schur_solver.py:205-230)."""
    x, info = SO.gmres(lambda v: v, np.array([3.0, -1.0, 2.0]), tol=1e-12)
    assert info["converged"] and info["iterations"] == 1
    d = np.arange(1.0, 6.0)
    x, info = SO.gmres(lambda v: d * v, np.ones(5), tol=1e-12)
    assert info["converged"] and info["iterations"] <= 5
    assert np.abs(x - 1.0 / d).max() < 1e-10
    d = np.arange(1.0, 101.0)
    x, info = SO.gmres(lambda v: d * v, np.ones(100), tol=1e-14, maxiter=3, restart=3)
    assert not info["converged"] and info["iterations"] == 3
    x, info = SO.gmres(lambda v: 2 * v, np.zeros(4))
    assert info["converged"] and np.abs(x).max() == 0.0


def test_oracle_singular_blocks():
    prob = S.make_problem(2, 1, 1, 1)
    A = prob["A"].copy()
    A[1] = 0.0
    o = SO.OracleSystem(A, prob["B"], prob["C"], prob["R_u"], prob["D"], prob["R_hat"],
                        prob["elem_face"], prob["face_elem"], prob["face_slot"], prob["t"])
    with pytest.raises(SO.SingularLocalBlock) as ei:
        o.factorize()
    assert ei.value.args[0] == 1
    D = prob["D"].copy()
    D[0] = 0.0
    o = SO.OracleSystem(prob["A"], prob["B"], prob["C"], prob["R_u"], D, prob["R_hat"],
                        prob["elem_face"], prob["face_elem"], prob["face_slot"], prob["t"])
    with pytest.raises(SO.SingularFaceBlock):
        o.factorize()


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_generator_and_tables_match_reference_run(name):
    """The seeded generator + tables reproduce the inputs the reference was run
    on (checked through the reference's condense tables and f checksum)."""
    g = golden(f"synthetic_{name}.npz")
    prob = S.config_problem(name, with_blocks=False)
    assert prob["zhat"] == int(g["zhat"])
    fid = np.nonzero(prob["uidx"] >= 0)[0]
    assert np.array_equal(fid, g["offsets_fid"])
    assert np.array_equal(fid.size, g["face_plan"].shape[0])
    fe, fs = prob["face_elem"], prob["face_slot"]
    t = prob["t"]
    plan = np.stack([fid, np.arange(fid.size) * t, fe[:, 0], fs[:, 0] * t,
                     fe[:, 1], np.where(fe[:, 1] >= 0, fs[:, 1] * t, -1)], axis=1)
    assert np.array_equal(plan, g["face_plan"])
