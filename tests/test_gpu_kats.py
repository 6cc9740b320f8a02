"""The reference's relational checks (tests/test_schur_solver.py
and tests/test_acceptance.py of mehdg) restated on blocks assembled on the device:
MF vs explicit Schur, symmetry for pure diffusion, explicit-Schur adjacency,
full-system residual, D^-1 round trip, linearity."""

from __future__ import annotations

import numpy as np
import pytest

import paper_2302_10917_b200 as P
from paper_2302_10917_b200.assembly import (ProblemData, StabilizationConfig,
                                            assemble_system_device, manufactured_tanh)

pytestmark = pytest.mark.gpu


def condensed(n, m, p, problem, stab=None):
    mesh = P.build_structured_macro_mesh(2, n, m)
    blk = assemble_system_device(mesh, problem, stab or StabilizationConfig(), p)
    sys_ = P.condense_arrays(mesh, blk.A, blk.B, blk.C, blk.R_u, blk.D, blk.R_hat,
                             P.SolverConfig(tol=1e-12), p=p, tables=blk.tables)
    return mesh, blk, sys_


def diffusion():
    return ProblemData(a=np.zeros(2), kappa=1.0, f=lambda x: np.ones(np.atleast_2d(x).shape[0]),
                       g_D=lambda x: np.zeros(np.atleast_2d(x).shape[0]))


@pytest.mark.parametrize("n,m,p", [(3, 2, 2), (4, 1, 3)])
def test_matrix_free_equals_explicit_schur(n, m, p):
    """criterion 2 (tests/test_acceptance.py:71-89): 20 random x, seed 42."""
    _, _, sys_ = condensed(n, m, p, manufactured_tanh())
    S = P.assemble_schur_explicit(sys_)
    rng = np.random.default_rng(42)
    for _ in range(20):
        x = rng.standard_normal(sys_.zhat)
        mb = S @ x
        assert np.linalg.norm(P.apply_schur(sys_, x) - mb) <= 1e-10 * np.linalg.norm(mb)


def test_symmetric_for_pure_diffusion():
    """a = 0 gives a symmetric trace system (tests/test_schur_solver.py:271-275)."""
    _, _, sys_ = condensed(3, 2, 2, diffusion())
    S = P.assemble_schur_explicit(sys_).toarray()
    assert np.abs(S - S.T).max() <= 1e-12 * np.abs(S).max()


def test_explicit_schur_adjacency():
    """S couples two faces only through a shared macro (tests/test_schur_solver.py:257-268)."""
    mesh, _, sys_ = condensed(3, 1, 2, manufactured_tanh())
    S = abs(P.assemble_schur_explicit(sys_).toarray()) > 0
    t = sys_.t
    uidx = sys_.tables["uidx"]
    share = np.eye(sys_.F, dtype=bool)
    for e in range(mesh.n_elem):
        us = [uidx[f] for f in mesh.elem_face[e] if uidx[f] >= 0]
        for a in us:
            for b in us:
                share[a, b] = True
    blocks = S.reshape(sys_.F, t, sys_.F, t).any(axis=(1, 3))
    assert not (blocks & ~share).any()
    assert blocks[np.eye(sys_.F, dtype=bool)].all()


def test_full_system_residual():
    """After the solve, [A B; C D] [u; uhat] = [R_u; R_hat] block by block
    (tests/test_schur_solver.py:308-322)."""
    mesh, blk, sys_ = condensed(3, 2, 2, manufactured_tanh())
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, P.SolverConfig(tol=1e-13),
                      precond=P.Preconditioner(sys_))
    assert info["converged"]
    U = np.stack(P.reconstruct_interior(sys_, x))
    A, B, Cm = (v.cpu().numpy() for v in (blk.A, blk.B, blk.C))
    Ru, D, Rh = blk.R_u.cpu().numpy(), blk.D.cpu().numpy(), blk.R_hat.cpu().numpy()
    t = sys_.t
    ef = sys_.tables["elem_ufac"]
    face_res = -Rh.copy()
    for e in range(mesh.n_elem):
        ue = np.zeros(B.shape[2])
        for k, u in enumerate(ef[e]):
            if u >= 0:
                ue[k * t:(k + 1) * t] = x[u * t:(u + 1) * t]
        r = A[e] @ U[e] + B[e] @ ue - Ru[e]
        assert np.linalg.norm(r) <= 1e-10 * (np.linalg.norm(Ru[e]) + np.linalg.norm(A[e] @ U[e]))
        cu = Cm[e] @ U[e]
        for k, u in enumerate(ef[e]):
            if u >= 0:
                face_res[u] += cu[k * t:(k + 1) * t]
    for u in range(sys_.F):
        face_res[u] += D[u] @ x[u * t:(u + 1) * t]
    assert np.abs(face_res).max() <= 1e-9 * max(np.abs(Rh).max(), np.abs(D).max() * np.abs(x).max())


def test_dinv_round_trip_on_assembled_faces():
    """D^-1 (D x) = x (tests/test_schur_solver.py:127-135); the assembled D blocks are
    negative definite, so the factor kind is the reference's chol-neg."""
    _, blk, sys_ = condensed(3, 2, 2, manufactured_tanh())
    assert set(sys_.face_kinds.tolist()) == {0}
    D = blk.D.cpu().numpy()
    t = sys_.t
    rng = np.random.default_rng(1)
    x = rng.standard_normal(sys_.zhat)
    Dx = np.concatenate([D[u] @ x[u * t:(u + 1) * t] for u in range(sys_.F)])
    assert np.abs(P.apply_preconditioner(sys_, Dx) - x).max() <= 1e-12 * np.abs(x).max() * 10


def test_linearity():
    """tests/test_schur_solver.py:93-101 and :353-367."""
    _, _, sys_ = condensed(3, 2, 2, manufactured_tanh())
    rng = np.random.default_rng(7)
    x, y = rng.standard_normal((2, sys_.zhat))
    a, b = 2.5, -0.75
    lhs = P.apply_schur(sys_, a * x + b * y)
    rhs = a * P.apply_schur(sys_, x) + b * P.apply_schur(sys_, y)
    assert np.linalg.norm(lhs - rhs) <= 1e-10 * np.linalg.norm(rhs)
    assert np.array_equal(P.apply_schur(sys_, np.zeros(sys_.zhat)), np.zeros(sys_.zhat))
