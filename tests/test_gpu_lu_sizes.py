"""Batched LU across block sizes: every tile-LU instantiation (8-row tile counts
6..32, including sizes that round up to a padded tile count) against
scipy.linalg.lu_factor (LAPACK getrf) on pivoting Gaussian blocks, plus the
apply through those factors against the oracle."""

from __future__ import annotations

import numpy as np
import pytest
import scipy.linalg as sla

import paper_2302_10917_b200 as P
from paper_2302_10917_b200 import synthetic as S
from oracle import solver_oracle as SO
from conftest import rel

pytestmark = pytest.mark.gpu

SIZES = [16, 32, 33, 40, 57, 64, 65, 80, 88, 91, 96, 97, 112, 120, 128, 129, 144, 160, 165,
         168, 190, 200, 220, 224, 250, 256]


def problem_with_blocks(Q, seed):
    """The smallest mesh (2 macros, t = 2) carrying Q x Q Gaussian blocks."""
    prob = S.make_problem(2, 1, 1, 1, seed=seed)
    rng = np.random.default_rng(seed)
    N, nc = prob["N"], prob["nc"]
    prob["Q"] = Q
    prob["A"] = rng.standard_normal((N, Q, Q))
    prob["Be"] = rng.standard_normal((N, nc, Q))
    prob["B"] = prob["Be"].transpose(0, 2, 1)
    prob["C"] = prob["Be"]
    prob["R_u"] = rng.standard_normal((N, Q))
    return prob


@pytest.mark.parametrize("Q", SIZES)
def test_lu_matches_lapack_across_sizes(Q, lu_kernel):
    if lu_kernel == "cta" and not 32 < Q <= 168:
        pytest.skip("the CTA-resident LU covers 32 < Q <= 168")
    if lu_kernel == "pipe" and not 32 < Q <= 224:
        pytest.skip("the pipelined LU covers 32 < Q <= 224")
    prob = problem_with_blocks(Q, seed=100 + Q)
    tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
              "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
    sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
    lu, piv = P.local_factors(sys_)
    for e in range(prob["N"]):
        ref_lu, ref_piv = sla.lu_factor(prob["A"][e])
        assert np.array_equal(piv[e], ref_piv), (Q, e)
        assert np.abs(lu[e] - ref_lu).max() <= 1e-11 * np.abs(ref_lu).max(), (Q, e)
    o = SO.system_from_problem(prob).factorize()
    u = np.random.default_rng(Q).standard_normal(sys_.zhat)
    assert rel(P.apply_schur(sys_, u), o.apply(u)) <= 1e-10


def test_staged_upload_large_blocks():
    """Block arrays above the pinned-staging threshold (32 MB: the threaded,
    chunked host -> device path of mh_upload_blocks) arrive intact: factors of
    sampled macro match LAPACK and the apply matches the oracle on a mesh whose
    A (217 MB) and op.C (51 MB, the pitched path) are not multiples of the 4 MB
    chunks or of the per-thread slices."""
    d, n, m, p = 2, 32, 2, 4  # N = 2048 macros, nc = 27
    prob = S.make_problem(d, n, m, p, seed=17)
    rng = np.random.default_rng(17)
    N, Q, nc = prob["N"], prob["Q"], prob["nc"]
    Qb = 115  # larger blocks
    prob["Q"] = Qb
    prob["A"] = rng.standard_normal((N, Qb, Qb)) + Qb * np.eye(Qb)
    prob["Be"] = rng.standard_normal((N, nc, Qb))
    prob["B"] = prob["Be"].transpose(0, 2, 1)
    prob["C"] = prob["Be"]
    prob["R_u"] = rng.standard_normal((N, Qb))
    assert prob["A"].nbytes > 32 << 20 and prob["Be"].nbytes > 32 << 20
    tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
              "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
    sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
    lu, piv = P.local_factors(sys_)
    for e in range(0, N, 37):
        ref_lu, ref_piv = sla.lu_factor(prob["A"][e])
        assert np.array_equal(piv[e], ref_piv), e
        assert np.abs(lu[e] - ref_lu).max() <= 1e-11 * np.abs(ref_lu).max(), e
    o = SO.system_from_problem(prob).factorize()
    u = np.random.default_rng(3).standard_normal(sys_.zhat)
    assert rel(P.apply_schur(sys_, u), o.apply(u)) <= 1e-12


MB_SIZES = [24, 40, 64, 91, 97, 128, 165, 190, 220, 250, 256]


@pytest.mark.parametrize("Q", MB_SIZES)
def test_element_schur_dmma_across_sizes(Q):
    """Every form_dmma_kernel instantiation (8-row tile counts 4..32; 250 / 256 stage
    -L / -U in two chunks) on pivoting Gaussian blocks: S_e = C A^-1 B against
    numpy, and the matrix-based apply (TMA-streamed) against the matrix-free one."""
    prob = problem_with_blocks(Q, seed=300 + Q)
    tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
              "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
    sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
    P.form_element_schur(sys_)
    from paper_2302_10917_b200._lib import lib, ptr, check
    N, nc = prob["N"], prob["nc"]
    blocks = np.empty((N, nc, nc))
    check(lib.mh_get_element_schur(sys_.handle, 0, N, ptr(blocks)))
    for e in range(N):
        ref = -(prob["Be"][e] @ np.linalg.solve(prob["A"][e], prob["Be"][e].T))
        assert np.abs(blocks[e] - ref).max() <= 1e-10 * np.abs(ref).max(), (Q, e)
    u = np.random.default_rng(Q).standard_normal(sys_.zhat)
    assert rel(P.apply_schur_mb(sys_, u), P.apply_schur(sys_, u)) <= 1e-10


@pytest.mark.parametrize("d,n,m,p", [(3, 1, 2, 4), (3, 1, 3, 3), (2, 3, 4, 3)])
@pytest.mark.parametrize("stream", ["1", "0"])
def test_mb_apply_matches_mf_baseline_shapes(d, n, m, p, stream, monkeypatch):
    """The BASELINE block shapes with many right-hand-side tile columns (c5: Q = 165,
    nc = 180; c4: Q = 220, nc = 220; c2: Q = 91, nc = 39), diagonally dominant: the
    matrix-based apply through the TMA stream and through plain loads both equal the
    matrix-free apply and the oracle to 1e-12."""
    monkeypatch.setenv("MEHDG_MB_STREAM", stream)
    prob = S.make_problem(d, n, m, p, seed=11)
    tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
              "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
    sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
    P.form_element_schur(sys_)
    o = SO.system_from_problem(prob).factorize()
    w = P.apply_schur_mb(sys_, prob["uhat"])
    assert rel(w, o.apply(prob["uhat"])) <= 1e-12
    assert rel(w, P.apply_schur(sys_, prob["uhat"])) <= 1e-12
