"""GPU parity: the CUDA path (through the C-ABI) against the reference's own
outputs (tests/golden) and the CPU oracle, on identical seeded inputs.

Tolerances (BASELINE north_star): integer tables bit-exact; operator apply,
RHS, preconditioner and factors <= 1e-12 relative; converged uhat / u
<= 1e-9 relative; GMRES iteration counts within +-1."""

from __future__ import annotations

import numpy as np
import pytest

from conftest import golden, rel
from oracle import solver_oracle as SO
import paper_2302_10917_b200 as P
from paper_2302_10917_b200 import synthetic as S

pytestmark = pytest.mark.gpu

APPLY_TOL = 1e-12
SOLVE_TOL = 1e-9


def condense_problem(prob, **kw):
    cfg = P.SolverConfig(tol=kw.pop("tol", 1e-10))
    tables = {"nfe": prob["d"] + 1, "elem_ufac": prob["elem_face"],
              "face_elem": prob["face_elem"], "face_slot": prob["face_slot"],
              "uidx": prob["uidx"], "F": prob["F"]}
    return P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"], prob["D"],
                             prob["R_hat"], cfg, tables=tables, **kw), cfg


@pytest.fixture(scope="module")
def c1(gpu):
    prob = S.config_problem("c1")
    sys_, cfg = condense_problem(prob)
    return prob, sys_, cfg


def test_c1_factors_match_reference(c1):
    prob, sys_, _ = c1
    g = golden("synthetic_c1.npz")
    lu, piv = P.local_factors(sys_)
    for k, e in enumerate(g["esel"][:8]):
        assert np.array_equal(piv[e], g["piv"][k])
        assert np.abs(lu[e] - g["lu"][k]).max() <= APPLY_TOL * np.abs(g["lu"][k]).max()
    assert np.array_equal(sys_.face_kinds, g["face_kinds"])


def test_c1_rhs_apply_precond_match_reference(c1):
    prob, sys_, _ = c1
    g = golden("synthetic_c1.npz")
    assert sys_.zhat == int(g["zhat"])
    assert rel(sys_.f_vec, g["f"]) <= APPLY_TOL
    w = P.apply_schur(sys_, prob["uhat"])
    assert rel(w, g["w"]) <= APPLY_TOL
    z = P.apply_preconditioner(sys_, w)
    assert rel(z, g["z"]) <= APPLY_TOL
    for x, ref in zip(g["mb_x"], g["mf_Sx"]):
        assert rel(P.apply_schur(sys_, x), ref) <= APPLY_TOL


def test_c1_gmres_and_reconstruct_match_reference(c1):
    prob, sys_, cfg = c1
    g = golden("synthetic_c1.npz")
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, cfg, precond=P.Preconditioner(sys_))
    assert info["converged"]
    assert abs(info["iterations"] - int(g["iterations"])) <= 1
    assert rel(x, g["x"]) <= SOLVE_TOL
    hist = np.array(info["residual_history"])
    n = min(hist.size, g["history"].size)
    assert np.allclose(hist[:n], g["history"][:n], rtol=1e-6)
    U = np.stack(P.reconstruct_interior(sys_, x))
    assert rel(U[g["esel"]], g["U"]) <= SOLVE_TOL


def test_c1_explicit_schur_matches_reference(c1):
    prob, sys_, _ = c1
    g = golden("synthetic_c1.npz")
    S_csr = P.assemble_schur_explicit(sys_)
    for x, ref in zip(g["mb_x"], g["mb_Sx"]):
        assert rel(S_csr @ x, ref) <= APPLY_TOL
        assert rel(P.apply_schur_mb(sys_, x), ref) <= APPLY_TOL


def test_apply_deterministic_and_linear(c1):
    prob, sys_, _ = c1
    rng = np.random.default_rng(0)
    x, y = rng.standard_normal((2, sys_.zhat))
    w1 = P.apply_schur(sys_, x)
    w2 = P.apply_schur(sys_, x)
    assert np.array_equal(w1, w2)
    assert np.abs(P.apply_schur(sys_, np.zeros(sys_.zhat))).max() == 0.0
    lhs = P.apply_schur(sys_, 2 * x + 3 * y)
    rhs = 2 * w1 + 3 * P.apply_schur(sys_, y)
    assert np.abs(lhs - rhs).max() < 1e-10 * max(1.0, np.abs(rhs).max())


def test_apply_schur_many_matches_single_applies(c1):
    """mh_apply_host_many (copies overlapped with the applies) is bitwise the
    per-vector apply, for a stack of vectors and for the repeat form."""
    _, sys_, _ = c1
    rng = np.random.default_rng(4)
    U = rng.standard_normal((5, sys_.zhat))
    W = P.apply_schur_many(sys_, U)
    for i in range(5):
        assert np.array_equal(W[i], P.apply_schur(sys_, U[i]))
    w1 = P.apply_schur_many(sys_, U[2].copy(), repeat=7)
    assert np.array_equal(w1, W[2])
    assert P.apply_schur_many(sys_, U[:0]).shape == (0, sys_.zhat)
    with pytest.raises(ValueError):
        P.apply_schur_many(sys_, U[:, :-1])


def test_device_tensor_path_matches_host_path(c1):
    import torch

    prob, sys_, _ = c1
    u = torch.as_tensor(prob["uhat"], device="cuda")
    w_dev = P.apply_schur(sys_, u)
    assert w_dev.is_cuda
    assert np.array_equal(w_dev.cpu().numpy(), P.apply_schur(sys_, prob["uhat"]))


@pytest.mark.parametrize("fx", ["real_tanh_n2m2p2.npz", "real_tanh_n3m1p3.npz"])
def test_reference_assembled_blocks(gpu, fx):
    """Real HDG blocks from the reference assembly: pivoting LU, C != B^T,
    chol-neg faces -- through the drop-in condense on LocalOperators."""
    g = golden(fx)
    n, m = int(g["n"]), int(g["m"])
    mesh = P.build_structured_macro_mesh(2, n, m)
    t = g["D"].shape[1]
    local_ops = [P.LocalOperators(macro_id=e, A=g["A"][e], B=g["B"][e], C=g["C"][e],
                                  R_u=g["R_u"][e],
                                  face_slots=[(int(f), slice(k * t, (k + 1) * t))
                                              for k, f in enumerate(g["slot_faces"][e])])
                 for e in range(g["A"].shape[0])]
    face_ops = {int(f): P.FaceOperator(face_id=int(f), D=g["D"][i], R_hat=g["R_hat"][i])
                for i, f in enumerate(g["face_ids"])}
    cfg = P.SolverConfig(tol=1e-12)
    sys_ = P.condense(mesh, local_ops, face_ops, cfg)
    assert {face_ops[int(f)].factor_kind for f in g["face_ids"]} == \
        {_kind(k) for k in g["face_kinds"]}
    lu, piv = P.local_factors(sys_)
    assert np.array_equal(piv, g["piv"])
    assert np.abs(lu - g["lu"]).max() <= APPLY_TOL * np.abs(g["lu"]).max()
    assert rel(sys_.f_vec, g["f"]) <= APPLY_TOL
    for x, w, z in zip(g["xs"], g["w"], g["z"]):
        assert rel(P.apply_schur(sys_, x), w) <= APPLY_TOL
        assert rel(P.apply_preconditioner(sys_, x), z) <= APPLY_TOL
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, cfg, precond=P.Preconditioner(sys_))
    assert abs(info["iterations"] - int(g["iterations"])) <= 1
    assert rel(x, g["x"]) <= SOLVE_TOL
    U = np.stack(P.reconstruct_interior(sys_, x))
    assert rel(U, g["U"]) <= SOLVE_TOL


def _kind(k):
    return {0: "chol-neg", 1: "chol-pos", 2: "lu"}[int(k)]


@pytest.mark.parametrize("d,n,m,p", [(2, 4, 4, 3), (2, 3, 2, 5), (3, 2, 2, 3), (3, 2, 1, 4),
                                     (3, 1, 3, 3), (2, 2, 3, 6), (3, 1, 2, 4), (3, 2, 2, 4)])
def test_against_oracle_small(gpu, d, n, m, p, lu_kernel):
    """Each BASELINE block shape family (Q = 15..220; c5's Q = 165, t = 45 on one and
    on eight cubes) against the oracle, diagonally dominant as in BASELINE."""
    prob = S.make_problem(d, n, m, p, seed=7)
    sys_, cfg = condense_problem(prob)
    o = SO.system_from_problem(prob).factorize()
    assert rel(sys_.f_vec, o.rhs()) <= APPLY_TOL
    w = P.apply_schur(sys_, prob["uhat"])
    assert rel(w, o.apply(prob["uhat"])) <= APPLY_TOL
    assert rel(P.apply_preconditioner(sys_, w), o.precond(w)) <= APPLY_TOL
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, cfg, precond=P.Preconditioner(sys_))
    xo, io = SO.gmres(o.apply, o.rhs(), tol=1e-10, precond=o.precond)
    assert abs(info["iterations"] - io["iterations"]) <= 1
    assert rel(x, xo) <= SOLVE_TOL
    assert rel(np.stack(P.reconstruct_interior(sys_, x)), o.reconstruct(xo)) <= SOLVE_TOL
    lu, piv = P.local_factors(sys_, 0, min(4, prob["N"]))
    for e in range(lu.shape[0]):
        assert np.array_equal(piv[e], o.lu[e][1])
        assert np.abs(lu[e] - o.lu[e][0]).max() <= APPLY_TOL * np.abs(o.lu[e][0]).max()


def test_pivoting_blocks(gpu):
    """Blocks that need row interchanges (no diagonal dominance)."""
    prob = S.make_problem(2, 3, 2, 2, seed=11)
    rng = np.random.default_rng(5)
    prob["A"] = rng.standard_normal(prob["A"].shape)
    sys_, cfg = condense_problem(prob)
    o = SO.system_from_problem(prob).factorize()
    lu, piv = P.local_factors(sys_)
    swaps = 0
    for e in range(prob["N"]):
        assert np.array_equal(piv[e], o.lu[e][1])
        swaps += int((piv[e] != np.arange(prob["Q"])).sum())
    assert swaps > 0
    assert rel(P.apply_schur(sys_, prob["uhat"]), o.apply(prob["uhat"])) <= 1e-11


@pytest.mark.parametrize("d,n,m,p", [(2, 2, 4, 2), (2, 2, 4, 3), (3, 1, 3, 2), (3, 1, 7, 1),
                                     (3, 1, 2, 4), (3, 1, 3, 3)])
@pytest.mark.parametrize("kind", ["gauss", "ties"])
def test_pivoting_blocks_tile_lu(gpu, d, n, m, p, kind, lu_kernel):
    """Row interchanges in the tile LU (Q = 45, 91, 84, 120 (padded tile), 165, 220):
    LAPACK pivots bit-exact, including first-index ties (small-integer blocks)."""
    prob = S.make_problem(d, n, m, p, seed=13)
    rng = np.random.default_rng(17)
    if kind == "gauss":
        prob["A"] = rng.standard_normal(prob["A"].shape)
    else:
        prob["A"] = rng.integers(-3, 4, prob["A"].shape).astype(np.float64)
    sys_, cfg = condense_problem(prob)
    o = SO.system_from_problem(prob).factorize()
    lu, piv = P.local_factors(sys_)
    swaps = 0
    for e in range(prob["N"]):
        assert np.array_equal(piv[e], o.lu[e][1])
        assert np.abs(lu[e] - o.lu[e][0]).max() <= 1e-11 * np.abs(o.lu[e][0]).max()
        swaps += int((piv[e] != np.arange(prob["Q"])).sum())
    assert swaps > 0
    assert rel(P.apply_schur(sys_, prob["uhat"]), o.apply(prob["uhat"])) <= 1e-10


def test_singular_local_block_raises_with_id(gpu):
    prob = S.make_problem(2, 2, 1, 1)
    prob["A"] = prob["A"].copy()
    prob["A"][5] = 0.0
    prob["A"][6] = 0.0
    with pytest.raises(P.SingularLocalBlock) as ei:
        condense_problem(prob)
    assert ei.value.args[0] == 5


@pytest.mark.parametrize("which", ["zero", "repeated_row"])
def test_singular_local_block_tile_lu(gpu, which, lu_kernel):
    """Tile LU (Q = 91): the singular test min|U_jj| <= 1e-13 max|A| reports the first
    singular macro; a zero pivot skips the exchange and scaling (dgetf2 info > 0)."""
    prob = S.make_problem(2, 2, 4, 3, seed=3)
    prob["A"] = prob["A"].copy()
    if which == "zero":
        prob["A"][3] = 0.0
        bad = 3
    else:
        prob["A"][5][7] = prob["A"][5][2]
        bad = 5
    with pytest.raises(P.SingularLocalBlock) as ei:
        condense_problem(prob)
    assert ei.value.args[0] == bad


def test_singular_threshold_exact_at_the_boundary(gpu):
    """min|U_jj| <= 1e-13 max|A| decided exactly when it is within the kernel's
    high-word bound on max|A| (the exact re-read path): block 2 sits on the
    threshold (singular), block 1 one ulp above it (regular)."""
    prob = S.make_problem(2, 2, 4, 3, seed=3)
    Q = prob["Q"]
    A = np.repeat(np.eye(Q)[None], prob["N"], axis=0)
    M = 1.9999999999  # low word of the bit pattern far from 0 and from 0xffffffff
    for e in (1, 2):
        A[e, 0, 0] = M
    A[2, 5, 5] = 1e-13 * M
    A[1, 5, 5] = np.nextafter(1e-13 * M, 1.0)
    prob["A"] = A
    with pytest.raises(P.SingularLocalBlock) as ei:
        condense_problem(prob)
    assert ei.value.args[0] == 2


def test_singular_face_block_raises(gpu):
    prob = S.make_problem(2, 2, 1, 1)
    prob["D"] = prob["D"].copy()
    prob["D"][2] = 0.0
    with pytest.raises(P.SingularFaceBlock) as ei:
        condense_problem(prob)
    assert ei.value.args[0] == 2


def test_indefinite_face_block_uses_lu(gpu):
    prob = S.make_problem(2, 2, 2, 2, seed=3)
    prob["D"] = prob["D"].copy()
    prob["D"][0] = np.diag(np.r_[1.0, -2.0, 3.0, -4.0, 5.0]) + 0.1
    sys_, _ = condense_problem(prob)
    assert sys_.face_kinds[0] == 2
    o = SO.system_from_problem(prob).factorize()
    w = np.random.default_rng(1).standard_normal(sys_.zhat)
    assert rel(P.apply_preconditioner(sys_, w), o.precond(w)) <= APPLY_TOL


def test_two_macro_mesh_counts(gpu):
    """test_schur_solver.py:116-124: one apply = 2 macro tasks + 1 face reduction."""
    prob = S.make_problem(2, 1, 1, 1)
    sys_, _ = condense_problem(prob)
    assert sys_.zhat == 2
    sys_.counters["macro_apply"] = sys_.counters["face_reduce"] = 0
    P.apply_schur(sys_, np.ones(2))
    assert sys_.counters == {"macro_apply": 2, "face_reduce": 1}


def test_gmres_kats_through_callbacks(gpu):
    """test_schur_solver.py:205-230 with Python operators (mh_gmres_op)."""
    cfg = P.SolverConfig(tol=1e-12)
    x, info = P.gmres(lambda v: v, np.array([3.0, -1.0, 2.0]), cfg)
    assert info["converged"] and info["iterations"] == 1
    assert np.abs(x - [3.0, -1.0, 2.0]).max() < 1e-12
    d = np.arange(1.0, 6.0)
    x, info = P.gmres(lambda v: d * v, np.ones(5), cfg)
    assert info["converged"] and info["iterations"] <= 5
    assert np.abs(x - 1.0 / d).max() < 1e-10
    d = np.arange(1.0, 101.0)
    x, info = P.gmres(lambda v: d * v, np.ones(100), P.SolverConfig(tol=1e-14, maxiter=3, restart=3))
    assert not info["converged"] and info["iterations"] == 3
    assert len(info["residual_history"]) >= 2
    x, info = P.gmres(lambda v: 2 * v, np.zeros(4), P.SolverConfig())
    assert info["converged"] and np.abs(x).max() == 0.0


def test_gmres_python_operator_equals_bound_operator(c1):
    prob, sys_, cfg = c1
    x1, i1 = P.gmres(P.SchurOperator(sys_), sys_.f_vec, cfg, precond=P.Preconditioner(sys_))
    x2, i2 = P.gmres(lambda v: P.apply_schur(sys_, v), sys_.f_vec, cfg,
                     precond=lambda v: P.apply_preconditioner(sys_, v))
    assert i1["iterations"] == i2["iterations"]
    assert rel(x1, x2) <= 1e-12


@pytest.mark.parametrize("name", ["c2", "c3"])
def test_full_config_against_reference_samples(gpu, name):
    """BASELINE c2 / c3 at full size vs the reference run (strided samples
    and whole-vector checksums), plus size-independent properties."""
    g = golden(f"synthetic_{name}.npz")
    prob = S.config_problem(name)
    sys_, cfg = condense_problem(prob)
    sel = g["sel"]
    f = sys_.f_vec
    assert rel(f[sel], g["f"]) <= APPLY_TOL
    assert abs(np.linalg.norm(f) - float(g["f_norm"])) <= APPLY_TOL * float(g["f_norm"])
    w = P.apply_schur(sys_, prob["uhat"])
    assert rel(w[sel], g["w"]) <= APPLY_TOL
    assert abs(np.linalg.norm(w) - float(g["w_norm"])) <= APPLY_TOL * float(g["w_norm"])
    z = P.apply_preconditioner(sys_, w)
    assert rel(z[sel], g["z"]) <= APPLY_TOL
    x, info = P.gmres(P.SchurOperator(sys_), sys_.f_device, cfg, precond=P.Preconditioner(sys_))
    assert info["converged"]
    assert abs(info["iterations"] - int(g["iterations"])) <= 1
    xh = x.cpu().numpy()
    assert rel(xh[sel], g["x"]) <= SOLVE_TOL
    U = P.reconstruct_interior(sys_, x).cpu().numpy()
    assert rel(U[g["esel"]], g["U"]) <= SOLVE_TOL
    # the converged residual, through the operator itself
    r = P.apply_preconditioner(sys_, sys_.f_vec - P.apply_schur(sys_, xh))
    assert np.linalg.norm(r) <= 10 * cfg.tol * np.linalg.norm(P.apply_preconditioner(sys_, sys_.f_vec))
    # bitwise determinism at full size
    assert np.array_equal(w, P.apply_schur(sys_, prob["uhat"]))


def test_mb_mode_solve_matches_mf(c1):
    """Criterion 4 (test_acceptance.py:122-135): matrix-based and matrix-free
    paths agree in iterations (+-1) and solution."""
    prob, sys_, _ = c1
    cfg_mf = P.SolverConfig(tol=1e-10, mode="mf")
    cfg_mb = P.SolverConfig(tol=1e-10, mode="mb")
    s_mf, _ = P.solve_condensed(sys_, cfg_mf)
    s_mb, _ = P.solve_condensed(sys_, cfg_mb)
    assert abs(s_mf.report.iterations - s_mb.report.iterations) <= 1
    assert rel(s_mb.uhat, s_mf.uhat) <= SOLVE_TOL
    rec = s_mb.report.to_record()
    assert rec["mode"] == "mb" and rec["converged"] is True
    assert rec["dof_global"] == sys_.zhat


def test_element_schur_blocks_match_oracle(gpu):
    """-S_e = -(C A^-1 B) per macro vs the oracle's explicit block (masked)."""
    prob = S.make_problem(3, 2, 2, 3, seed=2)
    sys_, _ = condense_problem(prob)
    P.form_element_schur(sys_)
    from paper_2302_10917_b200._lib import lib, ptr, check
    nc = prob["nc"]
    blocks = np.empty((prob["N"], nc, nc))
    check(lib.mh_get_element_schur(sys_.handle, 0, prob["N"], ptr(blocks)))
    o = SO.system_from_problem(prob).factorize()
    import scipy.linalg as sla
    for e in range(prob["N"]):
        ref = -(o.C[e] @ sla.lu_solve(o.lu[e], o.B[e]))
        assert np.abs(blocks[e] - ref).max() <= APPLY_TOL * np.abs(ref).max()


def test_preconditioner_round_trip(c1):
    """test_schur_solver.py:127-135: D^-1 (D x) = x to 1e-12."""
    prob, sys_, _ = c1
    x = np.random.default_rng(1).standard_normal(sys_.zhat)
    t = prob["t"]
    w = np.concatenate([prob["D"][u] @ x[u * t:(u + 1) * t] for u in range(prob["F"])])
    back = P.apply_preconditioner(sys_, w)
    assert np.abs(back - x).max() < 1e-12 * max(1.0, np.abs(x).max())


def test_host_factors_and_solve_driver(gpu):
    """condense(host_factors=True) fills op.lu like the reference; solve() with an
    assemble callable runs condense -> GMRES -> reconstruct and reports."""
    g = golden("real_tanh_n2m2p2.npz")
    n, m, p = int(g["n"]), int(g["m"]), int(g["p"])
    mesh = P.build_structured_macro_mesh(2, n, m)
    t = g["D"].shape[1]

    def assemble(mesh_, problem, stab, p_):
        local_ops = [P.LocalOperators(macro_id=e, A=g["A"][e], B=g["B"][e], C=g["C"][e],
                                      R_u=g["R_u"][e],
                                      face_slots=[(int(f), slice(k * t, (k + 1) * t))
                                                  for k, f in enumerate(g["slot_faces"][e])])
                     for e in range(g["A"].shape[0])]
        face_ops = {int(f): P.FaceOperator(face_id=int(f), D=g["D"][i], R_hat=g["R_hat"][i])
                    for i, f in enumerate(g["face_ids"])}
        return local_ops, face_ops

    lops, fops = assemble(mesh, None, None, p)
    sys_ = P.condense(mesh, lops, fops, P.SolverConfig(tol=1e-12), host_factors=True)
    for e, op in enumerate(lops):
        assert op.lu[0] == "dense"
        assert np.array_equal(op.lu[1][1], g["piv"][e])
        assert np.abs(op.lu[1][0] - g["lu"][e]).max() <= 1e-12 * np.abs(g["lu"][e]).max()
    sol, sys2 = P.solve(mesh, None, None, P.SolverConfig(tol=1e-12), p, assemble=assemble)
    rec = sol.report.to_record()
    assert rec["converged"] and abs(rec["iterations"] - int(g["iterations"])) <= 1
    # the local/global split of the solve time (schur_solver.py:518-535): the
    # element kernels' event time, and the rest of GMRES
    assert 0.0 < rec["t_local_s"] and rec["t_global_s"] >= 0.0
    assert rel(sol.uhat, g["x"]) <= SOLVE_TOL
    assert rel(np.stack(sol.local), g["U"]) <= SOLVE_TOL


@pytest.mark.parametrize("d,n,m,p", [(3, 2, 2, 3), (2, 4, 4, 3), (3, 2, 2, 4), (3, 1, 3, 3),
                                     (2, 3, 2, 5)])
@pytest.mark.parametrize("kind", ["dd", "gauss"])
def test_split_element_kernel_matches(gpu, d, n, m, p, kind, monkeypatch):
    """The apply with a macro split over its row groups (csrc/element_split.cuh,
    MEHDG_ELEM_SPLIT=1; Q = 84, 91, 165, 220, 66) equals the warp-per-macro kernel
    (same substitution order: 1e-14) and the oracle, with and without row
    permutations; a solve through it converges to the same solution."""
    prob = S.make_problem(d, n, m, p, seed=21)
    if kind == "gauss":
        prob["A"] = np.random.default_rng(5).standard_normal(prob["A"].shape)
    sys0, cfg = condense_problem(prob)
    w0 = P.apply_schur(sys0, prob["uhat"])
    monkeypatch.setenv("MEHDG_ELEM_SPLIT", "1")
    sys1, _ = condense_problem(prob)
    w1 = P.apply_schur(sys1, prob["uhat"])
    assert rel(w1, w0) <= 1e-14
    if kind == "dd":
        o = SO.system_from_problem(prob).factorize()
        assert rel(w1, o.apply(prob["uhat"])) <= APPLY_TOL
        x1, info = P.gmres(P.SchurOperator(sys1), sys1.f_vec, cfg, precond=P.Preconditioner(sys1))
        x0, _ = P.gmres(P.SchurOperator(sys0), sys0.f_vec, cfg, precond=P.Preconditioner(sys0))
        assert info["converged"] and rel(x1, x0) <= SOLVE_TOL
