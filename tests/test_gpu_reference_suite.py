"""The reference's own hot-path tests, restated against the drop-in.

The blocks come from the UNMODIFIED reference package installed offline in
baseline/_ref (``mehdg.assembly.assemble_system``, ``mehdg.mesh``,
``mehdg.bench.make_benchmark``), exactly as its tests build them; every
``mehdg.schur_solver`` call of those tests goes to ``paper_2302_10917_b200``
instead.  Sources of the checks (the reference's test files):

* tests/test_schur_solver.py:104-113  matrix-free == explicit Schur
* tests/test_schur_solver.py:116-124  one apply = 2 macro tasks + 1 face reduction
* tests/test_schur_solver.py:127-135  D^-1 round trip
* tests/test_schur_solver.py:138-147  replaced face factors (identity blocks)
* tests/test_schur_solver.py:150-171  M S x = x - D^-1 C A^-1 B x (reads op.lu)
* tests/test_schur_solver.py:205-230  GMRES known answers
* tests/test_schur_solver.py:325-333  bitwise determinism across worker counts
* tests/test_acceptance.py:71-89, 122-135, 138-150 (criterion 5), 258-282
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np
import pytest

import paper_2302_10917_b200 as P

pytestmark = pytest.mark.gpu

_REF = Path(__file__).resolve().parent.parent / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (_REF / "mehdg").is_dir():
        pytest.skip("the reference is not installed in baseline/_ref")
    if str(_REF) not in sys.path:
        sys.path.insert(0, str(_REF))
    import mehdg.assembly as RA
    import mehdg.bench as RB
    import mehdg.mesh as RM

    return RA, RM, RB


def build_system(ref, n, m, p, case=None, workers=1, tol=1e-6):
    """test_schur_solver.py:30-37, the condense step replaced by the drop-in."""
    RA, RM, RB = ref
    case = case or RB.make_benchmark("poly2", 1.0, (1.0, 2.0))
    mesh = RM.build_structured_macro_mesh(2, n, m)
    local_ops, face_ops = _assemble(ref, mesh, case, p, workers)
    sys_ = P.condense(mesh, local_ops, face_ops, P.SolverConfig(tol=tol, workers=workers))
    return mesh, sys_


def _assemble(ref, mesh, case, p, workers=1):
    RA, _, _ = ref
    import mehdg.schur_solver as RS  # the reference's assemble_system (block assembly)

    pool = RS.WorkerPool(workers)
    try:
        return RS.assemble_system(mesh, case.problem(), RA.StabilizationConfig(), p, pool)
    finally:
        pool.close()


@pytest.mark.parametrize("n,m,p", [(2, 1, 1), (2, 2, 2), (3, 2, 3)])
def test_matrix_free_matches_explicit(gpu, ref, n, m, p):
    _, sys_ = build_system(ref, n, m, p)
    S = P.assemble_schur_explicit(sys_)
    rng = np.random.default_rng(17)
    for _ in range(5):
        x = rng.standard_normal(sys_.zhat)
        mf = P.apply_schur(sys_, x)
        mb = S @ x
        assert np.linalg.norm(mf - mb) <= 1e-10 * np.linalg.norm(mb)


def test_two_macro_call_counts(gpu, ref):
    _, sys_ = build_system(ref, 1, 1, 1)
    sys_.counters["macro_apply"] = 0
    sys_.counters["face_reduce"] = 0
    P.apply_schur(sys_, np.ones(sys_.zhat))
    assert sys_.counters["macro_apply"] == 2
    assert sys_.counters["face_reduce"] == 1


def test_preconditioner_round_trip(gpu, ref):
    _, sys_ = build_system(ref, 2, 2, 2)
    rng = np.random.default_rng(1)
    x = rng.standard_normal(sys_.zhat)
    w = np.empty_like(x)
    for fid, start, nd, _ in sys_.face_plan:
        w[start:start + nd] = sys_.face_ops[fid].D @ x[start:start + nd]
    back = P.apply_preconditioner(sys_, w)
    assert np.abs(back - x).max() < 1e-12 * max(1.0, np.abs(x).max())


def test_preconditioner_identity_blocks(gpu, ref):
    """Face factors replaced after condense are what the preconditioner applies
    (also inside GMRES)."""
    import scipy.linalg as sla

    _, sys_ = build_system(ref, 2, 1, 1)
    for op in sys_.face_ops.values():
        op.D = np.eye(op.D.shape[0])
        op.factor = ("chol", 1.0, sla.cho_factor(op.D))
        op.factor_kind = "chol-pos"
    x = np.arange(1.0, sys_.zhat + 1.0)
    assert np.array_equal(P.apply_preconditioner(sys_, x), x)


def test_preconditioned_operator_structure(gpu, ref):
    """M S x = x - D^-1 (C A^-1 B) x against a dense oracle built from op.lu."""
    import scipy.linalg as sla

    _, sys_ = build_system(ref, 1, 1, 1)
    S = P.assemble_schur_explicit(sys_).toarray()
    op = sys_.local_ops
    D = np.zeros((sys_.zhat, sys_.zhat))
    CAB = np.zeros((sys_.zhat, sys_.zhat))
    for fid, start, nd, _ in sys_.face_plan:
        D[start:start + nd, start:start + nd] = sys_.face_ops[fid].D
    for e, o in enumerate(op):
        assert o.lu[0] == "dense"
        mask = sys_.gather_mask[e]
        gi = sys_.gather_idx[e]
        blk = o.C[mask] @ sla.lu_solve(o.lu[1], o.B[:, mask])
        CAB[np.ix_(gi, gi)] += blk
    rng = np.random.default_rng(4)
    x = rng.standard_normal(sys_.zhat)
    lhs = P.apply_preconditioner(sys_, P.apply_schur(sys_, x))
    rhs = x - np.linalg.solve(D, CAB @ x)
    assert np.abs(lhs - rhs).max() < 1e-11 * max(1.0, np.abs(rhs).max())
    assert np.abs(S - (D - CAB)).max() < 1e-11 * np.abs(S).max()


def test_gmres_known_answers(gpu):
    x, info = P.gmres(lambda v: v, np.array([3.0, -1.0, 2.0]), P.SolverConfig(tol=1e-12))
    assert info["converged"] and info["iterations"] == 1
    d = np.arange(1.0, 6.0)
    x, info = P.gmres(lambda v: d * v, np.ones(5), P.SolverConfig(tol=1e-12))
    assert info["converged"] and info["iterations"] <= 5
    assert np.abs(x - 1.0 / d).max() < 1e-10
    d = np.arange(1.0, 101.0)
    x, info = P.gmres(lambda v: d * v, np.ones(100),
                      P.SolverConfig(tol=1e-14, maxiter=3, restart=3))
    assert not info["converged"] and info["iterations"] == 3
    assert len(info["residual_history"]) >= 2
    x, info = P.gmres(lambda v: 2 * v, np.zeros(4), P.SolverConfig())
    assert info["converged"] and np.abs(x).max() == 0.0


def _solve(ref, case, n, m, p, **kw):
    """test_schur_solver.py:297-302 / the acceptance tests' solve(): the
    reference's assembly, the drop-in's condense / GMRES / reconstruct."""
    _, RM, _ = ref
    mesh = RM.build_structured_macro_mesh(2, n, m)
    cfg = P.SolverConfig(tol=kw.pop("tol", 1e-12), mode=kw.pop("mode", "mb"),
                         workers=kw.pop("workers", 1))

    def assemble(mesh_, problem, stab, p_):
        return _assemble(ref, mesh_, case, p_, cfg.workers)

    sol, sys_ = P.solve(mesh, case.problem(), None, cfg, p, assemble=assemble)
    return mesh, sol, sys_


def test_determinism_across_workers(gpu, ref):
    _, _, RB = ref
    case = RB.make_benchmark("poly2", 1.0, (1.0, 2.0))
    base = None
    for workers in (1, 2, 8):
        _, sol, _ = _solve(ref, case, 2, 2, 2, workers=workers, tol=1e-10)
        if base is None:
            base = sol.uhat
        else:
            assert np.array_equal(base, sol.uhat)


def test_acceptance_criterion_02(gpu, ref):
    """Matrix-free operator == assembled Schur on 20 random vectors (tanh)."""
    RA, RM, RB = ref
    case = RB.make_benchmark("tanh", 0.4, (1.0, 1.0))
    rng = np.random.default_rng(42)
    worst = 0.0
    for n, m, p in ((2, 1, 1), (2, 2, 2), (3, 2, 3)):
        mesh = RM.build_structured_macro_mesh(2, n, m)
        lops, fops = _assemble(ref, mesh, case, p)
        sys_ = P.condense(mesh, lops, fops, P.SolverConfig())
        S = P.assemble_schur_explicit(sys_)
        for _ in range(20):
            x = rng.standard_normal(sys_.zhat)
            diff = np.abs(P.apply_schur(sys_, x) - S @ x).max()
            worst = max(worst, diff / max(np.abs(S @ x).max(), 1.0))
    assert worst <= 1e-10


def test_acceptance_criterion_04(gpu, ref):
    """Matrix-based and matrix-free GMRES take the same iterations (+-1) at
    loose and tight tolerances (test_acceptance.py:122-135, via run_compare's
    solves, bench.py:236-260)."""
    _, _, RB = ref
    case = RB.make_benchmark("tanh", 0.4, (1.0, 1.0))
    for m in (1, 2):
        for tol in (1e-2, 1e-6):
            it = {}
            for mode in ("mb", "mf"):
                _, sol, _ = _solve(ref, case, 8 // m, m, 2, tol=tol, mode=mode)
                it[mode] = sol.report.iterations
            assert abs(it["mb"] - it["mf"]) <= 1, (m, tol, it)


def test_acceptance_criterion_05(gpu, ref):
    """Larger macros shrink the trace system at fixed resolution; sizes match
    the exact per-face count (sum over unknown faces of m_f p + 1)."""
    _, RM, RB = ref
    case = RB.make_benchmark("poly2", 1.0, (1.0, 2.0))
    p = 2
    sizes = []
    for n, m in ((8, 1), (4, 2), (2, 4)):
        mesh, sys_ = build_system(ref, n, m, p, case=case)
        expect = sum(f.m_f * p + 1 for f in mesh.skeleton if f.tag != "D")
        assert sys_.zhat == expect
        sizes.append(sys_.zhat)
    assert sizes[0] > sizes[1] > sizes[2]


def test_acceptance_criterion_10(gpu, ref):
    """Bitwise-identical traces for 1/2/8 workers; the load-balance factor of
    the report is in (0, 1] and >= 0.8 (one device: the whole solve on it)."""
    _, _, RB = ref
    case = RB.make_benchmark("tanh", 0.4, (1.0, 1.0))
    uh, lbf8 = {}, 0.0
    for workers in (1, 2, 8):
        _, sol, _ = _solve(ref, case, 4, 2, 2, tol=1e-6, mode="mf", workers=workers)
        uh[workers] = sol.uhat
        if workers == 8:
            lbf8 = sol.report.lbf
    assert np.array_equal(uh[1], uh[2]) and np.array_equal(uh[1], uh[8])
    assert 0.0 < lbf8 <= 1.0 and lbf8 >= 0.8
