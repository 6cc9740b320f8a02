"""Generate the golden fixtures in tests/golden/ from the REFERENCE itself.

Run in the build container, where /root/reference exists:

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference (`mehdg`, pure Python) is imported read-only and run on:
  * its own 2-D skeleton (build_structured_macro_mesh) and 3-D Kuhn tets;
  * the BASELINE synthetic operators of config c1 (whole vectors) and c2 / c3
    (strided samples + whole-vector checksums), injected through its
    LocalOperators / FaceOperator data contract exactly as SURVEY.md 8(c)
    describes (for d=3 the mesh is this repo's skeleton restatement, which the
    reference solver consumes duck-typed);
  * real HDG blocks from its own assembly (tanh benchmark, pivoting LU,
    chol-neg faces, C != B^T).
Outputs are small .npz files; the GPU box never reads /root/reference.
"""

from __future__ import annotations

import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, "/root/reference/pkg/src")

from mehdg import assembly as R_asm  # noqa: E402
from mehdg import mesh as R_mesh  # noqa: E402
from mehdg import schur_solver as R  # noqa: E402
from mehdg.bench import make_benchmark  # noqa: E402

from paper_2302_10917_b200 import synthetic as S  # noqa: E402
from paper_2302_10917_b200.mesh import build_structured_macro_mesh  # noqa: E402

STRIDE = 97


def ref_skeleton_tables(M):
    fl = np.array([(f.left.macro, f.left.edge) for f in M.skeleton], np.int64)
    fr = np.array([(f.right.macro, f.right.edge) if f.right else (-1, -1) for f in M.skeleton],
                  np.int64)
    tag = np.array([{"interior": 0, "D": 1, "N": 2}[f.tag] for f in M.skeleton], np.int64)
    ev = np.array([e.vertex_ids for e in M.macro_elements], np.int64)
    ef = np.array([[e.faces[k][0] for k in range(3)] for e in M.macro_elements], np.int64)
    lt = np.array([(f.left.t0, f.left.t1) for f in M.skeleton])
    rt = np.array([(f.right.t0, f.right.t1) if f.right else (0.0, 0.0) for f in M.skeleton])
    n = M.n
    verts = np.round(M.vertices * n).astype(np.int64)
    return dict(face_left=fl, face_right=fr, face_tag=tag, elem_verts=ev, elem_face=ef,
                face_left_t=lt, face_right_t=rt, verts=verts)


def make_skeletons():
    out = {}
    for n in (1, 2, 3, 4, 8):
        M = R_mesh.build_structured_macro_mesh(2, n, 2)
        for k, v in ref_skeleton_tables(M).items():
            out[f"n{n}_{k}"] = v
        out[f"n{n}_export_text"] = np.frombuffer(R_mesh.export_text(M).encode(), np.uint8)
    np.savez_compressed(HERE / "skeleton_2d.npz", **out)
    out = {}
    for n in (1, 2, 3, 4):
        K = R_mesh._build_kuhn_counting_mesh(n, 2)
        out[f"n{n}_elem_verts"] = np.array([e.vertex_ids for e in K.macro_elements], np.int64)
        out[f"n{n}_verts"] = np.round(K.vertices * n).astype(np.int64)
    np.savez_compressed(HERE / "kuhn_3d.npz", **out)


def inject(prob, mesh):
    """LocalOperators/FaceOperator of the reference from a synthetic problem."""
    t, nfe = prob["t"], prob["d"] + 1
    local_ops = []
    for e in range(prob["N"]):
        if prob["d"] == 2:
            fids = [mesh.macro_elements[e].faces[k][0] for k in range(3)]
        else:
            fids = [int(prob["mesh"].elem_face[e, k]) for k in range(nfe)]
        slots = [(fid, slice(k * t, (k + 1) * t)) for k, fid in enumerate(fids)]
        local_ops.append(R_asm.LocalOperators(
            macro_id=e, A=prob["A"][e], B=np.ascontiguousarray(prob["B"][e]),
            C=prob["C"][e], R_u=prob["R_u"][e], face_slots=slots, storage="dense"))
    face_ops = {}
    for face in mesh.skeleton:
        if face.tag == "D":
            continue
        u = prob["uidx"][face.id]
        face_ops[face.id] = R_asm.FaceOperator(face_id=face.id, D=prob["D"][u],
                                               R_hat=prob["R_hat"][u], tag=face.tag)
    return local_ops, face_ops


def run_reference(name, full: bool, gmres_tol=1e-10):
    d, n, m, p = S.CONFIGS[name]
    prob = S.make_problem(d, n, m, p, seed=0)
    mesh = R_mesh.build_structured_macro_mesh(2, n, m) if d == 2 else prob["mesh"]
    local_ops, face_ops = inject(prob, mesh)
    cfg = R.SolverConfig(tol=gmres_tol)
    t0 = time.time()
    sys_ = R.condense(mesh, local_ops, face_ops, cfg)
    t_cond = time.time() - t0
    u = prob["uhat"]
    t0 = time.time()
    w = R.apply_schur(sys_, u)
    t_apply = time.time() - t0
    z = R.apply_preconditioner(sys_, w)
    x, info = R.gmres(lambda v: R.apply_schur(sys_, v), sys_.f_vec, cfg,
                      precond=lambda v: R.apply_preconditioner(sys_, v))
    U = np.stack(R.reconstruct_interior(sys_, x))
    out = dict(f_norm=np.linalg.norm(sys_.f_vec), w_norm=np.linalg.norm(w),
               z_norm=np.linalg.norm(z), x_norm=np.linalg.norm(x), U_norm=np.linalg.norm(U),
               f_sum=sys_.f_vec.sum(), w_sum=w.sum(), z_sum=z.sum(), x_sum=x.sum(),
               U_sum=U.sum(), iterations=info["iterations"], converged=info["converged"],
               history=np.array(info["residual_history"]), zhat=sys_.zhat,
               t_condense=t_cond, t_apply=t_apply,
               offsets_start=np.array([sys_.offsets[f][0] for f in sorted(sys_.offsets)]),
               offsets_fid=np.array(sorted(sys_.offsets)))
    kinds = {"chol-neg": 0, "chol-pos": 1, "lu": 2}
    out["face_kinds"] = np.array([kinds[face_ops[f].factor_kind] for f in sorted(face_ops)])
    sel = np.arange(0, sys_.zhat, 1 if full else STRIDE)
    for k, v in dict(f=sys_.f_vec, w=w, z=z, x=x).items():
        out[k] = v[sel]
    out["sel"] = sel
    esel = np.arange(0, prob["N"], 1 if full else max(1, prob["N"] // 64))
    out["esel"] = esel
    out["U"] = U[esel]
    out["lu"] = np.stack([local_ops[e].lu[1][0] for e in esel[:8]])
    out["piv"] = np.stack([local_ops[e].lu[1][1] for e in esel[:8]])
    # face-plan encoding: (fid, start, left e, left slot start, right e, right slot start)
    fp = []
    for fid, start, nd, order in sys_.face_plan:
        row = [fid, start]
        for (e, sl) in order:
            row += [e, sl.start]
        row += [-1, -1] * (2 - len(order))
        fp.append(row)
    out["face_plan"] = np.array(fp, np.int64)
    out["gather_idx_concat"] = np.concatenate(sys_.gather_idx)
    # explicit Schur on random vectors (sampled rows)
    if full:
        Sx = R.assemble_schur_explicit(sys_)
        xs = np.random.default_rng(42).standard_normal((3, sys_.zhat))
        out["mb_x"] = xs
        out["mb_Sx"] = np.stack([Sx @ v for v in xs])
        out["mf_Sx"] = np.stack([R.apply_schur(sys_, v) for v in xs])
    np.savez_compressed(HERE / f"synthetic_{name}.npz", **out)
    print(name, "condense", round(t_cond, 2), "apply", round(t_apply, 3), "its",
          info["iterations"], info["converged"])


def _neumann_left(x):
    return "N" if x[0] < 1e-12 else "D"


def _g_neumann(x):
    x = np.atleast_2d(x)
    return np.sin(3.0 * x[:, 1]) + 0.5 * x[:, 0]


def run_real(n=2, m=2, p=2, supg=None, neumann=False, tag=""):
    """Reference assembly (tanh benchmark) -> blocks + reference results.
    supg: None or the SUPG variant; neumann: left side of the square tagged "N"
    with g_N = sin(3y) + x/2."""
    case = make_benchmark("tanh", 0.4, (1.0, 1.0))
    tagger = _neumann_left if neumann else None
    mesh = R_mesh.build_structured_macro_mesh(2, n, m, boundary_tagger=tagger)
    problem = case.problem()
    if neumann:
        problem = R_asm.ProblemData(a=problem.a, kappa=problem.kappa, f=problem.f,
                                    g_D=problem.g_D, g_N=_g_neumann)
    stab = R_asm.StabilizationConfig(supg=supg is not None,
                                     supg_variant=supg or "classical-minus")
    pool = R.WorkerPool(1)
    local_ops, face_ops = R.assemble_system(mesh, problem, stab, p, pool)
    cfg = R.SolverConfig(tol=1e-12)
    sys_ = R.condense(mesh, local_ops, face_ops, cfg, pool=pool)
    rng = np.random.default_rng(3)
    xs = rng.standard_normal((3, sys_.zhat))
    out = dict(
        A=np.stack([np.asarray(o.A.toarray() if hasattr(o.A, "toarray") else o.A)
                    for o in local_ops]),
        B=np.stack([o.B for o in local_ops]), C=np.stack([o.C for o in local_ops]),
        R_u=np.stack([o.R_u for o in local_ops]),
        D=np.stack([face_ops[f].D for f in sorted(face_ops)]),
        R_hat=np.stack([face_ops[f].R_hat for f in sorted(face_ops)]),
        face_ids=np.array(sorted(face_ops)),
        slot_faces=np.array([[fid for fid, _ in o.face_slots] for o in local_ops]),
        f=sys_.f_vec, xs=xs, w=np.stack([R.apply_schur(sys_, v) for v in xs]),
        z=np.stack([R.apply_preconditioner(sys_, v) for v in xs]),
        lu=np.stack([o.lu[1][0] for o in local_ops]) if local_ops[0].storage == "dense"
        else np.zeros(0),
        piv=np.stack([o.lu[1][1] for o in local_ops]) if local_ops[0].storage == "dense"
        else np.zeros(0),
        face_kinds=np.array([{"chol-neg": 0, "chol-pos": 1, "lu": 2}[face_ops[f].factor_kind]
                             for f in sorted(face_ops)]),
        n=n, m=m, p=p, supg=np.array(supg or ""), neumann=neumann,
        face_tags=np.array([face_ops[f].tag for f in sorted(face_ops)]))
    x, info = R.gmres(lambda v: R.apply_schur(sys_, v), sys_.f_vec, cfg,
                      precond=lambda v: R.apply_preconditioner(sys_, v))
    out.update(x=x, iterations=info["iterations"], history=np.array(info["residual_history"]),
               U=np.stack(R.reconstruct_interior(sys_, x)))
    np.savez_compressed(HERE / f"real_tanh_n{n}m{m}p{p}{tag}.npz", **out)
    print("real", n, m, p, tag, "zhat", sys_.zhat, "its", info["iterations"])


def mesh_arrays(M):
    """Plain-array description of a reference MacroMesh (incl. hanging faces) from
    which the tests rebuild a duck-typed mesh without importing the reference."""
    N, F = len(M.macro_elements), len(M.skeleton)
    faces = np.full((N, 6), -1, np.int64)
    for e in M.macro_elements:
        flat = [fid for k in range(3) for fid in e.faces[k]]
        faces[e.id, :len(flat)] = flat
    side = np.full((F, 2, 4), -1.0)
    for f in M.skeleton:
        for c, sd in enumerate(f.sides()):
            side[f.id, c] = (sd.macro, sd.edge, sd.t0, sd.t1)
    return dict(mesh_verts=np.stack([e.verts for e in M.macro_elements]),
                mesh_level=np.array([e.level for e in M.macro_elements]),
                mesh_m=np.array([e.m for e in M.macro_elements]),
                mesh_faces=faces,
                face_verts=np.stack([f.verts for f in M.skeleton]),
                face_side=side,
                face_tag=np.array([f.tag for f in M.skeleton]),
                face_mf=np.array([f.m_f for f in M.skeleton]),
                face_hanging=np.array([f.hanging for f in M.skeleton]))


def run_adaptive(n=2, m=2, p=2, marks=({0},), tag=""):
    """Reference blocks and results on a 2:1 refined mesh with hanging faces
    (mesh.py:428-463)."""
    case = make_benchmark("tanh", 0.4, (1.0, 1.0))
    M = R_mesh.build_structured_macro_mesh(2, n, m)
    for mk in marks:
        M = R_mesh.refine_macros(M, set(mk))
    pool = R.WorkerPool(1)
    stab = R_asm.StabilizationConfig()
    local_ops, face_ops = R.assemble_system(M, case.problem(), stab, p, pool)
    cfg = R.SolverConfig(tol=1e-12)
    sys_ = R.condense(M, local_ops, face_ops, cfg, pool=pool)
    rng = np.random.default_rng(3)
    xs = rng.standard_normal((3, sys_.zhat))
    nc_max = max(o.B.shape[1] for o in local_ops)
    nloc = local_ops[0].R_u.size

    def pad(b, axis):
        out = np.zeros((nloc, nc_max) if axis == 1 else (nc_max, nloc))
        if axis == 1:
            out[:, :b.shape[1]] = b
        else:
            out[:b.shape[0]] = b
        return out

    out = mesh_arrays(M)
    out.update(
        A=np.stack([np.asarray(o.A.toarray() if hasattr(o.A, "toarray") else o.A)
                    for o in local_ops]),
        B=np.stack([pad(o.B, 1) for o in local_ops]), C=np.stack([pad(o.C, 0) for o in local_ops]),
        nslot=np.array([len(o.face_slots) for o in local_ops]),
        R_u=np.stack([o.R_u for o in local_ops]),
        D=np.stack([face_ops[f].D for f in sorted(face_ops)]),
        R_hat=np.stack([face_ops[f].R_hat for f in sorted(face_ops)]),
        face_ids=np.array(sorted(face_ops)), f=sys_.f_vec, xs=xs,
        w=np.stack([R.apply_schur(sys_, v) for v in xs]),
        z=np.stack([R.apply_preconditioner(sys_, v) for v in xs]), n=n, m=m, p=p)
    x, info = R.gmres(lambda v: R.apply_schur(sys_, v), sys_.f_vec, cfg,
                      precond=lambda v: R.apply_preconditioner(sys_, v))
    out.update(x=x, iterations=info["iterations"], U=np.stack(R.reconstruct_interior(sys_, x)))
    np.savez_compressed(HERE / f"adaptive_tanh_n{n}m{m}p{p}{tag}.npz", **out)
    print("adaptive", n, m, p, tag, "N", len(local_ops), "hanging",
          int(sum(f.hanging for f in M.skeleton)), "zhat", sys_.zhat, "its", info["iterations"])


def make_fem_tables():
    """Reference-element tables of the device assembly (fem.py) from the
    reference's fem_basis / assembly helpers."""
    from mehdg import fem_basis as FB
    out = {}
    for m, p in ((1, 1), (2, 2), (3, 2), (2, 3), (1, 4), (2, 5)):
        for deg in (2 * p + 1, 2 * p + 2):
            key = f"m{m}p{p}d{deg}"
            rule = FB.quadrature_rule(2, deg)
            B = FB.LagrangeBasis(2, p)
            out[key + "_qp"] = rule.points_ref
            out[key + "_qw"] = rule.weights
            out[key + "_val"] = B.eval(rule.points_ref)
            out[key + "_grad"] = B.grad(rule.points_ref)
            out[key + "_hess"] = B.hess(rule.points_ref)
        dm = FB._patch_dof_map(m, p)
        out[f"m{m}p{p}_cell_map"] = np.array(dm.cell_maps)
        out[f"m{m}p{p}_edge_nodes"] = dm.edge_nodes
        mesh = R_mesh.build_structured_macro_mesh(2, 2, m)
        face = mesh.skeleton[1]
        side = face.sides()[0]
        s, w = R_asm._piecewise_quad(R_asm._face_breaks(face, side, m), p + 1)
        out[f"m{m}p{p}_face_s"] = s
        out[f"m{m}p{p}_face_w"] = w
        out[f"m{m}p{p}_trace"] = FB.TraceBasis(m, p).eval(s)
        g = lambda x: np.cos(2.0 * x[:, 0]) + x[:, 1] ** 2  # noqa: E731
        dfaces = [f for f in mesh.skeleton if f.tag == "D"][:4]
        out[f"m{m}p{p}_dface_verts"] = np.stack([f.verts for f in dfaces])
        out[f"m{m}p{p}_ghat"] = np.stack([R_asm.project_dirichlet(f, g, p) for f in dfaces])
    np.savez_compressed(HERE / "fem_tables.npz", **out)


if __name__ == "__main__":
    which = sys.argv[1:] or ["skeleton", "c1", "real", "c2", "c3"]
    if "skeleton" in which:
        make_skeletons()
    if "c1" in which:
        run_reference("c1", full=True)
    if "real" in which:
        run_real(2, 2, 2)
        run_real(3, 1, 3)
    if "fem" in which:
        make_fem_tables()
    if "adaptive" in which:  # hanging faces
        run_adaptive(2, 2, 2, marks=({0},))
        run_adaptive(2, 1, 3, marks=({0, 5}, {1}), tag="_2lev")
    if "asm" in which:  # device-assembly fixtures
        run_real(2, 2, 2, supg="classical-minus", tag="_supg")
        run_real(2, 2, 3, supg="paper-plus", tag="_supgplus")
        run_real(2, 3, 2, tag="")
        run_real(2, 2, 2, neumann=True, tag="_neumann")
    if "c2" in which:
        run_reference("c2", full=False)
    if "c3" in which:
        run_reference("c3", full=False)
