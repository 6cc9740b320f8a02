"""Oracle (test infrastructure): restatement of ``mehdg.schur_solver`` on arrays.

Every function follows ``/root/reference/pkg/src/mehdg/schur_solver.py`` line
for line in *algorithm* (per-macro LAPACK calls through scipy, the same
left-then-right face reduction, the same GMRES control flow), but consumes the
stacked-array data model of the B200 build instead of ``LocalOperators``
objects:

  A    (N, Q, Q)   reference ``op.A``            (assembly.py:63-72)
  B    (N, Q, nc)  reference ``op.B``  (= BASELINE B_e^T)
  C    (N, nc, Q)  reference ``op.C``  (= BASELINE B_e)
  R_u  (N, Q)
  D    (F, t, t)   ``FaceOperator.D`` of the F *unknown* faces (= BASELINE C_f)
  R_hat (F, t)
  elem_face (N, d+1)  unknown-face index of local face k, -1 if Dirichlet
  face_elem (F, 2), face_slot (F, 2)  (macro, local face) of left / right side

Slot k of a macro owns columns ``[k*t, (k+1)*t)`` of ``op.B`` -- the layout of
``face_slots`` in ``assemble_macro`` (assembly.py:241-249) on a conforming mesh.

It is the parity *checker* and the CPU baseline of bench.py; it is never on the
product path.
"""

from __future__ import annotations

import time

import numpy as np
import scipy.linalg as sla


class SingularLocalBlock(RuntimeError):
    """schur_solver.py:33-34"""


class SingularFaceBlock(RuntimeError):
    """schur_solver.py:37-38"""


FACE_KIND = {"chol-neg": 0, "chol-pos": 1, "lu": 2}


def factorize_local(A: np.ndarray):
    """``_factorize_local`` dense branch (schur_solver.py:105-111): LAPACK getrf
    with partial pivoting; singular if min|diag U| <= 1e-13 max|A|."""
    lu, piv = sla.lu_factor(A)
    diag = np.abs(np.diag(lu))
    singular = diag.min() <= 1e-13 * max(float(np.abs(A).max()), 1e-300)
    return lu, piv, bool(singular)


def factorize_face(D: np.ndarray):
    """``_factorize_face`` (schur_solver.py:130-147): chol(-D), chol(D), then LU.

    Returns (kind, sign, factor) or raises ValueError when singular."""
    for sign, kind in ((-1.0, "chol-neg"), (1.0, "chol-pos")):
        try:
            c = sla.cho_factor(sign * D)
        except np.linalg.LinAlgError:
            continue
        return kind, sign, ("chol", c)
    try:
        lu, piv = sla.lu_factor(D)
    except (np.linalg.LinAlgError, ValueError) as exc:
        raise ValueError("singular face block") from exc
    if np.abs(np.diag(lu)).min() < 1e-13 * max(np.abs(D).max(), 1e-300):
        raise ValueError("singular face block")
    return "lu", 1.0, ("lu", (lu, piv))


def solve_face(sign: float, fac, rhs):
    """``_solve_face`` (schur_solver.py:150-154)."""
    kind, f = fac
    if kind == "chol":
        return sign * sla.cho_solve(f, rhs)
    return sla.lu_solve(f, rhs)


def condense_tables(face_unknown: np.ndarray, elem_face_global: np.ndarray,
                    face_left: np.ndarray, face_right: np.ndarray, t: int) -> dict:
    """Integer tables of ``condense`` (schur_solver.py:198-241).

    face_unknown (F_all,) bool in skeleton order; elem_face_global (N, d+1)
    skeleton face ids; face_left/right (F_all, 2) = (macro, local face).
    Returns offsets start per unknown face, the unknown index map, the per-macro
    unknown-face table, gather_idx per macro and the left-then-right face plan.
    """
    F_all = face_unknown.size
    uidx = np.full(F_all, -1, dtype=np.int64)
    pos = 0
    starts = []
    for fid in range(F_all):  # skeleton order, skip "D" (schur_solver.py:198-206)
        if not face_unknown[fid]:
            continue
        uidx[fid] = len(starts)
        starts.append(pos)
        pos += t
    zhat = pos
    N, nf = elem_face_global.shape
    elem_face = np.where(elem_face_global >= 0, uidx[np.maximum(elem_face_global, 0)], -1)
    gather_idx = []
    gather_mask = []
    for e in range(N):  # schur_solver.py:214-223, face_slots in local-face order
        mask = np.zeros(nf * t, dtype=bool)
        idx = []
        for k in range(nf):
            u = elem_face[e, k]
            if u >= 0:
                mask[k * t:(k + 1) * t] = True
                idx.extend(range(starts[u], starts[u] + t))
        gather_mask.append(mask)
        gather_idx.append(np.array(idx, dtype=np.int64))
    Fu = len(starts)
    face_elem = np.full((Fu, 2), -1, dtype=np.int64)
    face_slot = np.full((Fu, 2), -1, dtype=np.int64)
    plan = []
    for fid in range(F_all):  # schur_solver.py:225-241: left side first, then right
        u = uidx[fid]
        if u < 0:
            continue
        order = []
        for col, side in enumerate((face_left[fid], face_right[fid])):
            if side[0] < 0:
                continue
            face_elem[u, col] = side[0]
            face_slot[u, col] = side[1]
            order.append((int(side[0]), slice(int(side[1]) * t, (int(side[1]) + 1) * t)))
        plan.append((fid, starts[u], t, order))
    return dict(uidx=uidx, starts=np.asarray(starts, dtype=np.int64), zhat=zhat,
                elem_face=elem_face, face_elem=face_elem, face_slot=face_slot,
                gather_idx=gather_idx, gather_mask=gather_mask, face_plan=plan)


class OracleSystem:
    """``CondensedSystem`` + ``condense`` restated on stacked arrays."""

    def __init__(self, A, B, C, R_u, D, R_hat, elem_face, face_elem, face_slot, t):
        self.A, self.B, self.C, self.R_u = A, B, C, R_u
        self.D, self.R_hat = D, R_hat
        self.elem_face = np.asarray(elem_face, dtype=np.int64)
        self.face_elem = np.asarray(face_elem, dtype=np.int64)
        self.face_slot = np.asarray(face_slot, dtype=np.int64)
        self.t = int(t)
        self.N, self.Q = A.shape[0], A.shape[1]
        self.F = D.shape[0]
        self.nc = B.shape[2]
        self.zhat = self.F * self.t
        self.counters = {"macro_apply": 0, "face_reduce": 0}
        self.timings = {}

    # -- condense (schur_solver.py:185-254) --------------------------------
    def factorize(self):
        t0 = time.perf_counter()
        self.lu = []
        for e in range(self.N):  # pool.map(_factorize_local) in macro order
            lu, piv, sing = factorize_local(self.A[e])
            if sing:
                raise SingularLocalBlock(e)
            self.lu.append((lu, piv))
        self.face_fac = []
        self.face_kind = np.empty(self.F, dtype=np.int64)
        for f in range(self.F):
            try:
                kind, sign, fac = factorize_face(self.D[f])
            except ValueError:
                raise SingularFaceBlock(f) from None
            self.face_fac.append((sign, fac))
            self.face_kind[f] = FACE_KIND[kind]
        self.timings["factorize"] = time.perf_counter() - t0
        return self

    def gather(self, uhat, e):
        """``CondensedSystem.gather`` (schur_solver.py:179-182)."""
        t = self.t
        ue = np.zeros(self.nc)
        for k, u in enumerate(self.elem_face[e]):
            if u >= 0:
                ue[k * t:(k + 1) * t] = uhat[u * t:(u + 1) * t]
        return ue

    def _face_reduce(self, base, vhat):
        """Step 4 / RHS reduction: seg = base_f - v_left - v_right (schur_solver.py:284-290, 247-253)."""
        t = self.t
        w = np.empty(self.zhat)
        for f in range(self.F):
            seg = base(f)
            for col in range(2):
                e = self.face_elem[f, col]
                if e < 0:
                    continue
                k = self.face_slot[f, col]
                seg = seg - vhat[e][k * t:(k + 1) * t]
            w[f * t:(f + 1) * t] = seg
            self.counters["face_reduce"] += 1
        return w

    def rhs(self):
        """f = R_hat - sum C A^-1 R_u (schur_solver.py:243-253)."""
        contrib = [self.C[e] @ sla.lu_solve(self.lu[e], self.R_u[e]) for e in range(self.N)]
        fvec = self._face_reduce(lambda f: self.R_hat[f].copy(), contrib)
        self.counters["face_reduce"] -= self.F
        return fvec

    def apply(self, uhat):
        """``apply_schur`` (schur_solver.py:267-293)."""
        vhat = []
        for e in range(self.N):
            ue = self.gather(uhat, e)
            x = self.B[e] @ ue                      # step 1
            y = sla.lu_solve(self.lu[e], x)         # step 2
            self.counters["macro_apply"] += 1
            vhat.append(self.C[e] @ y)              # step 3
        t = self.t
        return self._face_reduce(lambda f: self.D[f] @ uhat[f * t:(f + 1) * t], vhat)

    def precond(self, w):
        """``apply_preconditioner`` (schur_solver.py:296-305)."""
        t = self.t
        out = np.empty_like(w)
        for f in range(self.F):
            sign, fac = self.face_fac[f]
            out[f * t:(f + 1) * t] = solve_face(sign, fac, w[f * t:(f + 1) * t])
        return out

    def reconstruct(self, uhat):
        """``reconstruct_interior`` (schur_solver.py:423-431)."""
        return np.stack([
            sla.lu_solve(self.lu[e], self.R_u[e] - self.B[e] @ self.gather(uhat, e))
            for e in range(self.N)
        ]) if self.N else np.zeros((0, self.Q))

    def explicit_schur(self) -> np.ndarray:
        """Dense ``assemble_schur_explicit`` (schur_solver.py:388-420)."""
        S = np.zeros((self.zhat, self.zhat))
        t = self.t
        for e in range(self.N):
            mask = np.zeros(self.nc, dtype=bool)
            gi = []
            for k, u in enumerate(self.elem_face[e]):
                if u >= 0:
                    mask[k * t:(k + 1) * t] = True
                    gi.extend(range(u * t, (u + 1) * t))
            if not mask.any():
                continue
            Y = sla.lu_solve(self.lu[e], self.B[e][:, mask])
            S[np.ix_(gi, gi)] += -(self.C[e][mask] @ Y)
        for f in range(self.F):
            S[f * t:(f + 1) * t, f * t:(f + 1) * t] += self.D[f]
        return S


def gmres(apply_op, rhs, tol=1e-6, restart=100, maxiter=10000, precond=None):
    """Restarted left-preconditioned GMRES, MGS + Givens (schur_solver.py:308-385)."""
    n = rhs.size
    M = precond if precond is not None else (lambda v: v)
    x = np.zeros(n)
    history = []
    mb = M(rhs)
    bnorm = float(np.linalg.norm(mb))
    if bnorm == 0.0:
        return x, {"iterations": 0, "residual_history": [0.0], "converged": True}
    it = 0
    converged = False
    while it < maxiter and not converged:
        r = M(rhs - apply_op(x))
        beta = float(np.linalg.norm(r))
        if not history:
            history.append(beta)
        if beta / bnorm <= tol:
            converged = True
            break
        V = np.zeros((restart + 1, n))
        H = np.zeros((restart + 1, restart))
        cs = np.zeros(restart)
        sn = np.zeros(restart)
        g = np.zeros(restart + 1)
        V[0] = r / beta
        g[0] = beta
        k_used = 0
        breakdown = False
        for k in range(restart):
            wv = np.array(M(apply_op(V[k])), dtype=float)
            for i in range(k + 1):
                H[i, k] = float(V[i] @ wv)
                wv -= H[i, k] * V[i]
            H[k + 1, k] = float(np.linalg.norm(wv))
            if H[k + 1, k] > 1e-300:
                V[k + 1] = wv / H[k + 1, k]
            else:
                breakdown = True
            for i in range(k):
                tt = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = tt
            denom = float(np.hypot(H[k, k], H[k + 1, k]))
            if denom == 0.0:
                k_used = k + 1
                breakdown = True
                break
            cs[k], sn[k] = H[k, k] / denom, H[k + 1, k] / denom
            H[k, k] = denom
            H[k + 1, k] = 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            it += 1
            res = abs(g[k + 1])
            history.append(res)
            k_used = k + 1
            if res / bnorm <= tol:
                converged = True
                break
            if breakdown or it >= maxiter:
                break
        if k_used > 0:
            y = sla.solve_triangular(H[:k_used, :k_used], g[:k_used])
            x = x + V[:k_used].T @ y
        if breakdown and not converged:
            break
    if not converged:
        r = M(rhs - apply_op(x))
        converged = float(np.linalg.norm(r)) / bnorm <= tol
    return x, {"iterations": it, "residual_history": history, "converged": converged}


def system_from_problem(prob) -> OracleSystem:
    """OracleSystem from a ``paper_2302_10917_b200.synthetic`` problem dict."""
    return OracleSystem(prob["A"], prob["B"], prob["C"], prob["R_u"], prob["D"],
                        prob["R_hat"], prob["elem_face"], prob["face_elem"],
                        prob["face_slot"], prob["t"])


def slab_system(prob, e0: int, e1: int):
    """The oracle over the contiguous macro range [e0, e1) of a full-size problem
    (a mesh slab: SURVEY 8(e) partitions by contiguous macro ids).

    Keeps every unknown face touching a macro of the range, so each macro gathers
    its whole uhat; sides outside the range are dropped.  Returns
    ``(system, fidx, complete)``: ``fidx`` are the kept faces' global unknown-face
    ids and ``complete`` marks the faces all of whose sides lie in the range -- on
    those the slab's apply / RHS equal the whole mesh's (schur_solver.py:284-290,
    247-253 sum the sides of a face only)."""
    fe = np.asarray(prob["face_elem"], dtype=np.int64)
    fs = np.asarray(prob["face_slot"], dtype=np.int64)

    def inside(e):
        return (e >= e0) & (e < e1)

    touch = inside(fe[:, 0]) | inside(fe[:, 1])
    fidx = np.nonzero(touch)[0]
    remap = -np.ones(fe.shape[0], np.int64)
    remap[fidx] = np.arange(fidx.size)
    ef = np.asarray(prob["elem_face"][e0:e1], dtype=np.int64)
    ef = np.where(ef >= 0, remap[np.maximum(ef, 0)], -1)
    fe_s, fs_s = fe[fidx].copy(), fs[fidx].copy()
    out = ~inside(fe_s)
    fe_s[out], fs_s[out] = -1, -1
    fe_s[~out] -= e0
    complete = ~out[:, 0] & (~out[:, 1] | (fe[fidx, 1] < 0))
    o = OracleSystem(prob["A"][e0:e1], prob["B"][e0:e1], prob["C"][e0:e1], prob["R_u"][e0:e1],
                     prob["D"][fidx], prob["R_hat"][fidx], ef, fe_s, fs_s, prob["t"])
    return o, fidx, complete
