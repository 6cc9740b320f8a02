"""Pipelined LU (csrc/lu_pipe.cu) against the tile LU (bitwise) and LAPACK:
python tools/lu_pipe_check.py [Q ...].  Every 5th block is a plain Gaussian
block (row exchanges: handed back to the tile kernel), the others A + Q I."""
import os
import sys

import numpy as np
import scipy.linalg as sla

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402

Qs = [int(a) for a in sys.argv[1:]] or [33, 57, 84, 91, 115, 128, 165, 168, 200, 220, 224]
n = int(os.environ.get("CHECK_N", "24"))
bad = 0
for Q in Qs:
    prob = S.make_problem(2, n, 1, 1, seed=Q)
    rng = np.random.default_rng(Q)
    N, nc = prob["N"], prob["nc"]
    prob["Q"] = Q
    A = rng.standard_normal((N, Q, Q))
    A[np.arange(N) % 5 != 0] += Q * np.eye(Q)
    prob["A"] = A
    prob["Be"] = rng.standard_normal((N, nc, Q))
    prob["R_u"] = rng.standard_normal((N, Q))
    tables = {"nfe": 3, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
              "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
    out = {}
    for kind in ("tile", "pipe"):
        os.environ["MEHDG_LU"] = kind
        sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"],
                                 prob["D"], prob["R_hat"], P.SolverConfig(tol=1e-10), tables=tables)
        out[kind] = P.local_factors(sys_) + (P.apply_schur(sys_, np.ones(sys_.zhat)),)
        del sys_
    same = all(np.array_equal(a, b) for a, b in zip(out["tile"], out["pipe"]))
    err = 0.0
    pivok = True
    for e in range(0, N, max(1, N // 64)):
        ref_lu, ref_piv = sla.lu_factor(A[e])
        pivok &= np.array_equal(out["pipe"][1][e], ref_piv)
        err = max(err, np.abs(out["pipe"][0][e] - ref_lu).max() / np.abs(ref_lu).max())
    ok = same and pivok and err <= 1e-11
    bad += not ok
    print(f"Q={Q} N={N} bitwise_vs_tile={same} piv_vs_lapack={pivok} lu_err={err:.2e} "
          f"{'ok' if ok else 'FAIL'}", flush=True)
sys.exit(1 if bad else 0)
