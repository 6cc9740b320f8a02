"""Split element kernel (csrc/element_split.cuh, MEHDG_ELEM_SPLIT=1) against the
warp-per-macro kernel and the oracle: python tools/split_check.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2302_10917_b200 as P  # noqa: E402
from paper_2302_10917_b200 import synthetic as S  # noqa: E402
from oracle import solver_oracle as SO  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


bad = 0
shapes = [(3, 2, 2, 3), (2, 4, 4, 3), (3, 1, 2, 4), (3, 2, 2, 4), (3, 1, 3, 3), (2, 3, 2, 5),
          (3, 4, 2, 3), (2, 12, 4, 3)]
for d, n, m, p in shapes:
    for kind in ("dd", "gauss"):
        prob = S.make_problem(d, n, m, p, seed=21)
        if kind == "gauss":
            prob["A"] = np.random.default_rng(5).standard_normal(prob["A"].shape)
        tables = {"nfe": d + 1, "elem_ufac": prob["elem_face"], "face_elem": prob["face_elem"],
                  "face_slot": prob["face_slot"], "uidx": prob["uidx"], "F": prob["F"]}
        out = {}
        for split in ("0", "1"):
            os.environ["MEHDG_ELEM_SPLIT"] = split
            sys_ = P.condense_arrays(prob["mesh"], prob["A"], None, prob["Be"], prob["R_u"],
                                     prob["D"], prob["R_hat"], P.SolverConfig(tol=1e-10),
                                     tables=tables)
            out[split] = P.apply_schur(sys_, prob["uhat"])
            if split == "1":
                x, info = P.gmres(P.SchurOperator(sys_), sys_.f_vec, P.SolverConfig(tol=1e-10),
                                  precond=P.Preconditioner(sys_))
            del sys_
        tol = 1e-12 if kind == "dd" else 1e-9
        r01 = rel(out["1"], out["0"])
        ro = rel(out["1"], SO.system_from_problem(prob).factorize().apply(prob["uhat"])) if prob["N"] <= 400 else float("nan")
        ok = r01 <= tol and (not ro == ro or ro <= tol) and info["converged"]
        bad += not ok
        print(f"d={d} n={n} m={m} p={p} Q={prob['Q']} nc={prob['nc']} N={prob['N']} {kind}: "
              f"split vs warp-per-macro {r01:.2e}, vs oracle {ro:.2e}, gmres {info['iterations']} it "
              f"{'ok' if ok else 'FAIL'}", flush=True)
sys.exit(1 if bad else 0)
